# classic half-dot H3: k_h3s_half (bulk ring, default) vs the tile z-march (h3zold) and a 2-stage /
# 3 CTA-per-SM ring (h3s2); one line per run: tag, value, phase ms (H1, H2, H3), SM clock
mkdir -p gpurun_out
for r in 1 2; do for t in base h3zold h3s2; do
  timeout 300 python tools/run_variant.py $t --no-cpu --no-e2e --no-other --no-2d --schedule classic --dots half 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$t', round(d['value'],2), [round(x,4) for x in r['phase_ms_per_iter']], d['clocks']['sm_mhz'])" >> gpurun_out/h3s.log 2>&1
done; done
