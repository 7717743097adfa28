# classic schedule on the constant operator (NEXT-4, 17 passes): z-chunk sweep of the
# scalar-coupling H1 / H2 kernels (zc = zc2 = Z via --tiling 128,16,Z,0); one line per run
mkdir -p gpurun_out
for r in 1 2; do for z in 10 20 40 80 160; do
  timeout 300 python bench.py --no-cpu --no-e2e --no-other --no-2d --operator poisson-const --tiling 128,16,$z,0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('zc=$z', round(d['value'],2), [round(x,4) for x in r['phase_ms_per_iter']], round(r['whole_step_frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/cc_zc.log 2>&1
done; done
