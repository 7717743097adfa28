# H3 bulk stream: evict-first L2 hint on its input copies (h3hint) and 4 x 256-vector stages (h3ns4)
# against the product build; paired classic runs, phase ms per iteration
mkdir -p gpurun_out
for r in 1 2 3; do for t in base h3hint h3ns4; do
  timeout 300 python tools/run_variant.py $t --no-cpu --no-e2e --no-other --no-2d --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$t', round(d['value'],2), [round(x,4) for x in r['phase_ms_per_iter']], round(r['whole_step_frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/h3hint.log 2>&1
done; done
