# fp32 classic on the constant operator (scalar couplings): z-chunk sweep, phase ms per iteration
mkdir -p gpurun_out
for r in 1 2; do for z in 16 20 32 48 64; do
  timeout 300 python bench.py --precision fp32 --operator poisson-const --no-cpu --no-e2e --no-other --no-2d --no-tts --tiling 64,16,$z,0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('zc=$z', round(d['value'],2), [round(x,4) for x in r['phase_ms_per_iter']], round(r['whole_step_frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/fp32c_zc.log 2>&1
done; done
