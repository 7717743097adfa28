# fp32 element-wise work as FFMA2 (two RN fp32 FMAs per instruction) against scalar FFMA (build 'noff2'):
# the fp32 GPU tests on the product build, then paired fp32 bench runs of both schedules
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ff2_tests.log 2>&1; echo rc=$? >> gpurun_out/ff2_tests.log
for r in 1 2; do for t in base noff2; do
  timeout 300 python tools/run_variant.py $t --precision fp32 --no-cpu --no-e2e --no-2d --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; s=d['sr']; print('$t', round(d['value'],2), [round(x,4) for x in r['phase_ms_per_iter']], round(r['whole_step_frac'],4), 'sr', round(s['value'],2), round(s['roofline']['avg_launch_ms'],4), round(s['roofline']['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/ff2.log 2>&1
  timeout 300 python tools/run_variant.py $t --precision fp32 --operator poisson-const --no-cpu --no-e2e --no-2d --no-tts 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; s=d['sr']; print('$t const', round(d['value'],2), [round(x,4) for x in r['phase_ms_per_iter']], round(r['whole_step_frac'],4), 'sr', round(s['value'],2), round(s['roofline']['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/ff2.log 2>&1
done; done
