# tensor-core Gram for the SR sweep's twelve sums (STEN_SR_MMA=1 build 'mma') against the FMA dots:
# the SR / const / full-size SR tests on the variant, then paired bench runs (fields and constant)
mkdir -p gpurun_out
STEN_TEST_VARIANT=mma timeout 900 python -m pytest tests/test_gpu_sr.py tests/test_gpu_const.py tests/test_gpu_fullsize_sr.py -q -x > gpurun_out/mma_tests.log 2>&1; echo rc=$? >> gpurun_out/mma_tests.log
for r in 1 2; do for t in base mma; do for op in fields poisson-const; do
  timeout 300 python tools/run_variant.py $t --no-cpu --no-e2e --no-other --no-2d --no-tts --schedule sr --operator $op 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$t $op', round(d['value'],2), round(r['avg_launch_ms'],4), round(r['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/mma.log 2>&1
done; done; done
