for r in 1 2; do for t in base b2x2 b2x2p b2x4 b3x2 b4x2; do
  timeout 300 python tools/run_variant.py $t --no-cpu --no-e2e --no-other --schedule classic 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['value'],2), [round(x,4) for x in d['roofline']['phase_ms_per_iter']], d['clocks']['sm_mhz'])" >> gpurun_out/h3var2.log 2>&1
done; done
