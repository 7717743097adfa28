# SR build variants at config 3 (sweep ms, roofline frac, clock): bash tools/sr_var.sh tag1 tag2 ...
for r in 1 2; do for t in "$@"; do
  timeout 300 python tools/run_variant.py $t --no-cpu --no-e2e --no-other --schedule sr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$t', round(d['value'],2), round(r['avg_launch_ms'],4), round(r['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/srvar.log 2>&1
done; done
