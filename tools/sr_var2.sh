# SR build variants, any bench arguments: bash tools/sr_var2.sh "<bench args>" tag1 tag2 ...
# (two rounds, interleaved; one line per run: tag, value, sweep ms, frac, SM clock)
args="$1"; shift
for r in ${ROUNDS:-1 2}; do for t in "$@"; do
  timeout 300 python tools/run_variant.py $t --no-cpu --no-e2e --no-other --no-2d --schedule sr $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$t', '$args', round(d['value'],2), round(r['avg_launch_ms'],4), round(r['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/srvar2.log 2>&1
done; done
