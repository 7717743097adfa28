# SR chunk plans in the bench (graph-replayed 100-iteration solves): zc,tail_planes,zc_tail; two
# interleaved rounds; one line per run: plan, value, sweep ms, frac, SM clock
mkdir -p gpurun_out
for r in 1 2; do for c in default 64,0,64 48,0,48 96,0,96 64,192,32 96,288,48 128,256,64 80,320,40; do
  a=""; [ "$c" != default ] && a="--sr-chunks $c"
  timeout 300 python bench.py --no-cpu --no-e2e --no-other --no-2d --no-tts --schedule sr $a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', round(d['value'],2), round(r['avg_launch_ms'],4), round(r['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/sr_chunks.log 2>&1
done; done
