# SR sweep: uniform z-chunk length at config 3 (sweep ms); "def" = library default plan
for v in "" "--operator poisson-const" "--precision fp32"; do for zc in def 16 24 32 48 64 96 160; do
  T=""; [ "$zc" != "def" ] && T="--sr-tiling 0,0,0,$zc"
  timeout 300 python bench.py --no-cpu --no-e2e --no-other --schedule sr $v $T 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print('[$v] zc=$zc', round(d['value'],2), round(r.get('avg_launch_ms',0),4), round(r.get('frac',0),4), d['clocks']['sm_mhz'])" >> gpurun_out/srzc.log 2>&1
done; done
