# classic kernels: z-chunk length sweep at config 3 (phase ms per iteration); "def" = library default
for p in mixed fp32; do for zc in def 12 16 20 24 32 48; do
  T=""; [ "$zc" != "def" ] && T="--tiling 128,16,$zc,0"; [ "$zc" != "def" ] && [ "$p" = fp32 ] && T="--tiling 64,16,$zc,0"
  timeout 300 python bench.py --no-cpu --no-e2e --no-other --schedule classic --precision $p $T 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$p zc=$zc', round(d['value'],2), [round(x,4) for x in d['roofline']['phase_ms_per_iter']], d['clocks']['sm_mhz'])" >> gpurun_out/zc2.log 2>&1
done; done
