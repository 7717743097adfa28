# SR sweep geometry (by, stages, cstages, zc=keep, pack) at config 3, per operator / precision
for v in "--operator poisson-const" "" "--precision fp32"; do for c in def 8,3,2,0,16 8,3,2,0,8 8,2,2,0,8 16,2,2,0,8 8,3,3,0,16 16,2,2,0,16 8,2,2,0,16; do
  T=""; [ "$c" != "def" ] && T="--sr-tiling $c"
  timeout 300 python bench.py --no-cpu --no-e2e --no-other --schedule sr $v $T 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline',{}); print('[$v] $c', round(d['value'],2), round(r.get('avg_launch_ms',0),4), round(r.get('frac',0),4), d['clocks']['sm_mhz'])" >> gpurun_out/srcfg.log 2>&1
done; done
