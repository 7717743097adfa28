# constant-coefficient SR sweep occupancy experiment: base vs a build without the
# r_hat / x TMA rings (70 KB at 8-row tiles, 2 input stages: 3 CTAs per SM)
mkdir -p gpurun_out
for r in 1 2; do
for v in "base:" "base:--sr-tiling 8,2,2,160,16" "norh:--sr-tiling 8,2,2,160,16" "norh:--sr-tiling 8,3,2,160,16" "norh:"; do
  t=${v%%:*}; a=${v#*:}
  timeout 300 python tools/run_variant.py $t --no-cpu --no-e2e --no-other --no-2d --schedule sr --operator poisson-const $a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$t', '$a', round(d['value'],2), round(r['avg_launch_ms'],4), round(r['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/ccocc.log 2>&1
done; done
