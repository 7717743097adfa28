# SR sweep vs the TMA L2 promotion of its tensor maps (0 none, 1 64 B, 2 128 B, 3 256 B = default):
# timing (two interleaved rounds) and DRAM bytes of two sweeps under ncu
mkdir -p gpurun_out
for r in 1 2; do for p in 0 1 2 3; do
  timeout 300 python bench.py --no-cpu --no-e2e --no-other --no-2d --schedule sr --set-option TMA_L2_PROMOTION=$p 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('promo=$p', round(d['value'],2), round(r['avg_launch_ms'],4), round(r['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/sr_promo.log 2>&1
done; done
for p in 0 1 2 3; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_sr$' -s 2 -c 2 --csv python bench.py --steps 1 --warmup 1 --maxit 4 --no-cpu --no-e2e --no-other --no-2d --schedule sr --set-option TMA_L2_PROMOTION=$p > gpurun_out/sr_promo_ncu_$p.csv 2>/dev/null
done
