# fp32 SR sweep: chunk plans in the bench (two interleaved rounds) and their DRAM bytes under ncu
mkdir -p gpurun_out
for r in 1 2; do for c in default 32,0,32 48,0,48 96,0,96 128,0,128 160,320,64 96,192,48; do
  a=""; [ "$c" != default ] && a="--sr-chunks $c"
  timeout 300 python bench.py --precision fp32 --no-cpu --no-e2e --no-other --no-2d --no-tts --schedule sr $a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c', round(d['value'],2), round(r['avg_launch_ms'],4), round(r['frac'],4), d['clocks']['sm_mhz'])" >> gpurun_out/sr32_chunks.log 2>&1
done; done
for c in default 32,0,32 128,0,128 160,320,64; do
  a=""; [ "$c" != default ] && a="--sr-chunks $c"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_sr$' -s 2 -c 2 --csv python bench.py --precision fp32 --steps 1 --warmup 1 --maxit 4 --no-cpu --no-e2e --no-other --no-2d --no-tts --schedule sr $a > gpurun_out/sr32_ncu_${c//,/_}.csv 2>/dev/null
done
