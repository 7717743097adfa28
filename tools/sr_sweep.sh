#!/bin/bash
# SR kernel geometry sweep at 600x595x1536 mixed (bench.py, no e2e / cpu legs)
mkdir -p gpurun_out
for t in "16,2,2,64" "16,2,2,320,64,256,16" "16,2,2,320,64,256,8" "8,2,2,320,64,256,16" "8,3,2,320,64,256,16"; do
  echo "== $t"
  timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 --sr-tiling $t | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['config']['hbm_frac_whole_step'])"
done
echo "== classic"
timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 --schedule classic | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['roofline']['frac'])"
