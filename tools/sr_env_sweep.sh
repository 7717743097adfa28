#!/bin/bash
# SR sweep over layout / TMA-promotion knobs (env) at 600x595x1536 mixed
mkdir -p gpurun_out
run() {
  echo "== $*"
  env "$@" timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_ms'],4))"
}
run STEN_TMA_PROMO=3
run STEN_TMA_PROMO=2
run STEN_TMA_PROMO=1
run STEN_TMA_PROMO=0
run STEN_PITCH_ALIGN=8
run STEN_PITCH_ALIGN=32
run STEN_PITCH_ALIGN=8 STEN_TMA_PROMO=0
run STEN_SR_TILING=16,3,2,192
run STEN_SR_TILING=16,3,2,96
