#!/bin/bash
# SR bench under env variants (layout / geometry knobs) at 600x595x1536 mixed
mkdir -p gpurun_out
run() {
  echo "== $*"
  env "$@" timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 $BENCH_ARGS | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_ms'],4))"
}
for v in "$@"; do run $v; done
