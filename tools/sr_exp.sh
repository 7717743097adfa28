#!/bin/bash
# build-variant experiments for the SR kernel: tools/sr_exp.sh "<flags1>|<flags2>|..." "<bench args>"
mkdir -p gpurun_out
IFS='|' read -ra VARS <<< "$1"
for v in "${VARS[@]}"; do
  echo "== variant: [$v] $2"
  STEN_NVCC_EXTRA="$v" python -c "from paper_2010_03660_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 $2 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value'],2), round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_ms'],4))"
done
python -c "from paper_2010_03660_b200 import build; build.build(force=True)" > /dev/null 2>&1
