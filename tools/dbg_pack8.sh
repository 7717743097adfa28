#!/bin/bash
for v in 1; do
  STEN_NVCC_EXTRA="-DSTEN_DBG_STOP=$v" python -c "from paper_2010_03660_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build $v failed"; continue; }
  echo "== stop $v"; timeout 120 python tools/dbg_pack8.py mixed 2>&1 | tail -1
done
python -c "from paper_2010_03660_b200 import build; build.build(force=True)" > /dev/null 2>&1
