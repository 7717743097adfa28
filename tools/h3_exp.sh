for f in "" "-DSTEN_H3_QUAD=1" "" "-DSTEN_H3_QUAD=1"; do
  for b in 64 16; do
  STEN_NVCC_EXTRA="$f" python -c "from paper_2010_03660_b200 import build; build.build(force=True)" >/dev/null 2>&1
  STEN_EW_BPS=$b python bench.py --no-cpu --no-e2e --schedule classic 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"[$f] bps=$b\", round(d[\"value\"],2), [round(x,4) for x in d[\"roofline\"][\"phase_ms_per_iter\"]])"
  done
done
