#!/bin/bash
# Everything the round's numbers come from, in one GPU call: smoke, GPU tests, the
# default bench and its variants, SR profiles, small configs, CPU oracle timing.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
python bench.py > gpurun_out/bench.log 2>&1
for v in "--precision fp32" "--operator poisson-const" "--schedule classic" "--dots half" "--operator poisson-const --precision fp32"; do
  echo "== $v" >> gpurun_out/bench_variants.log
  python bench.py --no-cpu $v 2>&1 | tail -1 >> gpurun_out/bench_variants.log
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
./tools/profile_sr.sh > /dev/null 2>&1
python tools/small_configs.py > gpurun_out/small.log 2>&1; cp profiles/r1_small.md gpurun_out/ 2>/dev/null
timeout 1500 python tools/cpu_oracle_study.py > gpurun_out/cpu_oracle.log 2>&1; cp profiles/r1_cpu_oracle.md gpurun_out/ 2>/dev/null
ls gpurun_out
