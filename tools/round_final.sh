#!/bin/bash
# Round-end refresh in one GPU call: smoke, the GPU suite, the default bench and its variants.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
: > gpurun_out/bench_variants.jsonl
for v in "--precision fp32" "--operator poisson-const" "--schedule sr" "--dots half" "--operator poisson-const --precision fp32"; do
  echo "== $v" >> gpurun_out/bench_variants.jsonl
  timeout 600 python bench.py --no-cpu --no-2d --no-tts $v 2>&1 | tail -1 >> gpurun_out/bench_variants.jsonl
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
