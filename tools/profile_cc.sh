#!/bin/bash
# full-size ncu captures of the classic scalar-coupling kernels (constant operator, NEXT-4)
mkdir -p gpurun_out
N="--clock-control none"
K="python bench.py --steps 1 --warmup 1 --maxit 2 --no-e2e --no-cpu --no-other --no-2d --schedule classic --operator poisson-const"
$K > gpurun_out/cc_k.log 2>&1 && ncu --set full $N -k regex:'k_stencil|k_h3' -s 3 -c 3 -o gpurun_out/cc_full $K > gpurun_out/cc_full.log 2>&1
ncu -i gpurun_out/cc_full.ncu-rep --page raw --csv > gpurun_out/cc_full_raw.csv 2>/dev/null
ncu -i gpurun_out/cc_full.ncu-rep --page details --csv > gpurun_out/cc_full_details.csv 2>/dev/null
rm -f gpurun_out/cc_full.ncu-rep
