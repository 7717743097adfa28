#!/bin/bash
# full-size ncu capture of the fp32 classic kernels (H1, H2, H3) and the fp32 constant-coefficient ones
mkdir -p gpurun_out
N="--clock-control none"
K="python bench.py --precision fp32 --steps 1 --warmup 1 --maxit 2 --no-e2e --no-cpu --no-other --no-2d --no-tts --schedule classic"
$K > gpurun_out/f32_k.log 2>&1 && ncu --set full $N -k regex:'k_stencil|k_h3' -s 3 -c 3 -o gpurun_out/f32_full $K > gpurun_out/f32_full.log 2>&1
ncu -i gpurun_out/f32_full.ncu-rep --page raw --csv > gpurun_out/f32_full_raw.csv 2>/dev/null
rm -f gpurun_out/f32_full.ncu-rep
C="$K --operator poisson-const"
$C > gpurun_out/f32c_k.log 2>&1 && ncu --set full $N -k regex:'k_stencil|k_h3' -s 3 -c 3 -o gpurun_out/f32c_full $C > gpurun_out/f32c_full.log 2>&1
ncu -i gpurun_out/f32c_full.ncu-rep --page raw --csv > gpurun_out/f32c_full_raw.csv 2>/dev/null
rm -f gpurun_out/f32c_full.ncu-rep
