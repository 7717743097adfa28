#!/bin/bash
# full-size ncu capture of the classic half-dot kernels (R28): k_stencil<half, H1/H2, HD> and k_h3s_half
mkdir -p gpurun_out
N="--clock-control none"
K="python bench.py --steps 1 --warmup 1 --maxit 2 --no-e2e --no-cpu --no-other --no-2d --no-tts --schedule classic --dots half"
$K > gpurun_out/hd_k.log 2>&1 && ncu --set full $N -k regex:'k_stencil|k_h3' -s 3 -c 3 -o gpurun_out/hd_full $K > gpurun_out/hd_full.log 2>&1
ncu -i gpurun_out/hd_full.ncu-rep --page raw --csv > gpurun_out/hd_full_raw.csv 2>/dev/null
rm -f gpurun_out/hd_full.ncu-rep
