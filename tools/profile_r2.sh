#!/bin/bash
# Round-2 profiles (one GPU call): the default bench's launch list; full-size `ncu --set full`
# captures of the classic kernels (k_stencil H1, H2; k_h3), the mixed SR sweep, the fp32 SR sweep
# and the constant-coefficient sweep; the 2D solve kernels at 22800^2.  Every ncu pass runs only
# after the same command exited 0 without ncu.  The reports are reduced to CSV on the box (raw
# metrics + the details page; the source page of the headline kernel) to fit gpurun's 64 MiB.
mkdir -p gpurun_out
N="--clock-control none"
reduce() {  # $1 = report base name
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  if [ "$2" = "src" ]; then ncu -i gpurun_out/$1.ncu-rep --page source --csv > gpurun_out/$1_source.csv 2>/dev/null; fi
  rm -f gpurun_out/$1.ncu-rep
}
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$B > gpurun_out/r2_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum $N -c 600 --csv --log-file gpurun_out/r2_launches.csv $B > /dev/null 2>&1
C="python bench.py --steps 1 --warmup 1 --maxit 2 --no-e2e --no-cpu --no-other --schedule classic"
$C > gpurun_out/r2_c.log 2>&1 && ncu --set full $N --import-source on -k regex:'k_stencil|k_h3' -s 3 -c 3 -o gpurun_out/r2_classic_full $C > gpurun_out/r2_classic_full.log 2>&1 && reduce r2_classic_full src
S="python bench.py --steps 1 --warmup 1 --maxit 2 --no-e2e --no-cpu --no-other --schedule sr"
$S > gpurun_out/r2_s.log 2>&1 && ncu --set full $N --import-source on -k regex:'^k_sr$' -s 0 -c 1 -o gpurun_out/r2_sr_full $S > gpurun_out/r2_sr_full.log 2>&1 && reduce r2_sr_full
F="python bench.py --steps 1 --warmup 1 --maxit 2 --no-e2e --no-cpu --no-other --schedule sr --precision fp32"
$F > gpurun_out/r2_f.log 2>&1 && ncu --set full $N -k regex:'^k_sr$' -s 0 -c 1 -o gpurun_out/r2_sr32_full $F > gpurun_out/r2_sr32_full.log 2>&1 && reduce r2_sr32_full
K="python bench.py --steps 1 --warmup 1 --maxit 2 --no-e2e --no-cpu --no-other --schedule sr --operator poisson-const"
$K > gpurun_out/r2_k.log 2>&1 && ncu --set full $N -k regex:'^k_sr$' -s 0 -c 1 -o gpurun_out/r2_srcc_full $K > gpurun_out/r2_srcc_full.log 2>&1 && reduce r2_srcc_full
D="python tools/run_2d_once.py"
$D > gpurun_out/r2_d.log 2>&1 && ncu --set full $N -k regex:'k_bicg9|k_apply9|k_ring9|k_round9' -c 8 -o gpurun_out/r2_2d_full $D > gpurun_out/r2_2d_full.log 2>&1 && reduce r2_2d_full
du -sh gpurun_out; ls -la gpurun_out
