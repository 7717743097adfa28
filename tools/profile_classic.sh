#!/bin/bash
# Round-1 profiling of the classic schedule (Alg. 1 as printed): launch list, full-size DRAM
# traffic of the H1/H2/H3 kernels, one --set full capture at 600x595x384.  Each ncu pass runs
# only after the same command exited 0 without ncu.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --schedule classic"
$B > gpurun_out/r1_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_stencil|k_h3|k_init' -s 30 -c 6 --csv --log-file gpurun_out/r1_traffic_full.csv $B > /dev/null 2>&1
F="python bench.py --steps 1 --warmup 1 --maxit 2 --nz 384 --no-e2e --no-cpu --schedule classic"
$F > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:'k_stencil|k_h3' -s 0 -c 3 -o gpurun_out/r1_full $F > gpurun_out/r1_full.log 2>&1
ls -la gpurun_out
