#!/bin/bash
# Round-1 profiling of the default bench (SR schedule): launch list, full-size
# DRAM traffic of the sweep, one --set full capture at 600x595x384.
# Each ncu pass runs only after the same command exited 0 without ncu.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$B > gpurun_out/r1_sr_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_sr_launches.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_sr|k_init' -s 20 -c 4 --csv --log-file gpurun_out/r1_sr_traffic_full.csv $B > /dev/null 2>&1
F="python bench.py --steps 1 --warmup 1 --maxit 4 --nz 384 --no-e2e --no-cpu"
$F > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sr -s 2 -c 1 -o gpurun_out/r1_sr_full $F > gpurun_out/r1_sr_full.log 2>&1
ls -la gpurun_out
