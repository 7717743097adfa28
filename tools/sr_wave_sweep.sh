#!/bin/bash
# tools/sr_wave_probe.py under several meshes / tilings: time, then DRAM bytes of one sweep (ncu)
mkdir -p gpurun_out
for spec in "$@"; do
  set -- $spec
  timeout 300 python tools/sr_wave_probe.py "$@" 2>&1 | tail -1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_sr -s 25 -c 1 --csv python tools/sr_wave_probe.py "$@" 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' '{print "   ", $(NF-2), $(NF-1), $NF}'
done
