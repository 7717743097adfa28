#!/bin/bash
# DRAM bytes of one full-size SR sweep under layout / chunk variants (ncu, 1 launch each)
mkdir -p gpurun_out
run() {
  tag=$1; shift
  env "$@" python bench.py --steps 1 --warmup 1 --maxit 3 --no-e2e --no-cpu > /dev/null 2>&1 || { echo "$tag bench failed"; return; }
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_sr -s 6 -c 1 --csv python bench.py --steps 1 --warmup 1 --maxit 3 --no-e2e --no-cpu 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' -v t="$tag" '{print t, $(NF-2), $(NF-1), $NF}'
}
for v in "$@"; do run $v; done
