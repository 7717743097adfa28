#!/bin/bash
# tools/ncu_sweep.sh "<tilings>" [nz] [tag]: ncu DRAM/L2 counters of the stencil kernels per
# tiling, one CSV per tiling in gpurun_out/ (parse with tools/ncu_table.py)
NZ=${2:-384}
TAG=${3:-sw}
mkdir -p gpurun_out
for t in $1; do
  CMD="python bench.py --steps 1 --warmup 1 --maxit 2 --nz $NZ --no-e2e --no-cpu --tiling $t"
  $CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:'k_stencil|k_rows' -s 0 -c 2 --csv $CMD > gpurun_out/ncu_${TAG}_${t//,/_}.csv 2>/dev/null
done
