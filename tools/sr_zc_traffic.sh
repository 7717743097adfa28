# SR sweep DRAM bytes vs uniform z-chunk length (the drift hypothesis: short chunks keep neighbouring
# tiles marching together, as for the classic kernels); two sweeps under ncu per chunk length
mkdir -p gpurun_out
for z in 16 32 64 160 1536; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_sr$' -s 2 -c 2 --csv python bench.py --steps 1 --warmup 1 --maxit 4 --no-cpu --no-e2e --no-other --no-2d --no-tts --schedule sr --sr-tiling 16,2,2,$z,16 > gpurun_out/sr_zc_ncu_$z.csv 2>/dev/null
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'^k_sr$' -s 2 -c 2 --csv python bench.py --steps 1 --warmup 1 --maxit 4 --no-cpu --no-e2e --no-other --no-2d --no-tts --schedule sr > gpurun_out/sr_zc_ncu_default.csv 2>/dev/null
