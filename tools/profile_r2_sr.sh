#!/bin/bash
# the SR captures of tools/profile_r2.sh alone (mixed fields, fp32, constant coefficients)
mkdir -p gpurun_out
N="--clock-control none"
reduce() {
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
for v in "sr_full:" "sr32_full:--precision fp32" "srcc_full:--operator poisson-const"; do
  tag=${v%%:*}; opt=${v#*:}
  S="python bench.py --steps 1 --warmup 1 --maxit 2 --no-e2e --no-cpu --no-other --schedule sr $opt"
  $S > gpurun_out/r2_$tag.plain.log 2>&1 && ncu --set full $N -k regex:'^k_sr$' -s 0 -c 1 -o gpurun_out/r2_$tag $S > gpurun_out/r2_$tag.log 2>&1 && reduce r2_$tag
done
ls -la gpurun_out
