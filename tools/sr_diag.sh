# SR traffic diagnostics: DRAM bytes and time of one full-size k_sr launch per build variant
for t in base d1 d2 d4 d7; do
  C="python tools/run_variant.py $t --steps 1 --warmup 1 --maxit 2 --no-e2e --no-cpu --no-other --no-2d --schedule sr"
  $C > /dev/null 2>&1
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:'^k_sr$' -s 0 -c 1 --csv $C 2>/dev/null | grep -E "dram|duration" | awk -F'","' -v t=$t '{print t, $(NF-2), $NF}' >> gpurun_out/srdiag.log
done
