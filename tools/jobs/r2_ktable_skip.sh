# per-kernel tables of one end-to-end call with the exact-zero skipping (configs 3, 4, 5)
for c in 3 4 5; do
  python tools/e2e_once.py $c > gpurun_out/e2e_once_c$c.log 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/ktable_c$c.csv python tools/e2e_once.py $c > gpurun_out/ktable_c$c.log 2>&1
  python tools/kernel_table.py gpurun_out/ktable_c$c.csv --out gpurun_out/r2_kernel_table_c${c}_skip.json \
      --workload "C$c one gh_distance_host call, exact-zero skipping on" > gpurun_out/r2_kernel_table_c${c}_skip.txt 2>&1
  head -32 gpurun_out/r2_kernel_table_c${c}_skip.txt
done
