# per-kernel table of one end-to-end call at configs 5 and 4 with zero-level truncation
python -m pytest tests/test_gpu_parity.py -x -q -k "zero_level" 2>&1 | tail -3
for c in 5 4; do
  python tools/e2e_once.py $c > gpurun_out/e2e_once_c$c.log 2>&1 || exit 1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/ktable_c$c.csv python tools/e2e_once.py $c > gpurun_out/ktable_c$c.log 2>&1
  python tools/kernel_table.py gpurun_out/ktable_c$c.csv --out gpurun_out/r2_kernel_table_c${c}_trunc.json \
      --workload "C$c one gh_distance_host call, zero-level truncation" > gpurun_out/r2_kernel_table_c${c}_trunc.txt 2>&1
  head -40 gpurun_out/r2_kernel_table_c${c}_trunc.txt
done
