set -x
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"group|k_diffuse" --csv --log-file gpurun_out/e1_kernels_r2b.csv python tools/tol_time.py 3 200 > gpurun_out/e1_ncu_r2b.log 2>&1; echo ncu=$?
echo done
