set -x
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:"residual_rows|scatter_sq|walk" -c 3 --csv --log-file gpurun_out/e1_kernels_r2e.csv python tools/tol_time.py 3 200 > gpurun_out/e1_ncu_r2e.log 2>&1; echo ncu=$?
