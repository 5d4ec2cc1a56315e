timeout 600 python tools/e2e_once.py 4 > gpurun_out/e2e_once4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/kernels_c4_r2.csv python tools/e2e_once.py 4 > /dev/null 2>&1; echo k4=$?
timeout 600 python tools/e2e_config.py 4 1000 2 > gpurun_out/e2e_config4_r2.jsonl 2>&1; echo e4=$?
