set -x
timeout 600 python -m pytest tests/test_gpu_ipc.py -x -q > gpurun_out/pytest_ipc_r2.log 2>&1; echo ipc=$?
timeout 300 python tools/e2e_once.py 3 > gpurun_out/e2e_once3_r2b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_face|k_chain|k_bfs|k_inc" --csv --log-file gpurun_out/kernels_c3_r2b.csv python tools/e2e_once.py 3 > gpurun_out/ncu_k3_r2b.log 2>&1; echo k3=$?
timeout 600 python tools/e2e_once.py 5 > gpurun_out/e2e_once5_r2b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chain|k_bfs|k_edge|k_inc" --csv --log-file gpurun_out/kernels_c5_r2b.csv python tools/e2e_once.py 5 > gpurun_out/ncu_k5_r2b.log 2>&1; echo k5=$?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2b.log 2>&1; echo pytest=$?
echo done
