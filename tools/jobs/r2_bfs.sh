set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity_r2d.log 2>&1; echo parity=$?
timeout 600 python tools/e2e_once.py 5 > gpurun_out/e2e_once5_r2d.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chain|k_bfs" --csv --log-file gpurun_out/kernels_c5_r2d.csv python tools/e2e_once.py 5 > gpurun_out/ncu_k5_r2d.log 2>&1; echo k5=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chain|k_bfs" --csv --log-file gpurun_out/kernels_c3_r2d.csv python tools/e2e_once.py 3 > gpurun_out/ncu_k3_r2d.log 2>&1; echo k3=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; echo bench=$?
echo done
