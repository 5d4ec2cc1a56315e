set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cli.py tests/test_gpu_fullsize.py tests/test_gpu_eval.py -x -q > gpurun_out/pytest_chain.log 2>&1; echo tests=$?
timeout 600 python tools/e2e_once.py 5 > gpurun_out/e2e_once5_chain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chain|k_dchild|k_path|k_head|DeviceSelect|k_inc|k_dist" --csv --log-file gpurun_out/kernels_c5_chain.csv python tools/e2e_once.py 5 > /dev/null 2>&1; echo k5=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chain|k_dchild|k_path|k_head|DeviceSelect|k_inc|k_dist" --csv --log-file gpurun_out/kernels_c3_chain.csv python tools/e2e_once.py 3 > /dev/null 2>&1; echo k3=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chain|k_dchild|k_path|k_head|DeviceSelect|k_inc|k_dist" --csv --log-file gpurun_out/kernels_c4_chain.csv python tools/e2e_once.py 4 > /dev/null 2>&1; echo k4=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_chain|k_dchild|k_path|k_head|DeviceSelect|k_inc|k_dist" --csv --log-file gpurun_out/kernels_c2_chain.csv python tools/e2e_once.py 2 > /dev/null 2>&1; echo k2=$?
echo done
