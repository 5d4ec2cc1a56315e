set -x
timeout 900 python -m pytest tests/test_gpu_seqsum.py -x -q > gpurun_out/pytest_seqsum_r2i.log 2>&1; echo seqsum=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "residual_tolerance or golden" > gpurun_out/pytest_tol_r2i.log 2>&1; echo tol=$?
GH_E1_PROFILE=1 timeout 600 python tools/tol_time.py 3 200 > gpurun_out/tol_time3_r2i.json 2> gpurun_out/tol_time3_r2i.err; echo tt3=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "tolerance" > gpurun_out/pytest_tolfull_r2i.log 2>&1; echo tolfull=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"residual_rows|gather_sq|k_walk|k_seg" -c 12 --csv --log-file gpurun_out/e1_kernels_r2i.csv python tools/tol_time.py 3 200 > gpurun_out/e1_ncu_r2i.log 2>&1; echo ncu=$?
echo done
