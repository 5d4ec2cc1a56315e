set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "residual_tolerance or golden" > gpurun_out/pytest_tol_e1f.log 2>&1; echo tol=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "tolerance" > gpurun_out/pytest_tolfull_e1f.log 2>&1; echo tolfull=$?
GH_E1_PROFILE=1 timeout 600 python tools/tol_time.py 3 200 > gpurun_out/tol_time3_e1f.json 2> gpurun_out/tol_time3_e1f.err; echo tt3=$?
GH_TOL_SNAPSHOTS=1 timeout 600 python tools/tol_time.py 3 200 > gpurun_out/tol_time3_snap.json 2> gpurun_out/tol_time3_snap.err; echo tts=$?
timeout 600 python tools/tol_time.py 3 1000 > gpurun_out/tol_time3_e1f_1000.json 2>&1; echo tt1000=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_diffuse|gather_sq|k_walk|k_seg" -c 14 --csv --log-file gpurun_out/e1f_kernels.csv python tools/tol_time.py 3 200 > /dev/null 2>&1; echo ncu=$?
echo done
