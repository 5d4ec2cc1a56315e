timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "residual_tolerance" > gpurun_out/pytest_tol32.log 2>&1; echo tol=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "tolerance" > gpurun_out/pytest_tol32_full.log 2>&1; echo full=$?
timeout 600 python tools/tol_time.py 3 200 > gpurun_out/tol32_200.json 2>&1; echo t200=$?
timeout 900 python tools/tol_time.py 3 1000 > gpurun_out/tol32_1000.json 2>&1; echo t1000=$?
