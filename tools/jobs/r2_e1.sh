# round 2: batched E1 engine
set -x
timeout 900 python -m pytest tests/test_gpu_seqsum.py -x -q > gpurun_out/pytest_seqsum_r2b.log 2>&1; echo seqsum=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "residual_tolerance or tol" > gpurun_out/pytest_tol_r2b.log 2>&1; echo tol=$?
GH_E1_PROFILE=1 timeout 600 python tools/tol_time.py 3 200 > gpurun_out/tol_time3_r2b.json 2> gpurun_out/tol_time3_r2b.err; echo tt3=$?
GH_E1_PROFILE=1 timeout 600 python tools/tol_time.py 2 200 > gpurun_out/tol_time2_r2b.json 2> gpurun_out/tol_time2_r2b.err; echo tt2=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "tolerance" > gpurun_out/pytest_tolfull_r2b.log 2>&1; echo tolfull=$?
echo done
