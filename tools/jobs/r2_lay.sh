set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_lay.log 2>&1; echo tests=$?
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "4-face or 4 and face" > gpurun_out/pytest_lay_full.log 2>&1; echo full=$?
timeout 600 python tools/e2e_config.py 4 1000 2 > gpurun_out/e2e_config4_lay.jsonl 2>&1; echo e4=$?
timeout 600 python tools/profile_diffusion.py 4 200 2 > gpurun_out/lay_c4.log 2>&1; echo d4=$?
timeout 600 python tools/profile_diffusion.py 3 1000 2 > gpurun_out/lay_c3.log 2>&1; echo d3=$?
