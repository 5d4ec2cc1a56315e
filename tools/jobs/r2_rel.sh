timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "release or cached" > gpurun_out/pytest_rel.log 2>&1; echo rel=$?
