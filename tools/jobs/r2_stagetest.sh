timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pageable" > gpurun_out/pytest_stagetest.log 2>&1; echo st=$?
