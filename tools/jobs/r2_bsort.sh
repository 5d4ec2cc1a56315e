set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_io.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_bsort.log 2>&1; echo tests=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bucket" --csv --log-file gpurun_out/bsort_c4.csv python tools/e2e_once.py 4 > /dev/null 2>&1; echo k4=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bucket" --csv --log-file gpurun_out/bsort_c3.csv python tools/e2e_once.py 3 > /dev/null 2>&1; echo k3=$?
timeout 600 python tools/e2e_config.py 4 1000 2 > gpurun_out/e2e_config4_bsort.jsonl 2>&1; echo e4=$?
