set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cli.py -x -q > gpurun_out/pytest_pe.log 2>&1; echo tests=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "hash" > gpurun_out/pytest_pe_full.log 2>&1; echo full=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_inc|k_parent" --csv --log-file gpurun_out/pe_c5.csv python tools/e2e_once.py 5 > /dev/null 2>&1; echo k5=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_inc|k_parent" --csv --log-file gpurun_out/pe_c3.csv python tools/e2e_once.py 3 > /dev/null 2>&1; echo k3=$?
