set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cli.py -x -q > gpurun_out/pytest_bfs3.log 2>&1; echo tests=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "hash" > gpurun_out/pytest_bfs3_full.log 2>&1; echo full=$?
for c in 5 4 3 2; do
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bfs$|k_bfs\(" --csv --log-file gpurun_out/bfs3_c$c.csv python tools/e2e_once.py $c > /dev/null 2>&1; echo k$c=$?
done
