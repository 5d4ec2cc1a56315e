set -x
timeout 600 python -m pytest tests/test_gpu_ipc.py -x -q > gpurun_out/pytest_ipc_r2h.log 2>&1; echo ipc=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2h.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2h.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_r2h.json 2> gpurun_out/bench_r2h.err; echo bench=$?
echo done
