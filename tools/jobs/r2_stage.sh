set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_io.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_stage_r2.log 2>&1; echo tests=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err; echo bench=$?
echo done
