# final evidence with the exact-zero skipping opt-in (default: every update executed)
set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err || exit 1
python -c "import __graft_entry__ as g; g.smoke()"
python tools/sanitize_smoke.py 2>&1 | tail -2
for c in 3 4 5; do
  timeout 900 python tools/e2e_config.py $c 1000 3 skip > gpurun_out/e2e_config${c}_skip.jsonl 2>&1
  timeout 900 python tools/e2e_config.py $c 1000 2 > gpurun_out/e2e_config${c}_every.jsonl 2>&1
done
python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_c4_final.json 2>&1
python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench_c5_final.json 2>&1
python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_c2_final.json 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_final.log 2>&1
python tools/launch_summary.py gpurun_out/launches_final.csv > gpurun_out/launch_summary_final.txt 2>&1
echo done
