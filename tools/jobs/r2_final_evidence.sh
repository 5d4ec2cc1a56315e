# round-2 final evidence: GPU suite, bench line, launch list of the bench command, end to end on
# configs 3-5, per-kernel tables (each ncu pass only after its command exited 0 without ncu)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err || exit 1
tail -1 gpurun_out/bench_final.json
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_final.log 2>&1
python tools/launch_summary.py gpurun_out/launches_final.csv > gpurun_out/launch_summary_final.txt 2>&1
for c in 3 4 5; do
  timeout 900 python tools/e2e_config.py $c 1000 3 > gpurun_out/e2e_config${c}_final.jsonl 2>&1
  tail -2 gpurun_out/e2e_config${c}_final.jsonl | head -1
  timeout 600 python tools/e2e_once.py $c > gpurun_out/e2e_once_c$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/ktable_c$c.csv python tools/e2e_once.py $c > gpurun_out/ktable_c$c.log 2>&1
  python tools/kernel_table.py gpurun_out/ktable_c$c.csv --out gpurun_out/r2_kernel_table_c${c}_skip.json \
      --workload "C$c one gh_distance_host call, exact-zero skipping on" > gpurun_out/r2_kernel_table_c${c}_skip.txt 2>&1
done
python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_c4_final.json 2>&1
python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench_c5_final.json 2>&1
tail -c 1500 gpurun_out/bench_c5_final.json
echo done
