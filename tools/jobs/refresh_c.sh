# round-1 profile refresh, part C: bench line, launch list, large configs (after the allocator change)
set -x
python bench.py > gpurun_out/bench_r1q.json 2> gpurun_out/bench_r1q.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1q.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_r1q.log 2>&1
timeout 600 python tools/e2e_config.py 4 1000 3 > gpurun_out/e2e_config4_r1q.jsonl 2>&1
timeout 900 python tools/e2e_config.py 5 1000 3 > gpurun_out/e2e_config5_r1q.jsonl 2>&1
echo done
