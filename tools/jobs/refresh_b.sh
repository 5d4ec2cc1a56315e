# round-1 profile refresh, part B: bench line, launch list, parity at full scale, large configs
set -x
python bench.py > gpurun_out/bench_r1p.json 2> gpurun_out/bench_r1p.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1p.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_r1p.log 2>&1
timeout 900 python tools/e2e_parity.py --configs 2,3,4 --out gpurun_out/e2e_parity_r1p.json > gpurun_out/e2e_parity_r1p.log 2>&1
timeout 600 python tools/admm_stop_parity.py --configs 2,3 --iters 10,60 --out gpurun_out/admm_stop_parity_r1p.json > gpurun_out/admm_stop_parity_r1p.log 2>&1
timeout 600 python tools/e2e_config.py 4 1000 3 > gpurun_out/e2e_config4_r1p.jsonl 2>&1
timeout 900 python tools/e2e_config.py 5 1000 3 > gpurun_out/e2e_config5_r1p.jsonl 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1p.json 2> gpurun_out/bench_ref_r1p.err
echo done
