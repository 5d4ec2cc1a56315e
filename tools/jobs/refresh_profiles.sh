set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1m.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/bench_r1m.json 2> gpurun_out/bench_r1m.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1m.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_r1m.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_diffuse -c 1 -f -o gpurun_out/diffuse_r1m python tools/profile_diffusion.py 3 1000 > gpurun_out/ncu_r1m.log 2>&1
timeout 900 python tools/e2e_parity.py --configs 2,3,4 --out gpurun_out/e2e_parity_r1m.json > gpurun_out/e2e_parity_r1m.log 2>&1
timeout 600 python tools/admm_stop_parity.py --configs 2,3 --iters 10,60 --out gpurun_out/admm_stop_parity_r1m.json > gpurun_out/admm_stop_parity_r1m.log 2>&1
timeout 600 python tools/e2e_config.py 4 > gpurun_out/e2e_config4_r1m.jsonl 2>&1
timeout 900 python tools/e2e_config.py 5 > gpurun_out/e2e_config5_r1m.jsonl 2>&1
echo done
