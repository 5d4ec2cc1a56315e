# final evidence after the lean diffusion instances: GPU suite, bench, ncu capture + launch list, e2e configs 3-5
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err || exit 1
python tools/profile_diffusion.py 3 1000 2 > gpurun_out/diffuse_plain_c3_final.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_diffuse -c 1 -f -o gpurun_out/diffuse_c3_final python tools/profile_diffusion.py 3 1000 > gpurun_out/ncu_c3_final.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_final.log 2>&1
python tools/launch_summary.py gpurun_out/launches_final.csv > gpurun_out/launch_summary_final.txt 2>&1
for c in 3 4 5; do timeout 900 python tools/e2e_config.py $c 1000 3 > gpurun_out/e2e_config${c}_final.jsonl 2>&1; done
python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_c4_final.json 2>&1
python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench_c5_final.json 2>&1
python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_c2_final.json 2>&1
echo done
