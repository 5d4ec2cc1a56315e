# round 2 evidence: ncu captures of the diffusion kernel on configs 2, 4, 5 (L2 hit rates),
# per-kernel DRAM table of one C3 end-to-end call, bench launch list
set -x
for c in "2 1000" "4 200" "5 100"; do
  set -- $c
  timeout 600 python tools/profile_diffusion.py $1 $2 > gpurun_out/diffuse_plain_c$1_r2.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_diffuse -c 1 -f -o gpurun_out/diffuse_c$1_r2 python tools/profile_diffusion.py $1 $2 > gpurun_out/ncu_c$1_r2.log 2>&1; echo c$1=$?
done
timeout 300 python tools/e2e_once.py 3 > gpurun_out/e2e_once3_r2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/kernels_c3_r2.csv python tools/e2e_once.py 3 > gpurun_out/ncu_k3_r2.log 2>&1; echo k3=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_r2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_r2.log 2>&1; echo launches=$?
echo done
