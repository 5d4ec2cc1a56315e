# round-1 profile refresh, part A: ncu captures (run each only after its command exits 0 without ncu)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1p.log 2>&1; echo pytest=$?
timeout 300 python tools/profile_diffusion.py 3 1000 2 > gpurun_out/diffuse_plain_r1p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_diffuse -c 1 -f -o gpurun_out/diffuse_r1p python tools/profile_diffusion.py 3 1000 > gpurun_out/ncu_r1p.log 2>&1
timeout 300 python tools/e2e_once.py 3 > gpurun_out/e2e_once3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/kernels_c3_r1p.csv python tools/e2e_once.py 3 > gpurun_out/ncu_k3.log 2>&1
timeout 600 python tools/e2e_once.py 5 > gpurun_out/e2e_once5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/kernels_c5_r1p.csv python tools/e2e_once.py 5 > gpurun_out/ncu_k5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_face_g|k_face_lambda_c|k_edge_x|k_edge_lambda_w|k_normalize|k_bfs|k_chain" -c 7 -f -o gpurun_out/others_r1p python tools/e2e_once.py 3 > gpurun_out/ncu_others.log 2>&1
echo done
