# ncu --set full of the other hot kernels of the final build (config 3, one end-to-end call; each capture
# after the plain command exited 0): face ADMM kernels, BFS, chain; and the truncation's diffusion launches
set -x
python tools/e2e_once.py 3 > gpurun_out/e2e_once_c3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_face_g|k_face_lambda_pair|k_bfs|k_chain|k_normalize" -c 8 -f -o gpurun_out/others_final python tools/e2e_once.py 3 > gpurun_out/ncu_others_final.log 2>&1
GH_ZERO_LEVELS=1 python tools/e2e_once.py 4 > gpurun_out/e2e_once_c4_skip.log 2>&1 || exit 1
GH_ZERO_LEVELS=1 ncu --set full --clock-control none --import-source on -k regex:k_diffuse -c 7 -f -o gpurun_out/diffuse_c4_skip python tools/e2e_once.py 4 > gpurun_out/ncu_c4_skip.log 2>&1
ls -la gpurun_out/*.ncu-rep
