set -x
timeout 300 python tools/profile_diffusion.py 3 1000 2 > gpurun_out/diffuse_plain_c3_r2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_diffuse -c 1 -f -o gpurun_out/diffuse_c3_r2 python tools/profile_diffusion.py 3 1000 > gpurun_out/ncu_c3_r2.log 2>&1; echo c3=$?
ncu --set full --import-source on --clock-control none -k regex:"k_face_lambda_pair|k_face_g" --launch-skip 2 --launch-count 2 -f -o gpurun_out/face_admm_r2b python tools/e2e_once.py 3 > gpurun_out/face_admm_ncu_b.log 2>&1; echo fa=$?
