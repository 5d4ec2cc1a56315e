set -x
ncu --set full --import-source on --clock-control none -k regex:"k_face_lambda_c|k_face_g" --launch-skip 2 --launch-count 2 -f -o gpurun_out/face_admm_r2 python tools/e2e_once.py 3 > gpurun_out/face_admm_ncu.log 2>&1; echo ncu=$?
