for v in 1 5; do
  GH_FACE_LC_BLOCKS=$v timeout 600 python tools/profile_admm.py 3 100 > gpurun_out/admm2_lc$v.log 2>&1
  GH_FACE_LC_BLOCKS=$v timeout 600 python tools/profile_admm.py 4 20 >> gpurun_out/admm2_lc$v.log 2>&1
  GH_FACE_LC_BLOCKS=$v timeout 600 python tools/profile_admm.py 2 100 >> gpurun_out/admm2_lc$v.log 2>&1
done
GH_FACE_LC_BLOCKS=3 timeout 600 python tools/profile_admm.py 2 100 >> gpurun_out/admm2_lc3.log 2>&1
echo done
