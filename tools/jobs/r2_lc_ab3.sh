for rep in 1 2; do for v in 3 1 5; do
  GH_FACE_LC_BLOCKS=$v timeout 600 python tools/profile_admm.py 3 100 2>&1 | grep face | sed "s/^/v$v /" >> gpurun_out/admm3.log
  GH_FACE_LC_BLOCKS=$v timeout 600 python tools/profile_admm.py 4 20 2>&1 | grep face | sed "s/^/v$v /" >> gpurun_out/admm3.log
done; done
echo done
