set -x
for c in "3 1000" "2 1000" "4 200" "5 100"; do
  set -- $c
  timeout 600 python tools/profile_diffusion.py $1 $2 3 > gpurun_out/b2_c$1.log 2>&1
  GH_DIFFUSE_BLOCKS=3 timeout 600 python tools/profile_diffusion.py $1 $2 3 > gpurun_out/b3_c$1.log 2>&1
done
GH_DIFFUSE_BLOCKS=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or reduced or column_formats or more_levels" > gpurun_out/pytest_b3.log 2>&1; echo b3tests=$?
echo done
