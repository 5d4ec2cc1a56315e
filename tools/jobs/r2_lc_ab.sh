set -x
for v in 3 4 1 5; do
  GH_FACE_LC_BLOCKS=$v timeout 600 python tools/profile_admm.py 3 100 > gpurun_out/admm_lc$v.log 2>&1
  GH_FACE_LC_BLOCKS=$v timeout 600 python tools/profile_admm.py 4 20 >> gpurun_out/admm_lc$v.log 2>&1
done
GH_FACE_LC_BLOCKS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or reduced or admm" > gpurun_out/pytest_lc1.log 2>&1; echo lc1=$?
GH_FACE_LC_BLOCKS=5 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_admm_stop.py -x -q > gpurun_out/pytest_lc5.log 2>&1; echo lc5=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lambda" --csv --log-file gpurun_out/lc_pair.csv env GH_FACE_LC_BLOCKS=1 python tools/e2e_once.py 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lambda" --csv --log-file gpurun_out/lc_pair4.csv env GH_FACE_LC_BLOCKS=5 python tools/e2e_once.py 3 > /dev/null 2>&1
echo done
