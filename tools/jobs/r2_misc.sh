set -x
timeout 900 python tools/partition_model.py --configs 2,3,4,5 --out gpurun_out/r2_partition_model.json > gpurun_out/partition_model.log 2>&1; echo pm=$?
echo done
