timeout 1500 python tools/e2e_config.py 5 1000 2 > gpurun_out/e2e_config5_r2.jsonl 2>&1; echo e5=$?
