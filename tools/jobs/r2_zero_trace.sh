# per-launch trace of the zero-level truncation on configs 4 and 5
GH_ZERO_LEVELS_TRACE=1 python tools/profile_diffusion.py 4 1000 2 > gpurun_out/zero_trace_c4.log 2>&1
GH_ZERO_LEVELS_TRACE=1 python tools/profile_diffusion.py 5 1000 2 > gpurun_out/zero_trace_c5.log 2>&1
for f in gpurun_out/zero_trace_c4.log gpurun_out/zero_trace_c5.log; do tail -n 14 $f; done
