# ncu capture of the diffusion kernel at config 3, one 1000-sweep launch (steady state)
python tools/profile_diffusion.py 3 1000 2 > gpurun_out/diffuse_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_diffuse -c 1 -o gpurun_out/diffuse_c16 -f python tools/profile_diffusion.py 3 1000 > gpurun_out/ncu_c16.log 2>&1
echo rc=$?
