for rep in 1 2; do
for v in "64,512" "32,128" "16,64" "64,256" "128,1024"; do
  for c in "3 1000" "2 1000" "4 200"; do
    set -- $c
    GH_WAIT_NS=$v timeout 300 python tools/profile_diffusion.py $1 $2 2 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/wait_ab.log
  done
done; done
