# Record of a rejected A/B (integer bit-pattern compares in the sampler); the variant .so was a temporary build.
# render A/B: committed split (cell floors on XU) vs tools/libvtx_vE.so (sample bounds compared as integers); GPU tests
for rep in 1 2; do
  for lib in "" tools/libvtx_vE.so; do
    echo "lib=$lib cfg3" >> gpurun_out/ab_cmp.log
    VT_LIB=$lib timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab_cmp.log 2>&1
  done
done
for lib in "" tools/libvtx_vE.so; do
  echo "lib=$lib cfg2" >> gpurun_out/ab_cmp.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_cmp.log 2>&1
done
VT_LIB=tools/libvtx_vE.so timeout 900 python -m pytest tests -m gpu -q > gpurun_out/cmp_gputests.log 2>&1; echo rc=$? >> gpurun_out/cmp_gputests.log
