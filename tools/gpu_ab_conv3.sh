# Record of the A/B of the descent floors on the XU pipe (adopted); the variant .so was a temporary build.
# Record of the A/B that chose the conversion split now in render.cu (the variant .so files were temporary builds).
# render A/B: committed split (cell floors on XU) vs tools/libvtx_vD.so (descent floors on XU); GPU tests
for rep in 1 2; do
  for lib in "" tools/libvtx_vD.so; do
    echo "lib=$lib cfg3" >> gpurun_out/ab_conv3.log
    VT_LIB=$lib timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab_conv3.log 2>&1
  done
done
for lib in "" tools/libvtx_vD.so; do
  echo "lib=$lib cfg2" >> gpurun_out/ab_conv3.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_conv3.log 2>&1
done
