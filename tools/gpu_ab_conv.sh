# Record of the A/B that chose the conversion split now in render.cu (the variant .so files were temporary builds).
# render A/B of where the per-sample conversions run (tools/libvtx_vA.so: trilerp cell floors on the
# XU pipe; tools/libvtx_vB.so: node-box origins on the XU pipe; "": the committed split)
for rep in 1 2; do
  for lib in "" tools/libvtx_vA.so tools/libvtx_vB.so; do
    echo "lib=$lib cfg3" >> gpurun_out/ab_conv.log
    VT_LIB=$lib timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab_conv.log 2>&1
  done
done
for lib in "" tools/libvtx_vA.so tools/libvtx_vB.so; do
  echo "lib=$lib cfg2" >> gpurun_out/ab_conv.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_conv.log 2>&1
done
