# Record of the A/B that chose the split conversions now in render.cu (tools/libvtx_mix.so was that build).
# render A/B: corner conversions split between the XU pipe (a0) and the FP64 pipe (a1 - a0), tools/libvtx_mix.so
for lib in "" tools/libvtx_mix.so "" tools/libvtx_mix.so; do
  echo "lib=$lib cfg3" >> gpurun_out/ab_mix.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab_mix.log 2>&1
done
for lib in "" tools/libvtx_mix.so; do
  echo "lib=$lib cfg2" >> gpurun_out/ab_mix.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_mix.log 2>&1
done
