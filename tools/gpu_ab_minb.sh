# Render A/B of CTAs per SM (VT_RENDER_MINB builds in tools/, made with EXTRA="-DVT_RENDER_MINB=N");
# end of round 2: 5 (default) 4.69 ms cfg3 / 4.42 cfg2, 6: 4.88 / 4.38, 4: 5.08 / 4.47.
for lib in "" tools/libvtx_minb6.so tools/libvtx_minb4.so; do
  echo "lib=$lib cfg2" >> gpurun_out/ab_minb.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_minb.log 2>&1
  echo "lib=$lib cfg3" >> gpurun_out/ab_minb.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab_minb.log 2>&1
done
