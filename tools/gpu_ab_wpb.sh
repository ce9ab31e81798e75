# Records of a reverted experiment: needs the VT_WPB builds (tools/libvtx_wpb*.so) made from the
# render.cu variant described in DESIGN.md §5; kept for the numbers it produced.
# render A/B: warps per CTA of the full-frame kernel (VT_WPB builds in tools/)
for lib in "" tools/libvtx_wpb5.so tools/libvtx_wpb10.so tools/libvtx_wpb20.so; do
  echo "lib=$lib cfg2" >> gpurun_out/ab_wpb.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_wpb.log 2>&1
done
for lib in "" tools/libvtx_wpb5.so tools/libvtx_wpb10.so tools/libvtx_wpb20.so; do
  echo "lib=$lib cfg3" >> gpurun_out/ab_wpb.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab_wpb.log 2>&1
done
