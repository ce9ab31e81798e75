# render A/B against the committed library build in tools/libvtx_base.so (if present), then the render GPU tests
for lib in tools/libvtx_base.so ""; do
  [ -n "$lib" ] && [ ! -f "$lib" ] && continue
  echo "lib=$lib cfg2" >> gpurun_out/ab_render.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_render.log 2>&1
  echo "lib=$lib cfg3" >> gpurun_out/ab_render.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab_render.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests5.log 2>&1; echo rc=$? >> gpurun_out/gputests5.log
