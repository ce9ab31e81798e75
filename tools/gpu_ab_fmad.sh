# render A/B: FMA contraction in render.cu (tools/libvtx_fmad.so, RENDER_FMAD=true) vs the default
# -fmad=false build, then the GPU parity suite against the contracted build
for lib in "" tools/libvtx_fmad.so; do
  echo "lib=$lib cfg2" >> gpurun_out/ab_fmad.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_fmad.log 2>&1
  echo "lib=$lib cfg3" >> gpurun_out/ab_fmad.log
  VT_LIB=$lib timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab_fmad.log 2>&1
done
VT_LIB=tools/libvtx_fmad.so timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests_fmad.log 2>&1; echo rc=$? >> gpurun_out/gputests_fmad.log
