# Records of a reverted experiment (VT_RENDER_CARVEOUT); the committed library
# ignores the variable, the ncu capture still applies.
# render A/B of the shared-memory carveout + one ncu source-level capture
for v in -1 0 10 25 50 100; do
  echo "VT_RENDER_CARVEOUT=$v" >> gpurun_out/ab_co.log
  VT_RENDER_CARVEOUT=$v timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_co.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_render_fullframe -s 3 -c 1 \
  -o gpurun_out/r2s_render python tools/ab_render.py --frames 1 > gpurun_out/ncu_render.log 2>&1
