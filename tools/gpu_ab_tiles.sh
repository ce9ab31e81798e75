# Records of a reverted experiment (VT_TILE_SCHED, the persistent tile-scheduled render kernel,
# DESIGN.md §5); the committed library ignores the variable.
# render A/B: static grid vs dynamic tile scheduling (VT_TILE_SCHED = super-tile height)
for v in 0 4 8 16 32; do
  echo "VT_TILE_SCHED=$v cfg2" >> gpurun_out/ab_tiles.log
  VT_TILE_SCHED=$v timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab_tiles.log 2>&1
done
for v in 0 8 16; do
  echo "VT_TILE_SCHED=$v cfg3" >> gpurun_out/ab_tiles.log
  VT_TILE_SCHED=$v timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab_tiles.log 2>&1
done
