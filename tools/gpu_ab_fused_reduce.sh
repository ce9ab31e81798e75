# Records of a reverted experiment (VT_FUSED_REDUCE, the fused plane+reduce kernel, DESIGN.md §3 Threshold > 0).
# threshold > 0: fused plane+reduce (default) vs two launches per level, then the GPU tests
for v in 0 1; do
  echo "VT_FUSED_REDUCE=$v" >> gpurun_out/ab_fr.log
  VT_FUSED_REDUCE=$v timeout 300 python tools/prof_tau.py --modes slabs,stream >> gpurun_out/ab_fr.log 2>&1
  VT_FUSED_REDUCE=$v timeout 400 python tools/prof_tau.py --dims 2048 2048 64 --fmt uint16 --modes stream >> gpurun_out/ab_fr.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests7.log 2>&1; echo rc=$? >> gpurun_out/gputests7.log
