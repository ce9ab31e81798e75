# one ncu --set full capture of the cfg3 stream's fill_borders k_borders launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_borders -c 1 \
  -o gpurun_out/r2s_borders python tools/prof_stream3.py 2048 2048 1000 --reps 1 > gpurun_out/ncu_borders.log 2>&1
