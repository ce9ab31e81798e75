# cfg3 stream: phase timing, then the per-launch list of the tail kernels
timeout 300 python tools/prof_stream3.py 2048 2048 1000 --reps 2 > gpurun_out/tail_phases.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_borders|k_plane_copy|k_dense_level|k_finish|k_reduce|k_octant|k_plane" --csv --log-file gpurun_out/tail_launches.csv \
  python tools/prof_stream3.py 2048 2048 1000 --reps 1 > gpurun_out/tail_ncu.log 2>&1
