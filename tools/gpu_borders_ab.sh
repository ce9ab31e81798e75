# Records of a reverted experiment (the k_borders shell table).
# fill_borders after the k_borders table/lookup change: GPU tests, stream phases, ncu of k_borders, bench
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests6.log 2>&1; echo rc=$? >> gpurun_out/gputests6.log
timeout 300 python tools/prof_stream3.py 2048 2048 1000 --reps 3 > gpurun_out/tail_phases3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none \
  -k regex:"k_borders" --csv --log-file gpurun_out/borders_launch.csv python tools/prof_stream3.py 2048 2048 1000 --reps 1 > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/bench3.log 2>&1
