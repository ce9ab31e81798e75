set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests2.log 2>&1; echo rc=$? >> gpurun_out/gputests2.log
for v in "VT_PERSIST=0" "VT_PERSIST=1 VT_REFILL=4" "VT_PERSIST=1 VT_REFILL=8" "VT_PERSIST=1 VT_REFILL=16" "VT_PERSIST=1 VT_REFILL=24"; do
  echo "$v" >> gpurun_out/ab1.log
  env $v timeout 300 python tools/ab_render.py --frames 10 >> gpurun_out/ab1.log 2>&1
done
for v in "VT_PERSIST=0" "VT_PERSIST=1 VT_REFILL=8" "VT_PERSIST=1 VT_REFILL=16"; do
  echo "cfg3 $v" >> gpurun_out/ab1.log
  env $v timeout 300 python tools/ab_render.py --dims 2048 2048 1000 --frames 10 >> gpurun_out/ab1.log 2>&1
done
