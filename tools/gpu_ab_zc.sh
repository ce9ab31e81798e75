# A/B of zero-copy staging (VT_ZC_STAGE) on the threshold > 0 streams and the
# cfg2 whole-volume build; then the GPU test suite with the default
for v in 0 1; do
  echo "VT_ZC_STAGE=$v" >> gpurun_out/ab_zc.log
  VT_ZC_STAGE=$v timeout 300 python tools/prof_tau.py --modes slabs,stream >> gpurun_out/ab_zc.log 2>&1
  VT_ZC_STAGE=$v timeout 400 python tools/prof_tau.py --dims 2048 2048 64 --fmt uint16 --modes stream >> gpurun_out/ab_zc.log 2>&1
  VT_ZC_STAGE=$v timeout 300 python tools/ab_build.py 1024 3 >> gpurun_out/ab_zc.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests3.log 2>&1; echo rc=$? >> gpurun_out/gputests3.log
