# launch list (per-kernel device time) of the cfg1 threshold > 0 VSTR stream: what the per-insertion chain spends
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/tau_launches.csv \
  python tools/prof_tau.py --modes stream > gpurun_out/tau_ncu.log 2>&1
