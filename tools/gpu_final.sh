# end-of-session check: GPU tests, smoke, the default bench, the reference arm,
# and the launch list of a short bench run (ncu single-metric pass)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputests.log 2>&1; echo rc=$? >> gpurun_out/final_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench.log 2>&1; echo rc=$? >> gpurun_out/final_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1; echo rc=$? >> gpurun_out/final_bench_ref.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-tau --no-secondary --no-build-e2e > gpurun_out/final_ncu.log 2>&1
