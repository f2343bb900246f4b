# Final evidence run for one gpurun call: full c2 bench line (e2e + cpu_baseline), smoke(), c2 launch list
set -x
timeout 400 python bench.py > gpurun_out/final3_c2.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches3_c2.csv python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu3_c2.log 2>&1
