# r02 re-entry check: GPU suite, smoke, full c2 bench line, reference arm, c2 launch list
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 500 python bench.py > gpurun_out/bench_c2.log 2>&1
timeout 200 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c2b.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_c2.log 2>&1
nproc > gpurun_out/nproc.txt
