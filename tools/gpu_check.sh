# Re-check of the tree on a B200: GPU suite, smoke(), c2 bench line (full: e2e + cpu_baseline), reference arm (1 step)
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_reference_c2.json 2> gpurun_out/bench_reference_c2.err
