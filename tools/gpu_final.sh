# r02 final evidence on the final code: full-size parity c2 (20 iterations), bench lines c0-c4 and the reference
# arm, ncu captures (tools/gpu_r02_prof.sh), the GPU suite under guarded allocations, smoke()
set -x
timeout 900 python tools/trajectory_check.py c2 20 --out gpurun_out/r02_parity_full_c2.txt > gpurun_out/traj_c2.log 2>&1; echo rc=$? >> gpurun_out/traj_c2.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1200 python bench.py --config c3 --steps 10 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 1800 python bench.py --config c4 --steps 5 --e2e-steps 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config c0 > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_reference_c2.json 2> gpurun_out/bench_reference_c2.err
bash tools/gpu_r02_prof.sh
BSC_GUARD=1 timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_guard_suite.log 2>&1; echo rc=$? >> gpurun_out/t_guard_suite.log
BSC_GUARD=2 timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_guard2.log 2>&1; echo rc=$? >> gpurun_out/t_guard2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
