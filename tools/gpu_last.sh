# last refresh on the final tree: bench lines c0, c1, c3, c4 and one full-size c3 parity iteration
set -x
timeout 300 python bench.py --config c0 > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 1200 python bench.py --config c3 --steps 10 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 1800 python bench.py --config c4 --steps 5 --e2e-steps 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 1200 python tools/trajectory_check.py c3 1 --out gpurun_out/r02_parity_full_c3_final.txt > gpurun_out/traj_c3f.log 2>&1; echo rc=$? >> gpurun_out/traj_c3f.log
