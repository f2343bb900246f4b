# r02: GPU suite on the fused finish+slice path, A/B bench, ncu --set full of one c2 step's kernels, launch list
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c2_fused.log 2>&1
BSC_FUSED_FINISH=0 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c2_unfused.log 2>&1
timeout 600 python bench.py --config c3 --steps 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_fused.log 2>&1
BSC_FUSED_FINISH=0 timeout 600 python bench.py --config c3 --steps 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_unfused.log 2>&1
MR0=paper_1908_06843_b200/_lib_mr0/libprsp_bsc_b200.so
PRSP_BSC_LIB=$MR0 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c2_mr0.log 2>&1
PRSP_BSC_LIB=$MR0 timeout 600 python bench.py --config c3 --steps 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_mr0.log 2>&1
K='regex:select_kernel|lane_states|lane_finish|oz_gemm_kernel|enumerate_kernel'
timeout 300 python tools/profile_case.py c2 200000 2 > gpurun_out/plain_c2.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -s 6 -c 6 -f -o gpurun_out/r02_c2 python tools/profile_case.py c2 200000 2 > gpurun_out/ncu_c2.log 2>&1
timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/plain_bench.log 2>&1 &&
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launches.log 2>&1
