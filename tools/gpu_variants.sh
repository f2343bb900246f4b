# A/B of kernel variants (PRSP_BSC_LIB builds / env switches) at c2 / c3: GPU suite, bench kernel parts
set -x
timeout 1500 python -m pytest tests -m gpu -q --maxfail=6 > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 300 $B > gpurun_out/w_c2_main.log 2>&1
timeout 300 $B --config c1 > gpurun_out/w_c1_main.log 2>&1
timeout 600 $B --config c3 --steps 5 > gpurun_out/w_c3_main.log 2>&1
