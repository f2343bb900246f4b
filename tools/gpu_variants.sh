# GPU suite + bench kernel parts at c2 / c3
set -x
timeout 1500 python -m pytest tests -m gpu -q --maxfail=6 > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 300 $B > gpurun_out/p_c2_rows.log 2>&1
BSC_POTRF_ROWS=0 timeout 300 $B > gpurun_out/p_c2_block.log 2>&1
timeout 600 $B --config c3 --steps 5 > gpurun_out/p_c3_rows.log 2>&1
BSC_POTRF_ROWS=0 timeout 600 $B --config c3 --steps 5 > gpurun_out/p_c3_block.log 2>&1
