# Scratch driver for one gpurun call: GPU suite + c2 bench lines (outputs under gpurun_out/)
set -x
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 200 $B > gpurun_out/i_c2.log 2>&1
timeout 200 $B > gpurun_out/i_c2b.log 2>&1
