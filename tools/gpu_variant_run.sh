# Scratch driver for one gpurun call: GPU suite + c3/c2 bench lines (outputs under gpurun_out/)
set -x
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 $B --config c3 --steps 5 > gpurun_out/h_c3.log 2>&1
timeout 300 $B --config c3 --steps 5 > gpurun_out/h_c3b.log 2>&1
timeout 200 $B > gpurun_out/h_c2.log 2>&1
