# quick re-check: GPU suite + c2 / c3 bench kernel parts
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 300 $B > gpurun_out/k_c2.log 2>&1
timeout 600 $B --config c3 --steps 5 > gpurun_out/k_c3.log 2>&1
