# quick re-check: GPU suite + c2 bench line with e2e (no CPU baseline) + c3 e2e
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 5 > gpurun_out/k_c2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --config c3 --steps 5 --e2e-steps 2 > gpurun_out/k_c3.log 2>&1
