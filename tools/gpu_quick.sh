set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/k_c2.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --config c1 > gpurun_out/k_c1.log 2>&1
