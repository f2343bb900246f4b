set -x
timeout 1200 python -m pytest tests/test_gpu_guards.py -m gpu -q > gpurun_out/t_guards.log 2>&1; echo rc=$? >> gpurun_out/t_guards.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
