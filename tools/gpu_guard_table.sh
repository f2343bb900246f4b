set -x
timeout 900 python -m pytest tests/test_gpu_guards.py -m gpu -q > gpurun_out/t_guards.log 2>&1; echo rc=$? >> gpurun_out/t_guards.log
bash tools/gpu_r02_table.sh
