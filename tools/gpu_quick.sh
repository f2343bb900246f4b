set -x
CUDA_LAUNCH_BLOCKING=1 BSC_GUARD=3 timeout 2400 python tools/shape_sweep.py > gpurun_out/sweep3.log 2>&1
BSC_GUARD=3 timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_guard3.log 2>&1; echo rc=$? >> gpurun_out/t_guard3.log
