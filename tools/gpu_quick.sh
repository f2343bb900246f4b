CUDA_LAUNCH_BLOCKING=1 BSC_GUARD=1 timeout 2400 python tools/_tmp/sweep.py > gpurun_out/sweep.log 2>&1
