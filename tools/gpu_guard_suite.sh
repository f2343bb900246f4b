# The whole GPU suite under guarded device allocations (BSC_GUARD=1): every test ends with a guard check
BSC_GUARD=1 timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/t_guard_suite.log 2>&1; echo rc=$? >> gpurun_out/t_guard_suite.log
