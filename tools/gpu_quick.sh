# quick re-check: GPU suite + c2 bench line with e2e (no CPU baseline)
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 6 > gpurun_out/k_c2.log 2>&1
BSC_HOST_CHUNK=12544 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 6 --steps 5 > gpurun_out/k_c2_16chunks.log 2>&1
nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max --format=csv > gpurun_out/pcie.txt 2>&1
