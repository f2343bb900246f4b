# A/B of the M-step factor overlap (BSC_MSTEP_OVERLAP) + the GPU suite
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
for v in 1 0 1 0; do
  BSC_MSTEP_OVERLAP=$v timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 >> gpurun_out/ov_c2_$v.log 2>&1
done
BSC_MSTEP_OVERLAP=1 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 5 > gpurun_out/ov_c2_e2e.log 2>&1
for v in 1 0; do
  BSC_MSTEP_OVERLAP=$v timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 --config c3 --steps 5 > gpurun_out/ov_c3_$v.log 2>&1
  BSC_MSTEP_OVERLAP=$v timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --config c1 > gpurun_out/ov_c1_$v.log 2>&1
done
