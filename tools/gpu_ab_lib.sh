# A/B of two library builds (in-tree _lib vs PRSP_BSC_LIB=$1): c2 x2 interleaved, c1, c3
set -x
V=$1
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 >> gpurun_out/ab_main_c2.log 2>&1
  PRSP_BSC_LIB=$V timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 >> gpurun_out/ab_var_c2.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 --config c3 --steps 5 > gpurun_out/ab_main_c3.log 2>&1
PRSP_BSC_LIB=$V timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 --config c3 --steps 5 > gpurun_out/ab_var_c3.log 2>&1
PRSP_BSC_LIB=$V timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/ab_var_tests.log 2>&1; echo rc=$? >> gpurun_out/ab_var_tests.log
