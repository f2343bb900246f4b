# Final evidence run for one gpurun call: full c3/c4 bench lines and the c3 full-size parity check
set -x
timeout 600 python bench.py --config c3 --steps 10 > gpurun_out/final2_c3.log 2>&1
timeout 900 python bench.py --config c4 --steps 5 --e2e-steps 0 > gpurun_out/final2_c4.log 2>&1
timeout 1100 python tools/trajectory_check.py c3 1 > gpurun_out/parity2_c3.txt 2>&1
