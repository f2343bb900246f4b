# Final evidence run for one gpurun call: full bench lines (e2e + cpu_baseline) for c2/c3/c4 and the reference arm
set -x
timeout 400 python bench.py > gpurun_out/final_c2.log 2>&1
timeout 600 python bench.py --config c3 --steps 10 > gpurun_out/final_c3.log 2>&1
timeout 900 python bench.py --config c4 --steps 5 --e2e-steps 0 > gpurun_out/final_c4.log 2>&1
timeout 400 python bench.py --impl reference > gpurun_out/final_ref_c2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_c3.log 2>&1
