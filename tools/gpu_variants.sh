set -x
rm -f gpurun_out/probes3.log
timeout 300 tools/_probes/oz_tma 200000 300 256 20000 >> gpurun_out/probes3.log 2>&1
timeout 300 tools/_probes/oz_tma 1000 1000 576 >> gpurun_out/probes3.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --maxfail=6 > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 300 $B > gpurun_out/s_c2.log 2>&1
timeout 600 $B --config c3 --steps 5 > gpurun_out/s_c3.log 2>&1
