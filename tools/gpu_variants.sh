# GPU suite + bench kernel parts at c2 / c3
set -x
echo "== coal" >> gpurun_out/probes2.log
timeout 300 tools/_probes/oz_coal 200000 300 256 20000 >> gpurun_out/probes2.log 2>&1
timeout 300 tools/_probes/oz_coal 1000 1000 576 >> gpurun_out/probes2.log 2>&1
timeout 300 tools/_probes/oz_coal 333 77 100 999 >> gpurun_out/probes2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --maxfail=6 > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
B="python bench.py --no-cpu-baseline --e2e-steps 0"
timeout 300 $B > gpurun_out/z_c2_main.log 2>&1
timeout 600 $B --config c3 --steps 5 > gpurun_out/z_c3_main.log 2>&1
