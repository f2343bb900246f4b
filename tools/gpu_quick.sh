set -x
for n in 130 200000 199999; do
  CUDA_LAUNCH_BLOCKING=1 BSC_GUARD=1 timeout 300 python tools/_tmp/g1.py $n >> gpurun_out/g1_debug.log 2>&1
done
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --config g1 > gpurun_out/bench_g1.json 2> gpurun_out/bench_g1.err
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_all.log 2>&1; echo rc=$? >> gpurun_out/t_all.log
