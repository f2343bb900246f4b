# r02: the BASELINE.md table — one bench line per config (GPU value, e2e, roofline, cpu_baseline on the box's
# host cores incl. the 1-core figure) and the reference arm at c2
set -x
for c in c0 c1 c2; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 1200 python bench.py --config c3 --steps 10 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 1800 python bench.py --config c4 --steps 5 --e2e-steps 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_c2.json 2> gpurun_out/bench_reference_c2.err
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
