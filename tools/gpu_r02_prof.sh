# r02: ncu --set full of one c2 step's kernels (report kept on the box; CSV pages come back) + launch list
set -x
K='regex:select_kernel|lane_states|lane_finish|oz_gemm_kernel|enumerate_kernel|potrf_diag|solve_rows'
R=/tmp/r02_c2.ncu-rep
timeout 300 python tools/profile_case.py c2 200000 3 > gpurun_out/plain_c2.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -s 26 -c 13 -f -o /tmp/r02_c2 python tools/profile_case.py c2 200000 3 > gpurun_out/ncu_c2.log 2>&1
ncu -i $R --page raw --csv > gpurun_out/r02_c2_raw.csv 2> gpurun_out/ncu_export.log
ncu -i $R --page details --csv > gpurun_out/r02_c2_details.csv 2>> gpurun_out/ncu_export.log
for k in select_kernel lane_states lane_finish oz_gemm_kernel; do
  ncu -i $R --page source --csv --print-source sass --kernel-name regex:$k > gpurun_out/r02_c2_src_$k.csv 2>> gpurun_out/ncu_export.log
done
ls -la $R >> gpurun_out/ncu_export.log
timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/plain_bench.log 2>&1 &&
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launches.log 2>&1
du -sh gpurun_out >> gpurun_out/ncu_export.log
