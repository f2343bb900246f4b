# ncu --set full of the M-step row solves (third c2 step): raw metrics + SASS source page
set -x
R=/tmp/r02_solve.ncu-rep
timeout 300 python tools/profile_case.py c2 20000 3 > gpurun_out/plain_solve.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:solve_rows|potrf_diag|trsm_panel" -s 22 -c 11 -f -o /tmp/r02_solve python tools/profile_case.py c2 20000 3 > gpurun_out/ncu_solve.log 2>&1
ncu -i $R --page raw --csv > gpurun_out/r02_solve_raw.csv 2> gpurun_out/ncu_export_solve.log
ncu -i $R --page source --csv --print-source sass --kernel-name regex:solve_rows > gpurun_out/r02_solve_src.csv 2>> gpurun_out/ncu_export_solve.log
ncu -i $R --page source --csv --print-source sass --kernel-name regex:potrf_diag > gpurun_out/r02_potrf_src.csv 2>> gpurun_out/ncu_export_solve.log
