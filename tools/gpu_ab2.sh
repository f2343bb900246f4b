set -x
for i in 1 2; do
  for v in u u8; do
    PRSP_BSC_LIB=paper_1908_06843_b200/_lib_$v/libprsp_bsc_b200.so timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 >> gpurun_out/ab2_${v}_c2.log 2>&1
  done
done
for v in u u8; do
  PRSP_BSC_LIB=paper_1908_06843_b200/_lib_$v/libprsp_bsc_b200.so timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 --config c3 --steps 5 > gpurun_out/ab2_${v}_c3.log 2>&1
done
