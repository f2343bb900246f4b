# timing probes of the sliced GEMM at the c2 Y·W shape (tools/ozaki_test.cu built with -DOZ_PROBE=n)
for p in base noepi p4 p5; do
  echo "== $p" >> gpurun_out/probes2.log
  timeout 300 tools/_probes/oz_$p 200000 300 256 20000 >> gpurun_out/probes2.log 2>&1
done
