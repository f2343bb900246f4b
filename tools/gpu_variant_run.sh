# Scratch driver for one gpurun call: lane-pass carveout / e^P placement A/B (outputs under gpurun_out/)
set -x
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for c in 100 86 72; do BSC_LANE_CARVEOUT=$c timeout 300 $B --config c3 --steps 5 > gpurun_out/cv${c}_c3.log 2>&1; done
cd paper_1908_06843_b200/csrc && touch lane_kernels.cuh && timeout 600 make -j4 NVFLAGS="-std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I. -I../../include -I/usr/local/cuda/include -Xptxas -v -DLANE_EPG_MIN_PAIRS=40" > /dev/null 2>&1; cd ../..
for c in 100 72 58; do BSC_LANE_CARVEOUT=$c timeout 200 $B > gpurun_out/cvg${c}_c2.log 2>&1; done
