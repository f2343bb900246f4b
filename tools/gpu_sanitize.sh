# compute-sanitizer on the smoke case and a small c2-shaped step (one tool per gpurun call):
#   bash tools/gpu_sanitize.sh memcheck | racecheck | synccheck | initcheck
TOOL=${1:-memcheck}
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_plain_smoke.log 2>&1 &&
timeout 300 python tools/profile_case.py c2 3000 1 > gpurun_out/san_plain_c2.log 2>&1 &&
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_${TOOL}_smoke.log 2>&1
echo rc=$? >> gpurun_out/san_${TOOL}_smoke.log
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 python tools/profile_case.py c2 3000 1 > gpurun_out/san_${TOOL}_c2.log 2>&1
echo rc=$? >> gpurun_out/san_${TOOL}_c2.log
