# k_rfix_tiles: four tile elements per thread per step (loads of each stage issued together): GPU tests + rfix timing
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=300 > gpurun_out/pytest37.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest37.log
for k in 1 2; do timeout 600 python tools/class_times.py 2>&1 | grep -E "device|rfix"; done > gpurun_out/rfix37.log 2>&1; cat gpurun_out/rfix37.log
