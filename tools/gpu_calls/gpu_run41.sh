# occupancy: k_frontier (256, 6) and k_upstream (512, 3): GPU tests + frontier/sparse timing
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=300 > gpurun_out/pytest41.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest41.log
for k in 1 2; do timeout 600 python tools/class_times.py 2>&1 | grep -E "device|frontier|sparse"; done > gpurun_out/occ41.log 2>&1; cat gpurun_out/occ41.log
