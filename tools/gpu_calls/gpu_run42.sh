# k_fix_list with four list items per lane in flight (MSSZ_FIX_LIST_PER_LANE=4): GPU tests + fix timing
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=300 > gpurun_out/pytest42.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest42.log
for k in 1 2; do timeout 600 python tools/class_times.py 2>&1 | grep -E "device| fix"; done > gpurun_out/fix42.log 2>&1; cat gpurun_out/fix42.log
