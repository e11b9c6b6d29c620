# full label passes seed exit finals in k_label_tile (k_exit_reset skipped): parity tests, A/B timing (MSSZ_EXIT_RESET=1)
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=300 > gpurun_out/pytest33.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest33.log
{
echo "== seeded exits"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device|label"
echo "== k_exit_reset"; MSSZ_EXIT_RESET=1 timeout 600 python tools/class_times.py 2>&1 | grep -E "device|label"
} > gpurun_out/exits33.log 2>&1; cat gpurun_out/exits33.log
