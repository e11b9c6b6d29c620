# sparse R pass: X from scratch by the streaming k_cross_all: GPU tests, A/B timing (MSSZ_CROSS_CHUNKS=1)
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=300 > gpurun_out/pytest34.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest34.log
{
echo "== k_cross_all"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device|sparse"
echo "== k_cross_chunks"; MSSZ_CROSS_CHUNKS=1 timeout 600 python tools/class_times.py 2>&1 | grep -E "device|sparse"
} > gpurun_out/cross34.log 2>&1; cat gpurun_out/cross34.log
