# gdir refresh sweeps stamp changed chunks (kinds stay incremental, sparse X stays incremental): GPU tests, A/B (MSSZ_K1_NOSTAMP=1)
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=300 > gpurun_out/pytest44.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest44.log
{
echo "== stamped"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device|directions|detect|sparse"
echo "== not stamped"; MSSZ_K1_NOSTAMP=1 timeout 600 python tools/class_times.py 2>&1 | grep -E "device|directions|detect|sparse"
echo "== stamped"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device|directions|detect|sparse"
} > gpurun_out/stamp44.log 2>&1; cat gpurun_out/stamp44.log
