# K1 x-pairs shuffle the key only; R-batch full-sweep threshold sweep (MSSZ_RHUGE_DIVISOR) after the faster K1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest35.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest35.log
timeout 900 python tools/k1_ab.py > gpurun_out/k1_ab35.log 2>&1; echo "k1_ab rc=$?"; grep -c identical gpurun_out/k1_ab35.log
{
for d in 256 128 512 1024 256; do echo "== MSSZ_RHUGE_DIVISOR=$d"; MSSZ_RHUGE_DIVISOR=$d timeout 600 python tools/class_times.py 2>&1 | grep -E "device|directions|frontier|sparse|label_init"; done
} > gpurun_out/sweep35.log 2>&1; cat gpurun_out/sweep35.log
