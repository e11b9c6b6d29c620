# confirm the R-batch full-sweep threshold (MSSZ_RHUGE_DIVISOR) after the faster K1
mkdir -p gpurun_out
{
for d in 512 384 256 512 384 256; do echo "== MSSZ_RHUGE_DIVISOR=$d"; MSSZ_RHUGE_DIVISOR=$d timeout 600 python tools/class_times.py 2>&1 | grep -E "device"; done
} > gpurun_out/sweep36.log 2>&1; cat gpurun_out/sweep36.log
