# k_label_tile: exits straight to the tile store (40 KB dynamic smem: four CTAs per SM): GPU tests, timing
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=300 > gpurun_out/pytest39.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest39.log
for k in 1 2; do timeout 600 python tools/class_times.py 2>&1 | grep -E "device|label_init"; done > gpurun_out/lt39.log 2>&1; cat gpurun_out/lt39.log
