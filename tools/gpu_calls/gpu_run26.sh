# k_label_tile: byte-offset pointers, unconditional doubling stores, terminal label tables; validate f32 vectorised
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_slabs.py tests/test_gpu_verify.py -q -m gpu -x > gpurun_out/pytest26.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest26.log
timeout 600 python tools/class_times.py > gpurun_out/class26.log 2>&1; echo "class rc=$?"; cat gpurun_out/class26.log
