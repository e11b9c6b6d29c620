# k_label_tile: shared-window pointers (7 instr per doubling step), conditional stores, terminal label tables
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_slabs.py tests/test_gpu_verify.py -q -m gpu -x > gpurun_out/pytest27.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest27.log
timeout 600 python tools/class_times.py > gpurun_out/class27.log 2>&1; echo "class rc=$?"; cat gpurun_out/class27.log
