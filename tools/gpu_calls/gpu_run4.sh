mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -o faulthandler_timeout=120 -k "test_snapshots_r_targets_and_kernels and multi" -x > gpurun_out/hang_debug.log 2>&1; echo "hang test rc=$?"; tail -40 gpurun_out/hang_debug.log | head -60
timeout 1500 python -m pytest tests -q -m gpu -o faulthandler_timeout=300 --deselect "tests/test_gpu_scale_parity.py::test_snapshots_r_targets_and_kernels[multi-scale-dims0-0-0.001-float32]" > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu4.log
bash tools/sanitize.sh
bash tools/ncu_class_traffic.sh r02_subloop "k_subloop|k_rfix_tiles|k_label_tile|k_exit_reset|k_fix_list"
