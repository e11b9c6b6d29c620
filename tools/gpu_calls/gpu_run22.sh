# register-column K1 (k_directions_col3): A/B parity against k_directions_reg3 + C4 timing, GPU direction tests
mkdir -p gpurun_out
timeout 900 python tools/k1_ab.py --time > gpurun_out/k1_ab.log 2>&1; echo "k1_ab rc=$?"; tail -8 gpurun_out/k1_ab.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest22.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest22.log
