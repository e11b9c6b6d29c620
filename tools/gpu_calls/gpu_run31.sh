# k_label_tile TMA tile loads (cp.async.bulk.tensor.3d + mbarrier): parity tests, A/B timing (MSSZ_LABEL_TMA=0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_verify.py tests/test_gpu_slabs.py tests/test_gpu_scale_parity.py -q -m gpu -x > gpurun_out/pytest31.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest31.log
{
echo "== TMA"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device|label_init"
echo "== no TMA"; MSSZ_LABEL_TMA=0 timeout 600 python tools/class_times.py 2>&1 | grep -E "device|label_init"
} > gpurun_out/tma31.log 2>&1; cat gpurun_out/tma31.log
cuobjdump -sass paper_2406_09423_b200/_lib/libmssz_b200.so | grep -c UTMALDG
