# dense R batches (k_mark_targets + k_fix_bits) and k_label_tile (byte-offset pointers,
# per-thread face masks): GPU parity tests, then per-class C4 times:
# cur, cur with dense R batches off, A = both off (col3 K1 build)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py tests/test_gpu_slabs.py tests/test_gpu_verify.py -q -m gpu -x > gpurun_out/pytest29.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest29.log
cp paper_2406_09423_b200/_lib/libmssz_b200.so /tmp/cur.so
{
echo "== cur"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device|label_init|fix|rfix"
echo "== cur, dense R off"; MSSZ_RDENSE_DIVISOR=1 timeout 600 python tools/class_times.py 2>&1 | grep -E "device|label_init|fix|rfix"
cp build/variants/K.so paper_2406_09423_b200/_lib/libmssz_b200.so
echo "== K (K1 x-pairs shuffle the key only)"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device|directions"
cp build/variants/A.so paper_2406_09423_b200/_lib/libmssz_b200.so
echo "== A"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device|label_init|fix|rfix"
cp /tmp/cur.so paper_2406_09423_b200/_lib/libmssz_b200.so
} > gpurun_out/variants29.log 2>&1
cat gpurun_out/variants29.log
