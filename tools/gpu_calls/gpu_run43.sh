# k_fix_list items per lane: 4 (HEAD) vs 8 (variant build)
mkdir -p gpurun_out
cp paper_2406_09423_b200/_lib/libmssz_b200.so /tmp/cur.so
{
echo "== J=4"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device| fix"
cp build/variants/J8.so paper_2406_09423_b200/_lib/libmssz_b200.so
echo "== J=8"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device| fix"
cp /tmp/cur.so paper_2406_09423_b200/_lib/libmssz_b200.so
echo "== J=4"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device| fix"
} > gpurun_out/fix43.log 2>&1; cat gpurun_out/fix43.log
