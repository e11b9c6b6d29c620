# k_label_tile variants A/B (A = HEAD; B..E = shared-window pointers + terminal label tables at
# threads/minBlocks 512/2, 1024/1, 1024/2, 512/3): per-class times of a C4 derive
mkdir -p gpurun_out
cp paper_2406_09423_b200/_lib/libmssz_b200.so /tmp/cur.so
for v in A B C D E; do
  cp build/variants/$v.so paper_2406_09423_b200/_lib/libmssz_b200.so
  echo "== $v"; timeout 600 python tools/class_times.py 2>&1 | grep -E "device|label_init|label_jump|rfix"
done > gpurun_out/variants28.log
cp /tmp/cur.so paper_2406_09423_b200/_lib/libmssz_b200.so
cat gpurun_out/variants28.log
