mkdir -p gpurun_out
for i in 1 2 3; do
timeout -s ABRT 420 python -m pytest tests -q -m gpu -x -o faulthandler_timeout=100 -k "labels or derive or snapshot or verify or slab or segmentation" > gpurun_out/hang7_$i.log 2>&1; echo "run $i rc=$?"; tail -3 gpurun_out/hang7_$i.log
done
