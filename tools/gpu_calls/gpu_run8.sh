mkdir -p gpurun_out
for i in 1 2 3 4; do
timeout -s ABRT 600 python -m pytest tests -q -m gpu -o faulthandler_timeout=150 > gpurun_out/pytest8_$i.log 2>&1; echo "run $i rc=$?"; tail -2 gpurun_out/pytest8_$i.log
done
