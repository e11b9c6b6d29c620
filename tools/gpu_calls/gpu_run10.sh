mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
MSSZ_TRACE=1 timeout -s ABRT 200 python -m pytest tests -q -s -m gpu -x -o faulthandler_timeout=120 -k "test_troublemaker_kats or test_snapshots_r_targets_and_kernels" > gpurun_out/hang10_$i.log 2>&1; echo "run $i rc=$?"; tail -1 gpurun_out/hang10_$i.log
done
for i in 1 2; do
timeout -s ABRT 600 python -m pytest tests -q -m gpu -o faulthandler_timeout=150 > gpurun_out/pytest10_$i.log 2>&1; echo "full run $i rc=$?"; tail -1 gpurun_out/pytest10_$i.log
done
