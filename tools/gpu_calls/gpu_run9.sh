mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do
MSSZ_TRACE=1 timeout -s ABRT 200 python -m pytest tests -q -s -m gpu -x -o faulthandler_timeout=120 -k "test_troublemaker_kats or test_snapshots_r_targets_and_kernels" > gpurun_out/hang9_$i.log 2>&1; echo "run $i rc=$?"; grep -v "^\[mssz\] [CR] " gpurun_out/hang9_$i.log | grep "mssz\]" | tail -4
done
