mkdir -p gpurun_out
timeout 1200 python tools/parity_at_scale.py c4 --config C5 --out gpurun_out/parity_c5_snap.json > /dev/null 2> gpurun_out/parity_c5_snap.err; echo "c5 rc=$?"; tail -2 gpurun_out/parity_c5_snap.err
timeout 2400 python tools/parity_at_scale.py c4 --config C3 --out gpurun_out/parity_c3_snap.json > /dev/null 2> gpurun_out/parity_c3_snap.err; echo "c3 rc=$?"; tail -2 gpurun_out/parity_c3_snap.err
