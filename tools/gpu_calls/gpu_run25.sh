# K1 col3 v3 (cells in shared memory, C shuffled, 2 CTAs/SM, interior fast path): A/B parity + timing, ncu
mkdir -p gpurun_out
timeout 900 python tools/k1_ab.py --time > gpurun_out/k1_ab25.log 2>&1; echo "k1_ab rc=$?"; grep -v identical gpurun_out/k1_ab25.log | tail -6; grep -c identical gpurun_out/k1_ab25.log
bash tools/ncu_kernels.sh r25 "k_directions_col3"
python tools/sass_mix.py gpurun_out/r25_k_directions_col3_.source.csv 1073741824 > gpurun_out/r25_mix.txt 2>&1 || true
head -3 gpurun_out/r25_mix.txt
grep -E "Duration|Issue Slots Busy|Achieved Occupancy|No Eligible|DRAM Throughput" gpurun_out/r25_k_directions_col3_.details.txt
