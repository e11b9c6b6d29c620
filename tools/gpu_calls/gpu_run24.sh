# K1 col3 v2 (cells + cubes in shared memory, 3 CTAs/SM, interior fast path): A/B parity + timing, ncu
mkdir -p gpurun_out
timeout 900 python tools/k1_ab.py --time > gpurun_out/k1_ab24.log 2>&1; echo "k1_ab rc=$?"; grep -v identical gpurun_out/k1_ab24.log | tail -6; grep -c identical gpurun_out/k1_ab24.log
bash tools/ncu_kernels.sh r24 "k_directions_col3"
python tools/sass_mix.py gpurun_out/r24_k_directions_col3_.source.csv 1073741824 > gpurun_out/r24_mix.txt 2>&1 || true
head -3 gpurun_out/r24_mix.txt
grep -E "Duration|Issue Slots Busy|Achieved Occupancy|No Eligible|DRAM Throughput" gpurun_out/r24_k_directions_col3_.details.txt
