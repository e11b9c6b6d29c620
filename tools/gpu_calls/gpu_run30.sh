# HEAD (k_label_tile: byte-offset parents, per-thread face masks, full-tile label loop):
# GPU tests, smoke, C4 bench + reference arm, per-class times, launch list, ncu of k_label_tile
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -o faulthandler_timeout=300 > gpurun_out/g30_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/g30_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g30_smoke.log 2>&1; tail -1 gpurun_out/g30_smoke.log
timeout 600 python tools/class_times.py > gpurun_out/g30_class.log 2>&1; cat gpurun_out/g30_class.log
timeout 1500 python bench.py > gpurun_out/g30_bench_c4.json 2> gpurun_out/g30_bench_c4.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g30_bench_c4_ref.json 2> gpurun_out/g30_bench_c4_ref.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g30_launches_c4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile > gpurun_out/g30_launches_run.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/g30_launches_c4.csv > gpurun_out/g30_launches_c4_summary.txt 2>&1
bash tools/ncu_kernels.sh g30 "k_label_tile"
python tools/sass_mix.py gpurun_out/g30_k_label_tile_.source.csv 1073741824 > gpurun_out/g30_label_tile_mix.txt 2>&1 || true
grep -E "Duration|Issue Slots Busy|L1/TEX Cache Throughput|DRAM Throughput|Achieved Occupancy" gpurun_out/g30_k_label_tile_.details.txt
head -3 gpurun_out/g30_label_tile_mix.txt
