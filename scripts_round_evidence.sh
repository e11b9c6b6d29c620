#!/bin/bash
# Round evidence: GPU tests, smoke, default bench (C4 + CPU baseline + e2e), reference arm,
# ncu launch list, and full ncu captures of the top kernels (text exports only).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 300 gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile > gpurun_out/launches_run.log 2>&1; echo "launches rc=$?"
bash tools/ncu_kernels.sh full "k_label_tile" "k_directions_reg3" "k_rfix_tiles" "k_detect_kind" "k_fix_list"
SKIP=1 bash tools/ncu_kernels.sh full "k_subloop"
