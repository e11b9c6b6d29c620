#!/bin/bash
# Round evidence: tests, default bench (C4 + cpu baseline), reference arm, ncu launch list, ncu full capture.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_default.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"; tail -c 400 gpurun_out/bench_reference.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile > gpurun_out/launches_run.log 2>&1; echo "launches rc=$?"; wc -l gpurun_out/launches_c4.csv
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:k_(subloop|rfix|label_tile|directions_tiled|detect_kind|label_exit_jump|count_false)" -c 12 -o gpurun_out/prof_c4_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile > gpurun_out/prof_run.log 2>&1; echo "ncu full rc=$?"
