#!/bin/bash
# DRAM traffic of EVERY launch of the given kernels in one C4 bench step
# (metrics only, application replay: the engine is deterministic), summarised
# per kernel into gpurun_out/<tag>_traffic.json by tools/ncu_traffic_summary.py.
#   bash tools/ncu_class_traffic.sh <tag> <kernel-regex>
set -u
tag=$1; rx=$2
mkdir -p gpurun_out
timeout 2400 ncu --replay-mode application --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  -k "regex:$rx" --csv --log-file gpurun_out/${tag}_traffic.csv \
  python bench.py --config "${CONFIG:-C4}" --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile \
  > gpurun_out/${tag}_traffic.log 2>&1
echo "ncu traffic rc=$?"
python tools/ncu_traffic_summary.py gpurun_out/${tag}_traffic.csv > gpurun_out/${tag}_traffic.json
cat gpurun_out/${tag}_traffic.json
