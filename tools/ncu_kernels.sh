#!/bin/bash
# Full ncu captures of selected kernels of one bench step (one filtered pass per kernel).
#   bash tools/ncu_kernels.sh <tag> <kernel-regex> [<kernel-regex> ...]
# env: CONFIG (C4), COUNT (launches per kernel, default 1), SKIP (launches to skip, default 0),
#      KEEP=1 keeps the .ncu-rep (they are large: gpurun copies back <= 64 MiB)
# Writes gpurun_out/<tag>_<kernel>.{details.txt,raw.csv,source.csv}.
set -u
tag=$1; shift
mkdir -p gpurun_out
for k in "$@"; do
  name=$(echo "$k" | tr -c 'A-Za-z0-9_' '_' | cut -c1-40)
  rep="gpurun_out/${tag}_${name}"
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$k" \
    -s "${SKIP:-0}" -c "${COUNT:-1}" -o "$rep" -f \
    python bench.py --config "${CONFIG:-C4}" --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile \
    > "${rep}.log" 2>&1
  echo "$k rc=$?"
  ncu -i "${rep}.ncu-rep" --page details > "${rep}.details.txt" 2>&1
  ncu -i "${rep}.ncu-rep" --page raw --csv > "${rep}.raw.csv" 2>&1
  ncu -i "${rep}.ncu-rep" --page source --csv > "${rep}.source.csv" 2>&1
  [ "${KEEP:-0}" = 1 ] || rm -f "${rep}.ncu-rep"
done
