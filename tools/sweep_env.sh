#!/bin/bash
# Sweep one engine env knob on a config: VAR=MSSZ_SPARSE_DIVISOR VALS="..." CONFIG=C4 bash tools/sweep_env.sh
for v in ${VALS}; do
  env ${VAR}=$v timeout 900 python bench.py --config ${CONFIG:-C4} --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/sw_$v.json 2>gpurun_out/sw_$v.err
  python - $v <<'PY'
import json,sys
v=sys.argv[1]
try: d=json.loads(open(f"gpurun_out/sw_{v}.json").read().strip().splitlines()[-1])
except Exception as e: print(v,"fail",open(f"gpurun_out/sw_{v}.err").read()[-800:]); sys.exit()
print(v, "ms %.1f"%d["ms_per_step"], {k:(x["launches"],round(x["ms"],1)) for k,x in d["kernel_profile_ms_per_step"].items() if x["ms"]>1}, d["edit_stats"]["r_iterations"])
PY
done
