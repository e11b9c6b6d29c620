#!/bin/bash
# threshold sweep helper (experiments only)
for c in ${CONFIGS:-C3 C4}; do for h in ${DIVS:-64 1024 16384}; do
  MSSZ_HUGE_DIVISOR=$h timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/sw_${c}_$h.json 2>gpurun_out/sw_${c}_$h.err
  python - $c $h <<'PY'
import json,sys
c,h=sys.argv[1:]
try: d=json.loads(open(f"gpurun_out/sw_{c}_{h}.json").read().strip().splitlines()[-1])
except Exception as e: print(c,h,"fail",open(f"gpurun_out/sw_{c}_{h}.err").read()[-1500:]); sys.exit()
st=d["edit_stats"]
print(c, h, "ms %.1f" % d["ms_per_step"], "big", st["big_batches"], "huge", st["huge_batches"], {k:(v["launches"], round(v["ms"],1)) for k,v in d["kernel_profile_ms_per_step"].items() if v["ms"]>1})
PY
done; done
