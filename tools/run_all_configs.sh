#!/bin/bash
# helper for gpurun sessions: tests + bench sweep (not part of the product)
set -u
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
for c in ${CONFIGS:-C1 C2 C5 C3 C4}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup ${WARM:-1} --no-cpu ${EXTRA:-} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
  python - "$c" <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/bench_{c}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(c, "no json", e); print(open(f"gpurun_out/bench_{c}.err").read()[-2000:]); sys.exit()
r=d["roofline"] or {}
print(c, "value %.1f Mv/s  ms/step %.2f  e2e %s" % (d["value"], d["ms_per_step"], (d["e2e"] or {}).get("value")))
print("   roofline", r.get("kernel"), "%.0f GB/s frac %.2f share %.2f" % (r.get("achieved",0), r.get("frac",0), r.get("share_of_device_time") or 0))
print("   stats", d["edit_stats"])
print("   prof", {k:(v["launches"], round(v["ms"],3)) for k,v in d["kernel_profile_ms_per_step"].items()})
PY
done
