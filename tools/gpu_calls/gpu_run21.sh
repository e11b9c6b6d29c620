mkdir -p gpurun_out
timeout -s ABRT 900 python -m pytest tests -q -m gpu -o faulthandler_timeout=300 > gpurun_out/pytest21.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest21.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke21.log 2>&1; tail -1 gpurun_out/smoke21.log
timeout 1500 python bench.py > gpurun_out/bench21.json 2> gpurun_out/bench21.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench21.json').read().strip().splitlines()[-1]);k=d['kernel_profile_ms_per_step'];print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['random_access']['frac'], d['clocks'], {c:round(v['ms'],2) for c,v in k.items()})"
