mkdir -p gpurun_out
timeout -s ABRT 900 python -m pytest tests -q -m gpu -o faulthandler_timeout=300 > gpurun_out/pytest17.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest17.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench17.json 2> gpurun_out/bench17.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench17.json').read().strip().splitlines()[-1]);k=d['kernel_profile_ms_per_step'];print(d['ms_per_step'], {c:round(v['ms'],2) for c,v in k.items()})"
