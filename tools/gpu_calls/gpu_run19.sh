mkdir -p gpurun_out
timeout -s ABRT 900 python -m pytest tests -q -m gpu -o faulthandler_timeout=300 > gpurun_out/pytest19.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest19.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench19.json 2> gpurun_out/bench19.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench19.json').read().strip().splitlines()[-1]);k=d['kernel_profile_ms_per_step'];print(d['ms_per_step'], {c:round(v['ms'],2) for c,v in k.items()})"
sw() { echo "== $1"; VAR=$1 VALS="$2" bash tools/sweep_env.sh 2>&1 | sed -E 's/\{.*\}//'; }
sw MSSZ_RHUGE_DIVISOR "128 192 256 384"
sw MSSZ_SMALL_MAX "64 128 192"
