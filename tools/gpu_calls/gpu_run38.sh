# final HEAD verification: GPU tests, smoke, default bench (C4) + reference arm
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -o faulthandler_timeout=300 > gpurun_out/g38_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/g38_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g38_smoke.log 2>&1; tail -1 gpurun_out/g38_smoke.log
timeout 1500 python bench.py > gpurun_out/g38_bench_c4.json 2> gpurun_out/g38_bench_c4.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g38_bench_c4_ref.json 2> gpurun_out/g38_bench_c4_ref.err; echo "ref rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/g38_bench_c4.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks'])"
