# final build bench line (C4) + smoke
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g40_smoke.log 2>&1; tail -1 gpurun_out/g40_smoke.log
timeout 1500 python bench.py > gpurun_out/g40_bench_c4.json 2> gpurun_out/g40_bench_c4.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/g40_bench_c4.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks'], {c:round(v['ms_per_step'],2) for c,v in d['roofline']['per_class'].items()})"
