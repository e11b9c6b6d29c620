mkdir -p gpurun_out
cp paper_2406_09423_b200/_lib/libmssz_b200.so /tmp/main.so
run() { cp $2 paper_2406_09423_b200/_lib/libmssz_b200.so; timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench15_$1.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/bench15_$1.json').read().strip().splitlines()[-1]);k=d['kernel_profile_ms_per_step'];print('$1', round(d['ms_per_step'],2), {c:round(v['ms'],2) for c,v in k.items() if c in ('sparse','frontier','subloop')}, d['edit_stats']['touched'])"; }
run main /tmp/main.so
run var2 paper_2406_09423_b200/_lib/exp_var2.so
cp /tmp/main.so paper_2406_09423_b200/_lib/libmssz_b200.so
