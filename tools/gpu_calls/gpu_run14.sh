mkdir -p gpurun_out
cp paper_2406_09423_b200/_lib/libmssz_b200.so /tmp/main.so
run() { cp paper_2406_09423_b200/_lib/$2 paper_2406_09423_b200/_lib/libmssz_b200.so; timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench14_$1.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/bench14_$1.json').read().strip().splitlines()[-1]);k=d['kernel_profile_ms_per_step'];print('$1', round(d['ms_per_step'],2), {c:round(v['ms'],2) for c,v in k.items() if c in ('directions','label_jump','label_finish','subloop')}, d['edit_stats']['touched'])"; }
run var exp_var.so
run acc exp_acc.so
run j1 exp_j1.so
cp /tmp/main.so paper_2406_09423_b200/_lib/libmssz_b200.so
