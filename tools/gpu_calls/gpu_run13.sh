mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench13_base.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bench13_base.json').read().strip().splitlines()[-1]);k=d['kernel_profile_ms_per_step'];print('base', d['ms_per_step'], round(k['subloop']['ms'],2))"
cp paper_2406_09423_b200/_lib/libmssz_b200.so /tmp/base.so; cp paper_2406_09423_b200/_lib/exp_occ4.so paper_2406_09423_b200/_lib/libmssz_b200.so
timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench13_occ4.json 2>gpurun_out/bench13_occ4.err
python -c "import json;d=json.loads(open('gpurun_out/bench13_occ4.json').read().strip().splitlines()[-1]);k=d['kernel_profile_ms_per_step'];print('occ4', d['ms_per_step'], round(k['subloop']['ms'],2), d['edit_stats']['touched'])"
cp /tmp/base.so paper_2406_09423_b200/_lib/libmssz_b200.so
