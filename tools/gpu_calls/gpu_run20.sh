mkdir -p gpurun_out
for v in 0 1; do
  if [ $v = 1 ]; then export MSSZ_CROSS_FUSED=1; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench20_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/bench20_$v.json').read().strip().splitlines()[-1]);k=d['kernel_profile_ms_per_step'];print('fused=$v', round(d['ms_per_step'],2), round(k['sparse']['ms'],2), k['sparse']['launches'], d['edit_stats']['touched'])"
done
unset MSSZ_CROSS_FUSED
