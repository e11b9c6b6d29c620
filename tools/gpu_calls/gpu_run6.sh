mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "labels or derive or snapshot or verify or slab or segmentation" > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu6.log
for sk in 0 1; do
  MSSZ_LABEL_SKIP=$sk timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/lskip_$sk.json 2> gpurun_out/lskip_$sk.err
  echo "skip=$sk rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/lskip_$sk.json').read().strip().splitlines()[-1]);k=d['kernel_profile_ms_per_step'];print(round(d['ms_per_step'],2), k['label_init'], k['label_finish'])")"
done
