mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu3.log 2>&1; tail -3 gpurun_out/pytest_gpu3.log
for fetch in 0 32 64 128; do
  if [ $fetch = 0 ]; then unset MSSZ_L2_FETCH; else export MSSZ_L2_FETCH=$fetch; fi
  MSSZ_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/l2f_$fetch.json 2> gpurun_out/l2f_$fetch.err
  echo "fetch=$fetch rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/l2f_$fetch.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['kernel_profile_ms_per_step']['subloop'])")"
done
unset MSSZ_L2_FETCH
timeout 2400 python tools/parity_at_scale.py c4 --out gpurun_out/parity_c4.json > /dev/null 2> gpurun_out/parity_c4.err; echo c4 rc=$?; tail -3 gpurun_out/parity_c4.err
timeout 1800 python tools/parity_at_scale.py derive --configs C3 --out gpurun_out/parity_derive_c3.json > /dev/null 2> gpurun_out/parity_derive_c3.err; echo c3 rc=$?; tail -4 gpurun_out/parity_derive_c3.err
