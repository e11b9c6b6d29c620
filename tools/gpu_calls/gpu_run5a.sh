mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu5.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke5.log 2>&1; tail -1 gpurun_out/smoke5.log
bash tools/sanitize.sh
timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c4_ref.json 2> gpurun_out/bench_c4_ref.err; echo "ref c4 rc=$?"
for c in C1 C2 C5; do
  cd=""; [ $c = C5 ] && cd="--cpu-dims 3600x2400"
  timeout 900 python bench.py --config $c $cd > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  timeout 1500 python bench.py --config $c $cd --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${c}_ref.json 2> gpurun_out/bench_${c}_ref.err; echo "ref $c rc=$?"
done
