mkdir -p gpurun_out
timeout -s ABRT 900 python -m pytest tests -q -m gpu -o faulthandler_timeout=300 > gpurun_out/pytest11.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest11.log
timeout 900 python bench.py --shard --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_shard1.json 2> gpurun_out/bench_shard1.err; echo "shard rc=$?"; tail -c 400 gpurun_out/bench_shard1.json
