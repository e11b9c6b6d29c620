# round-2 evidence recipe (HEAD): GPU tests, smoke, bench lines + reference arm, launch list, DRAM traffic, sanitizers, C4 snapshot parity
mkdir -p gpurun_out
timeout -s ABRT 1200 python -m pytest tests -q -m gpu -o faulthandler_timeout=300 > gpurun_out/f4_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f4_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; tail -1 gpurun_out/f4_smoke.log
timeout 1500 python bench.py > gpurun_out/f4_bench_c4.json 2> gpurun_out/f4_bench_c4.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f4_bench_c4_ref.json 2> gpurun_out/f4_bench_c4_ref.err; echo "ref rc=$?"
for c in C1 C2 C5; do
  cd=""; [ $c = C5 ] && cd="--cpu-dims 3600x2400"
  timeout 900 python bench.py --config $c $cd > gpurun_out/f4_bench_$c.json 2> gpurun_out/f4_bench_$c.err; echo "bench $c rc=$?"
  timeout 1500 python bench.py --config $c $cd --impl reference --steps 2 --warmup 1 > gpurun_out/f4_bench_${c}_ref.json 2> gpurun_out/f4_bench_${c}_ref.err; echo "ref $c rc=$?"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f4_launches_c4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile > gpurun_out/f4_launches_run.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/f4_launches_c4.csv > gpurun_out/f4_launches_c4_summary.txt 2>&1
bash tools/ncu_class_traffic.sh f4 "k_subloop|k_rfix_tiles|k_label_tile|k_exit_jump_tiles|k_fix_list|k_directions_col3|k_label_finish"
# compute-sanitizer is closed on this pool (round 2): bash tools/sanitize.sh
timeout 2400 python tools/parity_at_scale.py c4 --out gpurun_out/f4_parity_c4.json > /dev/null 2> gpurun_out/f4_parity_c4.err; echo "c4 parity rc=$?"; tail -2 gpurun_out/f4_parity_c4.err
