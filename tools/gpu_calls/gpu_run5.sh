# round-2 evidence: bench lines (C4 + same-config C1/C2 with the reference arm),
# launch list, ncu captures of every hot-path kernel class
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke5.log 2>&1; tail -1 gpurun_out/smoke5.log
timeout 1200 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c4_ref.json 2> gpurun_out/bench_c4_ref.err; echo "ref c4 rc=$?"
for c in C1 C2 C5; do
  cd=""; [ $c = C5 ] && cd="--cpu-dims 3600x2400"
  timeout 900 python bench.py --config $c $cd > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  timeout 1500 python bench.py --config $c $cd --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${c}_ref.json 2> gpurun_out/bench_${c}_ref.err; echo "ref $c rc=$?"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile > gpurun_out/launches_run.log 2>&1; echo "launches rc=$?"
bash tools/ncu_kernels.sh full "k_label_finish" "k_exit_reset" "k_exit_jump_tiles" "k_label_exit_jump" "k_frontier" "k_compact_write" "k_compact_count" "k_cross_chunks" "k_cross<" "k_upstream" "k_validate" "k_detect_dirty" "k_count_false" "k_up_targets" "k_expand_targets" "k_fix_list" "k_rfix_tiles" "k_label_tile" "k_directions_reg3" "k_detect_kind"
SKIP=1 bash tools/ncu_kernels.sh full "k_subloop"
