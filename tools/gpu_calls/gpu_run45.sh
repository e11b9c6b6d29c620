# final build: launch list of one C4 bench step + DRAM traffic of the main kernels
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f5_launches_c4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile > gpurun_out/f5_launches_run.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/f5_launches_c4.csv > gpurun_out/f5_launches_c4_summary.txt 2>&1; head -16 gpurun_out/f5_launches_c4_summary.txt
bash tools/ncu_class_traffic.sh f5 "k_subloop|k_rfix_tiles|k_label_tile|k_exit_jump_tiles|k_fix_list|k_directions_col3|k_label_finish"
