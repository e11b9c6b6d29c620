mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rgp tools/random_gather_peak.cu && /tmp/rgp 4 > gpurun_out/random_gather_peak.json; cat gpurun_out/random_gather_peak.json
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/random_gather_ncu.csv /tmp/rgp 4 > /dev/null 2>&1; echo "rgp ncu rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-profile > gpurun_out/launches_run.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/launches_c4.csv > gpurun_out/launches_c4_summary.txt 2>&1; head -40 gpurun_out/launches_c4_summary.txt
bash tools/ncu_kernels.sh full "k_label_finish" "k_exit_reset" "k_exit_jump_tiles" "k_label_exit_jump" "k_frontier" "k_compact_write" "k_compact_count" "k_cross_chunks" "k_cross<" "k_upstream" "k_validate" "k_detect_dirty" "k_count_false" "k_up_targets" "k_expand_targets" "k_fix_list" "k_rfix_tiles" "k_label_tile" "k_directions_reg3" "k_detect_kind"
SKIP=1 bash tools/ncu_kernels.sh full "k_subloop"
