# ncu full capture of the register-column K1 (k_directions_col3), one launch of a C4 step
mkdir -p gpurun_out
bash tools/ncu_kernels.sh r23 "k_directions_col3"
python tools/ncu_full_summary.py gpurun_out/r23_k_directions_col3.details.txt > gpurun_out/r23_summary.txt 2>&1 || true
python tools/sass_mix.py gpurun_out/r23_k_directions_col3.source.csv 1073741824 > gpurun_out/r23_mix.txt 2>&1 || true
