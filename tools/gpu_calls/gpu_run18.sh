mkdir -p gpurun_out
sw() { echo "== $1"; VAR=$1 VALS="$2" bash tools/sweep_env.sh 2>&1 | sed -E 's/\{.*\}//'; }
sw MSSZ_SMALL_MAX "128 256 512 1024"
sw MSSZ_SPARSE_DIVISOR "32 64 128"
sw MSSZ_RHUGE_DIVISOR "256 512 1024"
sw MSSZ_HUGE_DIVISOR "32 64"
