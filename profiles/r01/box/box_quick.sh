mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_quick
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_quick.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_quick.log
MRS="${MRS2:-11 4,12 4}" bash profiles/sweep_tiling.sh 2
[ -n "$CFG4" ] && MRS="12 4" bash profiles/sweep_tiling.sh 4
[ -n "$CFG5" ] && BATCH=${CFG5} MRS="12 4" bash profiles/sweep_tiling.sh 5
true
