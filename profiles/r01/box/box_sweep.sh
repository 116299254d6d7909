mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_sweep
MRS="${MRS:-12 4,12 5,13 5,13 4,11 4,10 4,12 3}" bash profiles/sweep_tiling.sh ${1:-2}
