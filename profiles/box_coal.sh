mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_coal
for C in 2 3; do
  LSQ_COAL=$C MRS="12 4,11 4,13 4" bash profiles/sweep_tiling.sh 2
  LSQ_COAL=$C MRS="12 4,13 4" bash profiles/sweep_tiling.sh 4
done
LSQ_COAL=4 MRS="12 4,13 4" bash profiles/sweep_tiling.sh 4
