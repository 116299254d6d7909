# Re-validate HEAD on the box: GPU parity suite, default bench line, per-config lines.
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_head
T=${1:-head}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$T.log
timeout 900 python bench.py > gpurun_out/bench_${T}_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${T}_default.log | cut -c1-400
for C in ${CFGS:-1 3 4 5}; do
  timeout 1200 python bench.py --config $C --no-cpu > gpurun_out/bench_${T}_c$C.log 2>&1; echo "cfg$C rc=$?"; tail -1 gpurun_out/bench_${T}_c$C.log | cut -c1-250
done
