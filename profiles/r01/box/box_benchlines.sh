# Bench lines only (default cfg2 with planner tile choice + CPU leg, then cfg1/3/4/5).
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_final2
T=${1:-lines}
timeout 900 python bench.py > gpurun_out/bench_${T}_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${T}_default.log | python profiles/bench_brief.py
for C in ${CFGS:-1 3 4 5}; do
  timeout 1500 python bench.py --config $C --no-cpu > gpurun_out/bench_${T}_c$C.log 2>&1; echo "cfg$C rc=$?"; tail -1 gpurun_out/bench_${T}_c$C.log | python profiles/bench_brief.py
done
