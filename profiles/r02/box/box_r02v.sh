# Round 2 (session 5): GPU suite after the pass-search fix, then the per-layer plans rebuilt with the
# current compiler (searched passes / phases, merged diagonals, single-buffer forward kernels).
mkdir -p gpurun_out
T=${1:-r02v}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -5
mkdir -p gpurun_out/plans_old && cp profiles/plans/*.json gpurun_out/plans_old/
timeout 2400 python profiles/build_plans.py 4 3 2 5 > gpurun_out/build_plans_$T.log 2>&1; echo "build_plans rc=$?"; tail -6 gpurun_out/build_plans_$T.log
mkdir -p gpurun_out/plans_new && cp profiles/plans/*.json gpurun_out/plans_new/
for c in 4 3 2 5; do
  st=5; [ $c = 5 ] && st=2
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}.err
  echo "cfg$c newplan rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
done
