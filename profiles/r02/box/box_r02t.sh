# Round 2 (session 5): single-buffer forward kernels (LSQ_FWD_SINGLE: stage == exchange buffer, 4 CTAs/SM)
# A/B on cfg4/3/2/5; first-wave CTA skew re-measured on cfg4; GPU suite.
mkdir -p gpurun_out
T=${1:-r02t}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
run() { # cfg steps label env...
  c=$1; st=$2; lab=$3; shift 3
  env "$@" timeout 1200 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$lab.err
  echo "cfg$c $lab rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"
  cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
}
for c in 4 3 2; do
  run $c 5 single0 LSQ_FWD_SINGLE=0
  run $c 5 single1 LSQ_FWD_SINGLE=1
done
run 5 2 single0 LSQ_FWD_SINGLE=0
run 5 2 single1 LSQ_FWD_SINGLE=1
run 4 5 skew_m1_6000 LSQ_SKEW_NS=6000 LSQ_SKEW_MODE=1
run 4 5 skew_m3_12000 LSQ_SKEW_NS=12000 LSQ_SKEW_MODE=3
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA -x > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -5
