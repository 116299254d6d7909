# Round 2 (session 4): state check after container re-creation: GPU suite, cfg4 bench,
# and cfg4 with every RZ layer forced into diagonal runs (SPLIT everywhere) for A/B.
mkdir -p gpurun_out
T=${1:-r02m}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -8
for v in default noplan splitall; do
  env=""; fl=""
  [ $v = noplan ] && fl="--no-plan"
  [ $v = splitall ] && { env="LSQ_SPLIT_FORCE=1"; fl="--no-plan"; }
  env $env timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu $fl > /tmp/b.json 2> gpurun_out/bench_${T}_c4_$v.err
  echo "cfg4 $v rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"
  cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
done
