# Round 2: GPU suite on the current kernels + A/B of immediate-offset swizzled shared accesses.
mkdir -p gpurun_out
T=${1:-r02h}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -8
for c in 4 3 5; do
  for v in 0 1; do
    st=5; [ $c = 5 ] && st=2
    LSQ_SWZ_IMM=$v timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_imm$v.err
    echo "cfg$c swz_imm=$v rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
  done
done
