# Round 2: rebalancer A/B on cfg4/cfg3/cfg5 and L2-resident micro-batches on cfg2.
mkdir -p gpurun_out
T=${1:-r02g}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
for c in 4 3; do
  for rb in 0 1; do
    LSQ_REBALANCE=$rb timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_rb$rb.err
    echo "cfg$c rebalance=$rb rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
  done
done
for mb in 0 16 32 64 128; do
  LSQ_MICRO_BATCH=$mb timeout 900 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c2_mb$mb.err
  echo "cfg2 micro_batch=$mb rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
done
