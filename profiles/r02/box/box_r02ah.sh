# Round 2 (session 5): five forward CTAs per SM (LSQ_MINB_FWD5=5, 102 registers) on the other configs,
# as evidence for the next round (the default stays at 4).
mkdir -p gpurun_out
T=${1:-r02ah}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
run() { c=$1; st=$2; lab=$3; shift 3
  env "$@" timeout 1200 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$lab.err
  echo "cfg$c $lab rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl; }
for c in 3 2; do run $c 10 minb4 LSQ_MINB_FWD5=4; run $c 10 minb5 LSQ_MINB_FWD5=5; done
run 5 2 minb4 LSQ_MINB_FWD5=4; run 5 2 minb5 LSQ_MINB_FWD5=5
