# Round 2 (session 5): last knob sweep on cfg4 with the final compiler (single-buffer forward kernels,
# searched partitions): forward CTAs per SM, coupling chains, lazy swizzle bases, turnaround buffers.
mkdir -p gpurun_out
T=${1:-r02af}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
run() { # cfg steps label env...
  c=$1; st=$2; lab=$3; shift 3
  env "$@" timeout 1200 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$lab.err
  echo "cfg$c $lab rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
}
run 4 5 base LSQ_SKEW_NS=0
run 4 5 minb5 LSQ_MINB_FWD5=5
run 4 5 minb3 LSQ_MINB_FWD5=3
run 4 5 chains2 LSQ_COUPLING_CHAINS=2
run 4 5 lazy0 LSQ_LAZY_SX=0
run 4 5 rotturn0 LSQ_ROT_TURN=0
run 4 5 rfwd4 LSQ_R_FWD=4
run 4 5 base2 LSQ_SKEW_NS=0
