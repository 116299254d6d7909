# Round 2 (session 4): first-wave CTA skew experiment (de-phasing the CTAs that share an SM) on cfg4.
mkdir -p gpurun_out
T=${1:-r02o}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
run() { # label, env...
  lab=$1; shift
  env "$@" timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_$lab.err
  echo "cfg4 $lab rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"
  cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
}
run base LSQ_SKEW_NS=0
for m in 1 2 3; do
  for ns in 6000 12000; do
    run skew_m${m}_${ns} LSQ_SKEW_NS=$ns LSQ_SKEW_MODE=$m
  done
done
run skew_m3_12000_fwd LSQ_SKEW_NS=12000 LSQ_SKEW_MODE=3 LSQ_SKEW_FWD=1
run base2 LSQ_SKEW_NS=0
