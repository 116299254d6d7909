# Round 2 (session 5): stress seeds 3, 5..8 after the repeated-bit fix; rebalance budget sweep on cfg5 / cfg2.
mkdir -p gpurun_out
T=${1:-r02z}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
for s in 3 5 6 7 8; do
  timeout 1200 python profiles/stress_structured.py 100 $s > gpurun_out/stress_${T}_s$s.txt 2>&1; echo "stress seed $s rc=$? $(tail -1 gpurun_out/stress_${T}_s$s.txt)"
done
run() { # cfg steps label env...
  c=$1; st=$2; lab=$3; shift 3
  env "$@" timeout 1200 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$lab.err
  echo "cfg$c $lab rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
}
for b in 40 120 160 220; do run 2 10 budget$b LSQ_REBALANCE_BUDGET=$b; done
for b in 40 120 160; do run 5 2 budget$b LSQ_REBALANCE_BUDGET=$b; done
run 3 5 budget160 LSQ_REBALANCE_BUDGET=160
true
