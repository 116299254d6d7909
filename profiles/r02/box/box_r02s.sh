# Round 2 (session 5): first-phase freedom of the forward tiling (LSQ_FIRST_FREE) A/B on cfg4, then
# ncu --set full of one cfg4 step with the merged Euler diagonals and the searched phases.
mkdir -p gpurun_out
T=${1:-r02s}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
run() { # cfg steps label env...
  c=$1; st=$2; lab=$3; shift 3
  env "$@" timeout 1200 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$lab.err
  echo "cfg$c $lab rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"
  cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
}
run 4 5 ff0 LSQ_FIRST_FREE=0
run 4 5 ff1 LSQ_FIRST_FREE=1
C=4; B=0; SC=1; K=19; M=12
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:lsq_jit_p' -c $K -f -o /tmp/full_c${C} \
   python profiles/prof_step.py $C 1 $B > gpurun_out/ncu_full_c${C}_$T.log 2>&1; echo "ncu full cfg$C rc=$?"
python profiles/ncu_summary.py /tmp/full_c${C}.ncu-rep --json gpurun_out/ncu_full_c${C}_$T.json > gpurun_out/ncu_full_c${C}_$T.txt 2>&1
for k in p0_m2 p1_m2 p1_m0; do
  ncu -i /tmp/full_c${C}.ncu-rep --page source --csv --print-source sass -k regex:lsq_jit_$k > gpurun_out/src_${k}_$T.csv 2>/dev/null
  python profiles/sass_hist.py gpurun_out/src_${k}_$T.csv > gpurun_out/sass_hist_${k}_$T.txt 2>&1
done
ls -la gpurun_out | tail -12
