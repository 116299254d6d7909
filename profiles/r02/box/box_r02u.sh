# Round 2 (session 5): beam-searched pass partition (LSQ_PASS_BEAM: 1 = greedy) A/B on cfg4 at the
# benched plan and at M = 11 / 13 tile-only plans; GPU suite with it on.
mkdir -p gpurun_out
T=${1:-r02u}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
run() { # cfg steps label extra-args env...
  c=$1; st=$2; lab=$3; extra=$4; shift 4
  env "$@" timeout 1200 python bench.py --config $c --steps $st --warmup 3 --no-cpu $extra > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$lab.err
  echo "cfg$c $lab rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"
  cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
}
run 4 5 beam1 "" LSQ_PASS_BEAM=1
run 4 5 beam8 "" LSQ_PASS_BEAM=8
run 4 5 beam1_M13 "--M 13" LSQ_PASS_BEAM=1
run 4 5 beam8_M13 "--M 13" LSQ_PASS_BEAM=8
run 4 5 beam8_M11 "--M 11" LSQ_PASS_BEAM=8
run 3 5 beam8_M13 "--M 13" LSQ_PASS_BEAM=8
run 3 5 beam8_M12 "--M 12" LSQ_PASS_BEAM=8
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA -x > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -5
