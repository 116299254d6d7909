# Round 2 (session 5): old (session-3) plans vs the plans rebuilt in box_r02v, same box, cfg4 and cfg5;
# the tensor-core block measurement (profiles/micro/tf32_block.py); the new compiler-knob GPU tests.
mkdir -p gpurun_out
T=${1:-r02w}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
python profiles/micro/tf32_block.py > gpurun_out/tf32_block_$T.txt 2>&1; echo "tf32 rc=$?"; cat gpurun_out/tf32_block_$T.txt
cp profiles/plans/cfg4.json /tmp/cfg4_old.json; cp profiles/plans/cfg5.json /tmp/cfg5_old.json
run() { # cfg steps label
  c=$1; st=$2; lab=$3
  timeout 1200 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$lab.err
  echo "cfg$c $lab rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
}
run 4 5 oldplan
cp profiles/plans_candidates/cfg4_new.json profiles/plans/cfg4.json; run 4 5 newplan
cp /tmp/cfg4_old.json profiles/plans/cfg4.json; run 4 5 oldplan_again
run 5 2 oldplan
cp profiles/plans_candidates/cfg5_new.json profiles/plans/cfg5.json; run 5 2 newplan
cp /tmp/cfg5_old.json profiles/plans/cfg5.json
timeout 1500 python -m pytest tests -m gpu -q -rA -k "compiler_knobs" > gpurun_out/pytest_gpu_knobs_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_knobs_$T.log | tail -5
