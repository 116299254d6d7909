# Round 2: GPU suite (with the forced-variant parity test), per-layer plans for the BASELINE
# configs (profiles/plans/), bench cfg4 replaying its plan vs the tile-only choice.
mkdir -p gpurun_out profiles/plans
T=${1:-r02f}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -8
timeout 2400 python profiles/build_plans.py 4 3 2 5 > gpurun_out/build_plans_$T.log 2>&1; echo "plans rc=$?"; cat gpurun_out/build_plans_$T.log | tail -5
mkdir -p gpurun_out/plans; cp profiles/plans/*.json gpurun_out/plans/ 2>/dev/null
for c in 4 3; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c$c.err
  echo "cfg$c plan rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-plan > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_noplan.err
  echo "cfg$c noplan rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
done
