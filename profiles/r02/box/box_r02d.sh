# Round 2: GPU parity suite after the Euler phase tracking fix; cfg5 A/B of the branching
# Euler form; forward register budget A/B on cfg4.
mkdir -p gpurun_out
T=${1:-r02d}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -15
for br in 0 1; do
  LSQ_EULER_BRANCH=$br timeout 900 python bench.py --config 5 --M 12 --steps 2 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c5_$br.err
  echo "cfg5 branch=$br rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_ab_$T.jsonl
done
for mb in 3 2; do
  LSQ_MINB_FWD=$mb timeout 600 python bench.py --config 4 --M 12 --steps 5 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c4_mb$mb.err
  echo "cfg4 minb_fwd=$mb rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_ab_$T.jsonl
done
for M in 11 13; do
  timeout 600 python bench.py --config 4 --M $M --steps 5 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c4_M$M.err
  echo "cfg4 M=$M rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_ab_$T.jsonl
done
