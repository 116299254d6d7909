# Round 2 (session 5): state of HEAD after the container was re-created: GPU suite, default bench, cfg2/3/5 lines.
mkdir -p gpurun_out
T=${1:-r02p}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_$T.txt
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -5
timeout 1200 python bench.py > gpurun_out/bench_${T}_default.jsonl 2> gpurun_out/bench_${T}_default.err; echo "bench default rc=$?"
python profiles/bench_brief.py < gpurun_out/bench_${T}_default.jsonl
for C in 2 3 5; do
  st=10; [ $C = 5 ] && st=3
  timeout 1500 python bench.py --config $C --steps $st --no-cpu > gpurun_out/bench_${T}_c$C.jsonl 2> gpurun_out/bench_${T}_c$C.err; echo "cfg$C rc=$?"
  python profiles/bench_brief.py < gpurun_out/bench_${T}_c$C.jsonl
done
