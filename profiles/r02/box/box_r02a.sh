# Round 2, first box call: GPU parity suite (exact A2 floor, parity log), bench lines for
# cfg3/cfg4/cfg5, and one `ncu --set full` capture of every pass kernel of one step of
# cfg3, cfg4 and cfg5 (one 39-row chunk).
mkdir -p gpurun_out
T=${1:-r02a}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$T.txt
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1500 python -m pytest tests -m gpu -q -x -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_$T.log
for c in 4 3 5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu >> gpurun_out/bench_$T.jsonl 2> gpurun_out/bench_${T}_c$c.err
  echo "bench cfg$c rc=$?"
done
python profiles/bench_brief.py < gpurun_out/bench_$T.jsonl
for spec in "3 1 0" "4 1 0" "5 1 39"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:lsq_jit_p' -c 60 -f -o gpurun_out/full_c$1_$T \
     python profiles/prof_step.py $1 $2 $3 > gpurun_out/ncu_full_c$1_$T.log 2>&1; echo "ncu cfg$1 rc=$?"
  python profiles/ncu_summary.py gpurun_out/full_c$1_$T.ncu-rep --json gpurun_out/ncu_full_c$1_$T.json > gpurun_out/ncu_full_c$1_$T.txt 2>&1
done
