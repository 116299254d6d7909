# Round 2: GPU parity suite + A/B of the swizzled prefetch stage and the Euler tangent form
# (bench lines at M=12), then ncu --set full of one cfg4 step with both on.
mkdir -p gpurun_out
T=${1:-r02c}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -15
for c in 4 3; do
  for ab in "0 0" "1 0" "1 1"; do
    set -- $ab
    LSQ_STAGE_SWZ=$1 LSQ_EULER_TAN=$2 timeout 600 python bench.py --config $c --M 12 --steps 5 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$1$2.err
    echo "cfg$c swz=$1 euler=$2 rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_ab_$T.jsonl
  done
done
timeout 900 python bench.py --config 5 --M 12 --steps 2 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c5.err
echo "cfg5 rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_ab_$T.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:lsq_jit_p' -c 60 -f -o /tmp/full_c4_$T \
   python profiles/prof_step.py 4 1 0 12 > gpurun_out/ncu_full_c4_$T.log 2>&1; echo "ncu cfg4 rc=$?"
python profiles/ncu_summary.py /tmp/full_c4_$T.ncu-rep --json gpurun_out/ncu_full_c4_$T.json > gpurun_out/ncu_full_c4_$T.txt 2>&1
du -sh gpurun_out
