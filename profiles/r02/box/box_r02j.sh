# Round 2: accurate (sincospi) vs MUFU diagonal-run phases: GPU suite with the accurate ones,
# then bench A/B on every config (forward kernels at 2^5 amplitudes per thread).
mkdir -p gpurun_out
T=${1:-r02j}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -8
for c in 2 4 3 5; do
  for fp in 0 1; do
    st=5; [ $c = 5 ] && st=2; [ $c = 2 ] && st=10
    LSQ_FAST_PHASE=$fp timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_fp$fp.err
    echo "cfg$c fast_phase=$fp rc=$? $(python profiles/bench_brief.py < /tmp/b.json) gate=$(python -c "import json;d=json.load(open('/tmp/b.json'));g=d['parity_gate'];print('%.2e %.2e'%(g['grad_a2_rel_err'],g['zq_abs_err']))")"
    cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
  done
done
