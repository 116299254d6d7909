# Round 2 (session 4): Euler-point couplings (P1 after / Q1 before a constant-|U00| one-qubit
# group instead of X, Y, Z components after it): GPU suite + cfg4/cfg3 A/B.
mkdir -p gpurun_out
T=${1:-r02n}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -8
for c in 4 3; do
  for v in off on; do
    env="LSQ_EULER_COUP=1"; [ $v = off ] && env="LSQ_EULER_COUP=0"
    env $env timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$v.err
    echo "cfg$c eulercoup=$v rc=$? $(python profiles/bench_brief.py < /tmp/b.json) gate=$(python -c "import json;d=json.load(open('/tmp/b.json'));g=d['parity_gate'];print('%.2e %.2e'%(g['grad_a2_rel_err'],g['zq_abs_err']))")"
    cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
  done
done
