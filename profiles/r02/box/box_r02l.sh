# Round 2: phase accuracy micro-benchmark; MUFU-after-exact-reduction phases: GPU suite + cfg5/cfg2 bench.
mkdir -p gpurun_out
T=${1:-r02l}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
./profiles/micro/phase_acc | tee gpurun_out/phase_acc_$T.txt
LSQ_MUFU_REDUCED=1 LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest (mufu reduced) rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -8
for c in 5 2; do
  for v in default mufured; do
    st=2; [ $c = 2 ] && st=10
    env=""; [ $v = mufured ] && env="LSQ_MUFU_REDUCED=1"
    env $env timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$v.err
    echo "cfg$c phase=$v rc=$? $(python profiles/bench_brief.py < /tmp/b.json) gate=$(python -c "import json;d=json.load(open('/tmp/b.json'));g=d['parity_gate'];print('%.2e %.2e'%(g['grad_a2_rel_err'],g['zq_abs_err']))")"
    cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
  done
done
