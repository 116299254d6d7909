# Round 2: forward kernels with 2^5 amplitudes per thread (own phase plan, same partition):
# GPU suite, then A/B of LSQ_R_FWD (0 = the program's R=4) and the forward register budget.
mkdir -p gpurun_out
T=${1:-r02i}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -8
for c in 4 3; do
  for ab in "0 4" "5 4" "5 3" "5 5"; do
    set -- $ab
    LSQ_R_FWD=$1 LSQ_MINB_FWD5=$2 timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_r$1_m$2.err
    echo "cfg$c r_fwd=$1 minb5=$2 rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
  done
done
for r in 0 5; do
  LSQ_R_FWD=$r timeout 900 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c5_r$r.err
  echo "cfg5 r_fwd=$r rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
  LSQ_R_FWD=$r timeout 900 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c2_r$r.err
  echo "cfg2 r_fwd=$r rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"; cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
done
