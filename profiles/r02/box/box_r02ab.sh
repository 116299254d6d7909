# Round 2 (session 5): all-gates random stress again after the observable-folding fix (8 seeds), the
# structured stress once more (2 seeds), then the GPU suite (round-end log).
mkdir -p gpurun_out
T=${1:-r02ab}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
for s in 0 1 2 3 4 5 6 7; do
  timeout 1500 python profiles/stress_random.py 100 $s > gpurun_out/stress_random_${T}_s$s.txt 2>&1; echo "random stress seed $s rc=$? $(tail -1 gpurun_out/stress_random_${T}_s$s.txt)"
  grep FAIL gpurun_out/stress_random_${T}_s$s.txt | head -5
done
for s in 21 22; do
  timeout 1200 python profiles/stress_structured.py 100 $s > gpurun_out/stress_${T}_s$s.txt 2>&1; echo "structured stress seed $s rc=$? $(tail -1 gpurun_out/stress_${T}_s$s.txt)"
done
LSQ_PARITY_OUT=gpurun_out/parity_r02final.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_r02final.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_r02final.log | tail -5
true
