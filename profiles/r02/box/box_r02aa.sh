# Round 2 (session 5): GPU stress over random circuits of all 17 gate kinds (profiles/stress_random.py).
mkdir -p gpurun_out
T=${1:-r02aa}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
for s in 0 1 2 3; do
  timeout 1500 python profiles/stress_random.py 100 $s > gpurun_out/stress_random_${T}_s$s.txt 2>&1; echo "random stress seed $s rc=$? $(tail -1 gpurun_out/stress_random_${T}_s$s.txt)"
  grep FAIL gpurun_out/stress_random_${T}_s$s.txt | head -5
done
true
