# Round 2 (session 5): all-gate random stress at wider states: n = 12..15, M = 9..13, 2 seeds x 60 cases.
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_r02ae
for s in 41 42; do
  timeout 2400 python profiles/stress_random.py 60 $s 12 16 9 > gpurun_out/stress_random_wide_r02ae_s$s.txt 2>&1; echo "wide random stress seed $s rc=$? $(tail -1 gpurun_out/stress_random_wide_r02ae_s$s.txt)"
  grep FAIL gpurun_out/stress_random_wide_r02ae_s$s.txt | head
done
true
