# Round 2 (session 5): structured stress at BASELINE-like kernel shapes: n = 14..17, M = 10..12 (256-thread
# tiles, several tiles per row, stage prefetch, rotating buffers), 2 seeds x 60 cases.
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_r02ad
for s in 31 32; do
  timeout 2400 python profiles/stress_structured.py 60 $s 14 18 10 13 > gpurun_out/stress_wide_r02ad_s$s.txt 2>&1; echo "wide stress seed $s rc=$? $(tail -1 gpurun_out/stress_wide_r02ad_s$s.txt)"
  grep FAIL gpurun_out/stress_wide_r02ad_s$s.txt | head
done
true
