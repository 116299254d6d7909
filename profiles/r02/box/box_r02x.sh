# Round 2 (session 5): GPU stress of the compiler searches / Euler-form kernels on randomised
# hardware-style circuits against the oracle (profiles/stress_structured.py).
mkdir -p gpurun_out
T=${1:-r02x}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
timeout 2400 python profiles/stress_structured.py 50 11 > gpurun_out/stress_$T.txt 2>&1; echo "stress rc=$?"
tail -4 gpurun_out/stress_$T.txt; grep -c FAIL gpurun_out/stress_$T.txt
