# Round 2 (session 5): which code-generation feature carries the extra noise of the four marginal cases
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_r02ac
timeout 1500 python profiles/marginal_cases.py > gpurun_out/marginal_cases_r02ac.txt 2>&1; echo "rc=$?"; cat gpurun_out/marginal_cases_r02ac.txt | cut -c1-200
