# Round 2 (session 5): the round-end GPU suite (deep-circuit test at six blocks) and smoke().
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_final4
LSQ_PARITY_OUT=gpurun_out/parity_r02final.json timeout 1800 python -m pytest tests -m gpu -q -rA --durations=8 > gpurun_out/pytest_gpu_r02final.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_r02final.log | tail -5; grep -A9 "slowest" gpurun_out/pytest_gpu_r02final.log | head -12
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
timeout 600 python profiles/stress_structured.py 100 21 > gpurun_out/stress_r02final4_s21.txt 2>&1; echo "structured stress seed 21 rc=$? $(tail -1 gpurun_out/stress_r02final4_s21.txt)"
