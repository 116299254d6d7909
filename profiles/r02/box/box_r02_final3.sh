# Round 2 (session 5): the GPU suite with the plan-budget tests added after the artifact run, and the
# cfg5 bench line again (ncu traffic scaled to the bench's rows per launch).
mkdir -p gpurun_out
T=r02final
export LSQ_CACHE_DIR=/tmp/lsq_jit_final3
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -5
timeout 1500 python bench.py --config 5 --steps 3 --no-cpu > gpurun_out/bench_${T}_c5.jsonl 2> gpurun_out/bench_${T}_c5.err; echo "cfg5 rc=$?"
python profiles/bench_brief.py < gpurun_out/bench_${T}_c5.jsonl
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
