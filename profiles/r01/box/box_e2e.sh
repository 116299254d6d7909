mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_e2e
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_e2e.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_e2e.log
python profiles/api_overhead.py 2>&1 | tail -40 > gpurun_out/api_overhead.log
head -3 gpurun_out/api_overhead.log; grep "ms/call" gpurun_out/api_overhead.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_e2e.log 2>&1; tail -1 gpurun_out/bench_e2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
