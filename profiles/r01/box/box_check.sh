# GPU check: parity tests, then short bench lines per config (no CPU baseline).
# usage: bash profiles/box_check.sh [TAG] [CFGS]   (CFGS default "2 1 3 4")
mkdir -p gpurun_out
TAG=${1:-chk}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$TAG
python -c "from paper_2506_04891_b200 import _native; _native.lib(); print('nvrtc', _native.jit_compiler())"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
for C in ${2:-2 1 3 4}; do
  timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_c$C.log 2>&1
  tail -1 gpurun_out/bench_${TAG}_c$C.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('cfg$C', round(d['value']), 'evals/s', round(d['ms_per_step'],3), 'ms', 'frac', d['roofline']['frac'], 'e2e', round(d['e2e']['value']))
except Exception as e: print('cfg$C failed', e)"
done
