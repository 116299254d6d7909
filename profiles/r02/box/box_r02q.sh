# Round 2 (session 5): merged Euler diagonals (LSQ_EULER_MERGE = minimum run length, 0 = off) A/B on
# cfg4 / cfg3, the GPU suite with it on, the on-chip exchange bandwidth microbenchmark, and the
# bench under torchrun with one rank (the NCCL init / all-reduce path of the scaling run).
mkdir -p gpurun_out
T=${1:-r02q}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
./profiles/micro/onchip_bw > gpurun_out/onchip_bw_$T.txt 2>&1; echo "onchip_bw rc=$?"; cat gpurun_out/onchip_bw_$T.txt
run() { # cfg label env...
  c=$1; lab=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > /tmp/b.json 2> gpurun_out/bench_${T}_c${c}_$lab.err
  echo "cfg$c $lab rc=$? $(python profiles/bench_brief.py < /tmp/b.json)"
  cat /tmp/b.json >> gpurun_out/bench_$T.jsonl
}
for c in 4 3; do
  run $c merge0 LSQ_EULER_MERGE=0
  run $c merge2 LSQ_EULER_MERGE=2
  run $c merge3 LSQ_EULER_MERGE=3
done
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA -x > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -5
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_${T}_torchrun1.jsonl 2> gpurun_out/bench_${T}_torchrun1.err
echo "torchrun rc=$?"; python profiles/bench_brief.py < gpurun_out/bench_${T}_torchrun1.jsonl; tail -3 gpurun_out/bench_${T}_torchrun1.err
