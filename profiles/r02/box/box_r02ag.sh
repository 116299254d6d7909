# Round 2 (session 5): the reference arm launched the way the driver launches it for N > 1 (torchrun, two
# ranks): rank 0 alone runs and prints the line, rank 1 exits 0 without work.
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > gpurun_out/bench_reference_torchrun2.jsonl 2> gpurun_out/bench_reference_torchrun2.err
echo "rc=$?"; wc -l gpurun_out/bench_reference_torchrun2.jsonl; cut -c1-300 gpurun_out/bench_reference_torchrun2.jsonl; tail -3 gpurun_out/bench_reference_torchrun2.err
