# Round artifacts: GPU tests, bench lines, reference arm, ncu launch list + one full capture.
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_final
T=${1:-final}
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$T.log
timeout 900 python bench.py > gpurun_out/bench_${T}_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${T}_default.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${T}_reference.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_${T}_reference.log | cut -c1-300
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_${T}.csv \
    python bench.py > gpurun_out/ncu_launch_${T}.log 2>&1; echo "ncu launch rc=$?"
M=$(tail -1 gpurun_out/bench_${T}_default.log | python -c "import json,sys; print(json.loads(sys.stdin.read())['config']['tile_bits'])")
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lsq_jit -s 24 -c 12 -f -o gpurun_out/full_${T}_cfg2 \
    python profiles/prof_step.py 2 3 0 $M > gpurun_out/ncu_full_${T}.log 2>&1; echo "ncu full rc=$? M=$M"
for C in 1 3 4 5; do
  timeout 1200 python bench.py --config $C --no-cpu > gpurun_out/bench_${T}_c$C.log 2>&1; echo "cfg$C rc=$?"; tail -1 gpurun_out/bench_${T}_c$C.log | cut -c1-200
done
