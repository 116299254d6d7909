# Round artifacts (session 2): full GPU suite, default bench line (planner tile choice + CPU leg),
# reference arm, ncu launch list of the same bench command, bench lines for cfg1/3/4/5.
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_final2
T=${1:-final2}
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_$T.log
timeout 900 python bench.py > gpurun_out/bench_${T}_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_${T}_default.log | python profiles/bench_brief.py
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${T}_reference.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_${T}_reference.log | cut -c1-200
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/launches_${T}.csv \
    python bench.py --steps 2 --warmup 1 --M 11 > gpurun_out/ncu_launch_${T}.log 2>&1; echo "ncu launch rc=$?"  # --M: the planner would time M differently under ncu
python profiles/launch_table.py gpurun_out/launches_${T}.csv > gpurun_out/launches_${T}.txt 2>&1; head -8 gpurun_out/launches_${T}.txt
for C in 1 3 4 5; do
  timeout 1500 python bench.py --config $C --no-cpu > gpurun_out/bench_${T}_c$C.log 2>&1; echo "cfg$C rc=$?"; tail -1 gpurun_out/bench_${T}_c$C.log | python profiles/bench_brief.py
done
