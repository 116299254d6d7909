mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_final2
T=r1f
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node -c 40000 --csv --log-file gpurun_out/launches_${T}.csv \
    python bench.py --steps 2 --warmup 1 --M 11 > gpurun_out/ncu_launch_${T}.log 2>&1; echo "ncu launch rc=$?"
python profiles/launch_table.py gpurun_out/launches_${T}.csv > gpurun_out/launches_${T}.txt 2>&1; head -14 gpurun_out/launches_${T}.txt; wc -l gpurun_out/launches_${T}.csv
