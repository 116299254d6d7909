# cfg2 (n=16, default bench workload) full ncu capture of one step's pass kernels + the
# packed-FP32 pattern microbenchmark.
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_prof2
T=${1:-p2}
./profiles/micro/u1_rate > gpurun_out/u1rate_$T.log 2>&1; cat gpurun_out/u1rate_$T.log
python profiles/prof_step.py 2 2 0 11 > gpurun_out/prof2_$T.log 2>&1 || { echo prof failed; tail gpurun_out/prof2_$T.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lsq_jit -s 12 -c 12 -f -o gpurun_out/full2_$T \
    python profiles/prof_step.py 2 2 0 11 > gpurun_out/ncu_full2_$T.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu_full2_$T.log
