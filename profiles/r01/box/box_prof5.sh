# cfg5 (n=24) kernel profile: FFMA/FFMA2 issue-rate microbenchmark, then one ncu --set full
# capture of a light and a heavy pass in forward and adjoint mode (8 rows per launch).
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_prof5
T=${1:-p5}
./profiles/micro/ffma2_rate > gpurun_out/micro_$T.log 2>&1; cat gpurun_out/micro_$T.log
python profiles/prof_step.py 5 2 8 > gpurun_out/prof5_$T.log 2>&1 || { echo prof failed; tail gpurun_out/prof5_$T.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:lsq_jit_p[23]_m[02]' -s 4 -c 4 -f -o gpurun_out/full5_$T \
    python profiles/prof_step.py 5 2 8 > gpurun_out/ncu_full5_$T.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_full5_$T.log
