mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_prof2
python profiles/prof_step.py 5 1 32 > gpurun_out/prof5.log 2>&1 || { cat gpurun_out/prof5.log; exit 1; }
python profiles/prof_step.py 4 1 32 > gpurun_out/prof4.log 2>&1 || { cat gpurun_out/prof4.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"lsq_jit_p(0|7|8)_m(1|2)" -c 6 -f -o gpurun_out/full_cfg5 \
    python profiles/prof_step.py 5 1 32 > gpurun_out/ncu5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"lsq_jit_p(4|5)_m(0|2)" -c 4 -f -o gpurun_out/full_cfg4 \
    python profiles/prof_step.py 4 1 32 > gpurun_out/ncu4.log 2>&1
tail -2 gpurun_out/ncu5.log gpurun_out/ncu4.log
