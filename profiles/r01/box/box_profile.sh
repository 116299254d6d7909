# Launch list of the bench command + one full ncu capture of a cfg2 step (12.9 NVRTC cubins).
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_prof
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/b.log 2>&1 || { echo bench failed; tail gpurun_out/b.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
python profiles/prof_step.py 2 2 > gpurun_out/prof.log 2>&1 || { echo prof failed; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:lsq_jit -s 12 -c 12 -f -o gpurun_out/full_cfg2 \
    python profiles/prof_step.py 2 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
