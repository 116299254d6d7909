# Round 2: GPU parity suite without -x (full parity log), then ncu --set full of one step's
# pass kernels for cfg3/cfg4/cfg5; reports stay in /tmp, only summaries come back.
mkdir -p gpurun_out
T=${1:-r02b}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
nproc > gpurun_out/host_$T.txt; free -g >> gpurun_out/host_$T.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host_$T.txt
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -15
for spec in "4 1 0" "3 1 0" "5 1 39"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:lsq_jit_p' -c 60 -f -o /tmp/full_c$1_$T \
     python profiles/prof_step.py $1 $2 $3 > gpurun_out/ncu_full_c$1_$T.log 2>&1; echo "ncu cfg$1 rc=$?"
  python profiles/ncu_summary.py /tmp/full_c$1_$T.ncu-rep --json gpurun_out/ncu_full_c$1_$T.json > gpurun_out/ncu_full_c$1_$T.txt 2>&1
  ncu -i /tmp/full_c$1_$T.ncu-rep --page raw --csv > /tmp/raw_c$1.csv 2>/dev/null; gzip -c /tmp/raw_c$1.csv > gpurun_out/ncu_raw_c$1_$T.csv.gz
done
du -sh gpurun_out
