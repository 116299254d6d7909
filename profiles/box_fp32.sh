# Executed-FP32 capture for bench.py's FP32 view: one step's pass kernels per config under
# ncu source counters (small batches; flops per row do not depend on the batch).
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_fp32
T=${1:-fp32}
for spec in "2 512 11 11" "3 8 12 7" "4 8 12 19" "5 8 12 31"; do
  set -- $spec; C=$1; B=$2; M=$3; K=$4
  python profiles/prof_step.py $C 1 $B $M 4 > /dev/null 2>&1 || { echo "prof $C failed"; continue; }
  timeout 1200 ncu --section SourceCounters --metrics gpu__time_duration.sum --clock-control none \
      -k regex:lsq_jit -s $K -c $K -f -o gpurun_out/${T}_c$C python profiles/prof_step.py $C 2 $B $M 4 \
      > gpurun_out/${T}_c$C.log 2>&1; echo "cfg$C ncu rc=$?"
done
