# Executed-FP32 capture for bench.py's FP32 view: one step's pass kernels per config under
# ncu source counters (small batches; flops per row do not depend on the batch), reduced on
# the box to gpurun_out/ncu_fp32.json; plus one ncu --set full capture of a cfg2 step.
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_fp32
T=${1:-fp32}
for spec in "2 512 11 11" "3 8 12 7" "4 8 12 19" "5 8 12 31"; do
  set -- $spec; C=$1; B=$2; M=$3; K=$4
  python profiles/prof_step.py $C 1 $B $M 4 > /dev/null 2>&1 || { echo "prof $C failed"; continue; }
  timeout 1200 ncu --section SourceCounters --metrics gpu__time_duration.sum --clock-control none \
      -k regex:lsq_jit -s $K -c $K -f -o /tmp/${T}_c$C python profiles/prof_step.py $C 2 $B $M 4 \
      > gpurun_out/${T}_c$C.log 2>&1; echo "cfg$C ncu rc=$?"
  python profiles/ncu_fp32.py /tmp/${T}_c$C.ncu-rep ${C}_M${M}_R4 $B --json gpurun_out/ncu_fp32.json \
      > gpurun_out/${T}_fp32_c$C.txt 2>&1; tail -3 gpurun_out/${T}_fp32_c$C.txt
done
python profiles/prof_step.py 2 2 0 11 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lsq_jit -s 11 -c 11 -f -o gpurun_out/${T}_full_c2 \
    python profiles/prof_step.py 2 2 0 11 4 > gpurun_out/${T}_full_c2.log 2>&1; echo "ncu full rc=$?"
python profiles/ncu_summary.py gpurun_out/${T}_full_c2.ncu-rep --json gpurun_out/${T}_full_c2.json > /dev/null 2>&1
ls -la gpurun_out | tail -5
