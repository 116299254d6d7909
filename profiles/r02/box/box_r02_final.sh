# Round-2 artifacts in one call, in dependency order:
# 1. ncu --set full of one step of cfg3/cfg4/cfg5 (the benched plans) -> summaries and the
#    per-kernel-family DRAM traffic table bench.py reads (profiles/ncu_traffic.json);
# 2. executed-FP32 source counters of cfg2..cfg5 -> profiles/ncu_fp32.json (bench FP32 view);
# 3. the GPU suite with the parity log;
# 4. bench lines: default (cfg4 + CPU leg), the reference arm, cfg1/2/3/5;
# 5. the ncu launch list of the default bench command.
mkdir -p gpurun_out
T=${1:-r02final}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_$T.txt
passes() { python -c "
import sys,os; sys.path.insert(0,'.')
import warnings; warnings.simplefilter('ignore')
from paper_2506_04891_b200.configs import make_workload
from paper_2506_04891_b200.planner import load_plan, KernelKind
from paper_2506_04891_b200.core import plan_kernels
from paper_2506_04891_b200.schedule import compile_circuit
wl=make_workload($1, batch=1); p=load_plan('profiles/plans/cfg$1.json'); k=plan_kernels(wl.circuit,p)
s=lambda kk:[i for i,x in enumerate(k) if x is kk]
prog=compile_circuit(wl.circuit,M=p.tile_bits,R=4,isolate=s(KernelKind.ISOLATED),prefix=True,fold=True,split=True,direct=s(KernelKind.DIRECT),split_layers=s(KernelKind.SPLIT),rebalance_budget=p.rebalance_budget)
print(2*len(prog.passes)-1, p.tile_bits)"; }
for spec in "4 0 1 256" "3 0 1 128" "5 39 1 39"; do
  set -- $spec; C=$1; B=$2; SC=$3; ROWS=$4
  read K M <<< "$(passes $C)"
  timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:lsq_jit_p' -c $K -f -o /tmp/full_c${C} \
     python profiles/prof_step.py $C 1 $B > gpurun_out/ncu_full_c${C}_$T.log 2>&1; echo "ncu full cfg$C rc=$? K=$K M=$M"
  python profiles/ncu_summary.py /tmp/full_c${C}.ncu-rep --json gpurun_out/ncu_full_c${C}_$T.json > gpurun_out/ncu_full_c${C}_$T.txt 2>&1
  python profiles/ncu_traffic.py /tmp/full_c${C}.ncu-rep $(python -c "from paper_2506_04891_b200.configs import CONFIG_NAMES; print(CONFIG_NAMES[$C])") $M $SC $ROWS >> gpurun_out/ncu_traffic_$T.log 2>&1
done
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
rm -f gpurun_out/ncu_fp32.json
for spec in "2 512" "3 8" "4 8" "5 8"; do
  set -- $spec; C=$1; B=$2
  read K M <<< "$(passes $C)"
  python profiles/prof_step.py $C 1 $B > /dev/null 2>&1 || { echo "prof $C failed"; continue; }
  timeout 1500 ncu --section SourceCounters --metrics gpu__time_duration.sum --clock-control none \
      -k regex:lsq_jit -s $K -c $K -f -o /tmp/fp32_c$C python profiles/prof_step.py $C 2 $B \
      > gpurun_out/fp32_c${C}_$T.log 2>&1; echo "fp32 cfg$C ncu rc=$?"
  python profiles/ncu_fp32.py /tmp/fp32_c$C.ncu-rep ${C}_M${M}_R4 $B --json gpurun_out/ncu_fp32.json \
      > gpurun_out/fp32_table_c${C}_$T.txt 2>&1; tail -2 gpurun_out/fp32_table_c${C}_$T.txt
done
cp gpurun_out/ncu_fp32.json profiles/ncu_fp32.json
LSQ_PARITY_OUT=gpurun_out/parity_$T.json timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_$T.log 2>&1
echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu_$T.log | tail -5
timeout 1200 python bench.py > gpurun_out/bench_${T}_default.jsonl 2> gpurun_out/bench_${T}_default.err; echo "bench default rc=$?"
python profiles/bench_brief.py < gpurun_out/bench_${T}_default.jsonl
timeout 1800 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${T}_reference.jsonl 2> gpurun_out/bench_${T}_reference.err; echo "reference rc=$?"
cut -c1-400 gpurun_out/bench_${T}_reference.jsonl
for C in 1 2 3 5; do
  st=10; [ $C = 5 ] && st=3
  timeout 1500 python bench.py --config $C --steps $st --no-cpu > gpurun_out/bench_${T}_c$C.jsonl 2> gpurun_out/bench_${T}_c$C.err; echo "cfg$C rc=$?"
  python profiles/bench_brief.py < gpurun_out/bench_${T}_c$C.jsonl
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv --log-file gpurun_out/launches_${T}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_${T}.log 2>&1; echo "ncu launch rc=$?"
python profiles/launch_table.py gpurun_out/launches_${T}.csv > gpurun_out/launches_${T}.txt 2>&1; head -12 gpurun_out/launches_${T}.txt
du -sh gpurun_out
