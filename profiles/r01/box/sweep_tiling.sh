#!/bin/bash
# Tile-bits / register-bits sweep of the default workload (cfg2) -- numbers for DESIGN.md.
CFG=${1:-2}
IFS=, read -ra LIST <<< "${MRS:-13 5,13 4,12 4,11 4,11 3,10 5,9 4,10 4}"
for MR in "${LIST[@]}"; do
  set -- $MR
  LOG=gpurun_out/sweep_c${CFG}_M$1_R$2_coal${LSQ_COAL:-4}.log
  python bench.py --config $CFG --steps ${STEPS:-5} --warmup 3 --no-cpu --M $1 --R $2 ${BATCH:+--batch $BATCH} > $LOG 2>&1
  python - "$1" "$2" "$LOG" <<'PY'
import json, sys
M, R, f = sys.argv[1:]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    pk = d["roofline"]["per_kernel"]
    print(f"coal={__import__('os').environ.get('LSQ_COAL','4')} M={M} R={R} evals/s={d['value']:.0f} ms/step={d['ms_per_step']:.3f} passes={d['config']['passes']} " +
          " ".join(f"{k.split(' ')[0].split('_')[-1]}:{v['GBps']}GB/s,{v['ms_per_step']:.2f}ms" for k, v in pk.items()))
except Exception as e:
    print(f"M={M} R={R} failed: {e}"); print(open(f).read()[-800:])
PY
done
