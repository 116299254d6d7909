# Round 2: source-level ncu of the cfg4 kernels (SASS view, per-instruction shared-memory
# wavefronts and stalls), then the compute-sanitizer pass.
mkdir -p gpurun_out
T=${1:-r02e}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
python profiles/prof_step.py 4 1 0 12 > gpurun_out/prof_$T.log 2>&1
for k in p1_m0 p5_m0 p0_m2 p1_m2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lsq_jit_${k}\$ -c 1 -f -o /tmp/src_$k \
     python profiles/prof_step.py 4 1 0 12 > gpurun_out/ncu_src_${k}_$T.log 2>&1; echo "ncu $k rc=$?"
  ncu -i /tmp/src_$k.ncu-rep --page source --csv --print-source sass > /tmp/src_$k.csv 2>/dev/null
  gzip -c /tmp/src_$k.csv > gpurun_out/ncu_src_${k}_$T.csv.gz
done
bash profiles/box_sanitize.sh $T
du -sh gpurun_out
