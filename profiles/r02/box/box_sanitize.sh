# compute-sanitizer over every kernel mode of the specialised pass kernels at small n
# (profiles/sanitize_step.py): racecheck (shared-memory hazards), synccheck (barrier
# misuse), memcheck (out-of-bounds / misaligned), initcheck (uninitialised global reads).
mkdir -p gpurun_out
T=${1:-san}
export LSQ_CACHE_DIR=/tmp/lsq_jit_$T
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python profiles/sanitize_step.py > gpurun_out/sanitize_${tool}_$T.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_${tool}_$T.log
done
