# three-way: default, $AB_B, $AB_C (short bench lines, cfg2 + n>=20 configs)
export LSQ_CACHE_DIR=/tmp/lsq_jit_iter
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_ab3.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_ab3.log
run() { timeout 600 python bench.py --no-cpu "$@" 2>/dev/null | tail -1 | python profiles/bench_brief.py; }
for c in "2 --M 11" "3 --M 12 --steps 5" "4 --M 12 --batch 64 --steps 5" "5 --M 12 --batch 39 --steps 3"; do
  echo "A"; run --config $c; echo "B ($AB_B)"; env $AB_B bash -c "$(declare -f run); run --config $c"
  echo "C ($AB_C)"; env $AB_C bash -c "$(declare -f run); run --config $c"; done
