# A/B repeated: default build vs $AB_OFF, alternating, cfg2 three times each + one line per
# other config (no pytest).
export LSQ_CACHE_DIR=/tmp/lsq_jit_iter
run() { timeout 600 python bench.py --no-cpu "$@" 2>/dev/null | tail -1 | python profiles/bench_brief.py; }
for i in 1 2 3; do echo "new"; run --config 2 --M 11; echo "base"; env $AB_OFF bash -c "$(declare -f run); run --config 2 --M 11"; done
for c in "3 --M 12 --steps 5" "4 --M 12 --batch 64 --steps 5" "5 --M 12 --batch 39 --steps 3"; do
  echo "new"; run --config $c; echo "base"; env $AB_OFF bash -c "$(declare -f run); run --config $c"; done
