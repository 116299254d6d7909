# COAL (low physical bits always inside a tile) sweep on cfg2 and cfg5
export LSQ_CACHE_DIR=/tmp/lsq_jit_coal
run() { timeout 600 python bench.py --no-cpu "$@" 2>/dev/null | tail -1 | python profiles/bench_brief.py; }
for C in 4 3 5; do echo "COAL=$C"; LSQ_COAL=$C bash -c "$(declare -f run); run --config 2 --M 11; run --config 2 --M 12; run --config 5 --M 12 --batch 39 --steps 3"; done
