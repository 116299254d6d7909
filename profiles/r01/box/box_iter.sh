# Iteration loop on the box: GPU parity subset, then short bench lines per config
# (fixed tile size, no CPU leg) summarised per kernel family.
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_iter
T=${1:-it}
# PYEXPR: pytest -k expression ("all" = the whole GPU suite)
PYEXPR=${PYEXPR:-small_configs or cfg1_full or full_width or random_circuits or checkpoint or bit_exact or prefix}
if [ "$PYEXPR" = all ]; then PYK=(); else PYK=(-k "$PYEXPR"); fi
timeout 900 python -m pytest tests -q -m gpu -x "${PYK[@]}" > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$T.log
run() { timeout 600 python bench.py --no-cpu "$@" 2>/dev/null | tail -1 | python profiles/bench_brief.py; }
run --config 2 --M 11
[ -z "$QUICK" ] && run --config 3 --M 12 --steps 5
[ -z "$QUICK" ] && run --config 4 --M 12 --batch 64 --steps 5
[ -z "$QUICK" ] && run --config 5 --M 12 --batch 39 --steps 3
true
