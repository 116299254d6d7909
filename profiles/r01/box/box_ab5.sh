# cfg5-only three-way A/B: default, $AB_B, $AB_C
export LSQ_CACHE_DIR=/tmp/lsq_jit_iter
run() { timeout 600 python bench.py --no-cpu "$@" 2>/dev/null | tail -1 | python profiles/bench_brief.py; }
c="5 --M 12 --batch 39 --steps 3"
echo "A"; run --config $c; echo "B ($AB_B)"; env $AB_B bash -c "$(declare -f run); run --config $c"
echo "C ($AB_C)"; env $AB_C bash -c "$(declare -f run); run --config $c"
echo "A again"; run --config $c
