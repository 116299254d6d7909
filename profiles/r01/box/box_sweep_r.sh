export LSQ_CACHE_DIR=/tmp/lsq_jit_sw
run() { timeout 600 python bench.py --no-cpu "$@" 2>/dev/null | tail -1 | python profiles/bench_brief.py; }
for MR in "11 4" "11 3" "10 3" "12 3" "10 4" "12 4"; do set -- $MR; echo "M=$1 R=$2"; run --config 2 --M $1 --R $2; done
for MR in "12 3" "11 3" "13 3"; do set -- $MR; echo "cfg5 M=$1 R=$2"; run --config 5 --M $1 --R $2 --batch 39 --steps 3; done
for MR in "12 3"; do set -- $MR; echo "cfg3 M=$1 R=$2"; run --config 3 --M $1 --R $2 --steps 5; done
