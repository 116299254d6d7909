# Round 2 (session 5): HEAD sanity: build(), the default bench line and the cfg3 / cfg2 lines once more.
mkdir -p gpurun_out
export LSQ_CACHE_DIR=/tmp/lsq_jit_final5
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_final5.log 2>&1; echo "build rc=$?"
timeout 1500 python bench.py > gpurun_out/bench_head_default.jsonl 2> gpurun_out/bench_head_default.err; echo "bench default rc=$?"
python profiles/bench_brief.py < gpurun_out/bench_head_default.jsonl
for C in 3 2; do
  timeout 900 python bench.py --config $C --no-cpu > gpurun_out/bench_head_c$C.jsonl 2> gpurun_out/bench_head_c$C.err; echo "cfg$C rc=$?"
  python profiles/bench_brief.py < gpurun_out/bench_head_c$C.jsonl
done
