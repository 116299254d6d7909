# Round 2 (session 5): plans rebuilt with the measured pass-rebalancing budget, then the round-end
# artifacts (box_r02_final.sh) with those plans, all on one box.
mkdir -p gpurun_out/plans_final
export LSQ_CACHE_DIR=/tmp/lsq_jit_final2
timeout 2400 python profiles/build_plans.py 4 3 2 5 > gpurun_out/build_plans_r02final.log 2>&1; echo "build_plans rc=$?"; tail -5 gpurun_out/build_plans_r02final.log
cp profiles/plans/*.json gpurun_out/plans_final/
grep -H rebalance_budget profiles/plans/*.json
bash profiles/r02/box/box_r02_final.sh r02final
