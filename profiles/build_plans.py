"""Build the per-layer CUDA-variant plans of the BASELINE configs on the GPU box (reference
protocol: planner.build_plan, Objective.FORWARD_BACKWARD, CUDA-event timing) and save them as
plan JSON under profiles/plans/, where bench.py replays them.
usage: python profiles/build_plans.py [CFG ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04891_b200.configs import CONFIG_SHAPES, make_workload  # noqa: E402
from paper_2506_04891_b200.planner import Objective, build_plan, save_plan  # noqa: E402

out_dir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plans")
os.makedirs(out_dir, exist_ok=True)
for cfg in [int(a) for a in sys.argv[1:]] or [4, 3, 2, 5]:
    n, B = CONFIG_SHAPES[cfg]
    rows = max(1, min(B, (2 << 30) // (16 << n)))  # <= 2 GiB of psi + lambda per timing
    wl = make_workload(cfg, batch=1)
    t0 = time.time()
    plan = build_plan(wl.circuit, rows, Objective.FORWARD_BACKWARD, reps=3, warmup=2)
    path = os.path.join(out_dir, f"cfg{cfg}.json")
    save_plan(plan, path)
    kinds = {}
    for k in plan.assignments:
        kinds[k.value] = kinds.get(k.value, 0) + 1
    print(f"cfg{cfg}: M={plan.tile_bits} rebalance_budget={plan.rebalance_budget} {kinds} on {rows} rows in {time.time() - t0:.0f} s -> {path}", flush=True)
