"""Profiling driver: a few fwd+bwd steps of a BASELINE config through the engine (used
under ncu; never a bench number).  usage: prof_step.py CFG STEPS [BATCH] [M] [R]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_04891_b200.configs import make_workload
from paper_2506_04891_b200.engine import Engine

a = sys.argv[1:] + [None] * 5
cfg = int(a[0] or 2); steps = int(a[1] or 3)
batch = int(a[2]) if a[2] not in (None, "0") else None
M = int(a[3]) if a[3] else None; R = int(a[4]) if a[4] else None
wl = make_workload(cfg, batch=batch)
# the program bench.py times: its saved per-layer plan when one exists and no M is forced
plan_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plans", f"cfg{cfg}.json")
kw = {}
if M is None and os.path.exists(plan_path):
    import warnings

    from paper_2506_04891_b200.core import plan_kernels
    from paper_2506_04891_b200.planner import KernelKind, load_plan

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        plan = load_plan(plan_path)
    kinds = plan_kernels(wl.circuit, plan)
    sel = lambda kk: [i for i, k in enumerate(kinds) if k is kk]  # noqa: E731
    M = plan.tile_bits
    kw = dict(isolate=sel(KernelKind.ISOLATED), direct=sel(KernelKind.DIRECT), split_layers=sel(KernelKind.SPLIT),
              rebalance_budget=plan.rebalance_budget)
eng = Engine(wl.circuit, M=M, R=R, **kw)
th = torch.as_tensor(wl.theta, device="cuda"); x = torch.as_tensor(wl.x, device="cuda")
w = torch.as_tensor(wl.weights, device="cuda")
bufs = None
for _ in range(steps):
    r = eng.fwd_bwd(th, x, batch=wl.batch, weights=w, rows=False, encoding_grads=False, buffers=bufs)
    bufs = r["buffers"]
torch.cuda.synchronize()
print("ok", len(eng.program.passes), "passes")
