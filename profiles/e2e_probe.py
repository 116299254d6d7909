"""Where the e2e time goes (box only, never a bench number): device time of the full-output
step graph vs run_host vs the public gradient() call. usage: e2e_probe.py [CFG]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2506_04891_b200 import gradient
from paper_2506_04891_b200.configs import make_workload
from paper_2506_04891_b200.core import _engine
from paper_2506_04891_b200.planner import plan_for_tile_bits

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = make_workload(cfg)
dev = torch.device("cuda", 0)
M = {2: 11}.get(cfg, 12)
plan = plan_for_tile_bits(wl.circuit, wl.batch, M)
res = gradient(wl.circuit, wl.theta, wl.x, batch=wl.batch, weights=wl.weights, device=dev, plan=plan)
eng = _engine(wl.circuit, plan, dev)
step = list(eng._steps.values())[0]
K = 20
for rows, eg in ((False, False), (True, False), (True, True)):
    s = eng.make_step(wl.batch, rows=rows, encoding_grads=eg)
    s.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        s.graph.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"graph replay rows={rows} egrads={eg}: {e0.elapsed_time(e1) / K:.3f} ms")
t0 = time.perf_counter()
for _ in range(K):
    step.run_host(wl.theta, wl.x, wl.weights)
print(f"run_host: {(time.perf_counter() - t0) / K * 1e3:.3f} ms")
t0 = time.perf_counter()
for _ in range(K):
    gradient(wl.circuit, wl.theta, wl.x, batch=wl.batch, weights=wl.weights, device=dev, plan=plan)
print(f"gradient(): {(time.perf_counter() - t0) / K * 1e3:.3f} ms")
if "--prof" in sys.argv:
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as p:
        for _ in range(3):
            gradient(wl.circuit, wl.theta, wl.x, batch=wl.batch, weights=wl.weights, device=dev, plan=plan)
    print(p.key_averages().table(sort_by="cuda_time_total", row_limit=15))
