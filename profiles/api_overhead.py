"""Host-side overhead of the public gradient() call (cfg2): wall time per stage."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_04891_b200 import gradient
from paper_2506_04891_b200.configs import make_workload
from paper_2506_04891_b200.engine import engine_for
wl = make_workload(2)
for _ in range(3):
    r = gradient(wl.circuit, wl.theta, wl.x, batch=512, weights=wl.weights)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    r = gradient(wl.circuit, wl.theta, wl.x, batch=512, weights=wl.weights)
torch.cuda.synchronize()
print("gradient() ms/call", (time.perf_counter() - t) * 100)
eng = engine_for(wl.circuit)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(10):
    r = gradient(wl.circuit, wl.theta, wl.x, batch=512, weights=wl.weights)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
th = torch.as_tensor(wl.theta, device="cuda"); x = torch.as_tensor(wl.x, device="cuda"); w = torch.as_tensor(wl.weights, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10):
    d = eng.fwd_bwd(th, x, batch=512, weights=w)
torch.cuda.synchronize()
print("engine.fwd_bwd (device inputs, rows) ms/call", (time.perf_counter() - t) * 100)
t = time.perf_counter()
for _ in range(10):
    d = eng.fwd_bwd(th, x, batch=512, weights=w, rows=False, encoding_grads=False)
torch.cuda.synchronize()
print("engine.fwd_bwd (device inputs, no rows) ms/call", (time.perf_counter() - t) * 100)
