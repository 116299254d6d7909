"""Profiling driver: a few fwd+bwd steps of a BASELINE config through the engine (used
under ncu; never a bench number)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_04891_b200.configs import make_workload
from paper_2506_04891_b200.engine import Engine

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
batch = int(sys.argv[3]) if len(sys.argv) > 3 else None
wl = make_workload(cfg, batch=batch)
eng = Engine(wl.circuit)
th = torch.as_tensor(wl.theta, device="cuda"); x = torch.as_tensor(wl.x, device="cuda")
w = torch.as_tensor(wl.weights, device="cuda")
bufs = None
for _ in range(steps):
    r = eng.fwd_bwd(th, x, batch=wl.batch, weights=w, rows=False, encoding_grads=False, buffers=bufs)
    bufs = r["buffers"]
torch.cuda.synchronize()
print("ok", len(eng.program.passes), "passes")
