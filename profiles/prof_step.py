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
eng = Engine(wl.circuit, M=M, R=R)
th = torch.as_tensor(wl.theta, device="cuda"); x = torch.as_tensor(wl.x, device="cuda")
w = torch.as_tensor(wl.weights, device="cuda")
bufs = None
for _ in range(steps):
    r = eng.fwd_bwd(th, x, batch=wl.batch, weights=w, rows=False, encoding_grads=False, buffers=bufs)
    bufs = r["buffers"]
torch.cuda.synchronize()
print("ok", len(eng.program.passes), "passes")
