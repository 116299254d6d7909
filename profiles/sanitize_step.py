"""Driver for compute-sanitizer (racecheck / synccheck / memcheck / initcheck): every kernel
mode of the specialised pass kernels at small n, with multi-pass tilings so the next-tile
prefetch stage, rotating exchange buffers, prefix synthesis, folded observables, checkpoint and
recompute adjoints, and the turnaround all run. Never a timing run.
usage: python profiles/sanitize_step.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04891_b200 import apply_circuit, gradient  # noqa: E402
from paper_2506_04891_b200.configs import make_workload  # noqa: E402
from paper_2506_04891_b200.engine import Engine  # noqa: E402
from paper_2506_04891_b200.planner import plan_for_tile_bits  # noqa: E402
from paper_2506_04891_b200.states import zero_state  # noqa: E402

kinds = 0
for cfg, n, M, b in [(2, 11, 8, 3), (3, 11, 8, 2), (4, 11, 9, 2), (5, 12, 9, 2), (1, 8, None, 3)]:
    wl = make_workload(cfg, n=n, batch=b)
    eng = Engine(wl.circuit, M=M)
    for ck in (True, False):
        r = eng.fwd_bwd(wl.theta, wl.x, batch=b, weights=wl.weights, checkpoint=ck)
        kinds += 1
    # micro-batched (partial last chunk)
    eng.fwd_bwd(wl.theta, wl.x, batch=b, weights=wl.weights, micro_batch=max(1, b - 1), checkpoint=True)
    # forward-only program (no prefix, no folding) + backward from a given state
    st = apply_circuit(wl.circuit, wl.theta, wl.x, state=zero_state(n, b), plan=plan_for_tile_bits(wl.circuit, b, M or n))
    from paper_2506_04891_b200 import backward_sweep

    backward_sweep(wl.circuit, wl.theta, wl.x, st, weights=wl.weights)
    gradient(wl.circuit, wl.theta, wl.x, batch=b, weights=wl.weights)  # CUDA-graph step
    torch.cuda.synchronize()
    print(f"cfg{cfg} n={n} M={M}: {len(eng.program.passes)} passes ok", flush=True)
print("sanitize driver done")
