"""The four random all-gate stress cases that sit at 1.03-1.11x the A2 bound
(profiles/r02/stress_random_summary.txt), re-run with individual code-generation features switched
off, to see which one (if any) carries the extra fp32 noise. usage: python profiles/marginal_cases.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from circuit_helpers import random_circuit  # noqa: E402
from oracle import layersim_oracle as orc  # noqa: E402
from paper_2506_04891_b200 import codegen  # noqa: E402
from paper_2506_04891_b200.engine import Engine  # noqa: E402


def draw(seed, case):
    rng = np.random.default_rng(seed)
    for _ in range(case + 1):
        n = int(rng.integers(6, 13))
        M = int(rng.integers(5, n + 1))
        circ = random_circuit(rng, n, int(rng.integers(6, 18)))
        B = int(rng.integers(1, 4))
        theta = rng.uniform(-3, 3, circ.trainable_count)
        x = rng.uniform(0, 3, (B, circ.encoding_count))
        w = rng.normal(size=n)
    return circ, n, M, B, theta, x, w


def a2(g, gr):
    return float(np.max(np.abs(g - gr) / np.maximum(np.abs(gr), 1e-2 * np.abs(gr).max())))


VARIANTS = [("default", {}, {}), ("no prefix/fold", {}, dict(prefix=False, fold=False)), ("no fold", {}, dict(fold=False)),
            ("no split", {}, dict(split=False)), ("EULER_TAN=0", dict(EULER_TAN=False), {}),
            ("UNIT_CONST=0", dict(UNIT_CONST=False), {}), ("TAN_ROT=0", dict(TAN_ROT=False), {}),
            ("FOLD_DRUN=0", dict(FOLD_DRUN=False), {}), ("EULER_MERGE=0", dict(EULER_MERGE=0), {}),
            ("EULER_COUP=0", dict(EULER_COUP=False), {})]
for seed, case in ((1, 91), (2, 14), (5, 57), (7, 31)):
    circ, n, M, B, theta, x, w = draw(seed, case)
    ref = orc.gradient(circ, theta, x, batch=B, weights=w)
    gr = np.concatenate([ref["grads"], ref["encoding_grads"]], 1)
    r32 = orc.gradient(circ, theta, x, batch=B, weights=w, dtype=np.complex64)
    print(f"seed {seed} case {case}: n={n} M={M} B={B}  complex64 model A2 {a2(np.concatenate([r32['grads'], r32['encoding_grads']], 1), gr):.2e}")
    for name, flags, kw in VARIANTS:
        saved = {k: getattr(codegen, k) for k in flags}
        for k, v in flags.items():
            setattr(codegen, k, v)
        try:
            r = Engine(circ, M=M, **kw).fwd_bwd(theta, x, batch=B, weights=w)
            host = lambda t: np.zeros((B, 0)) if t is None else t.cpu().numpy()  # noqa: E731
            g = np.concatenate([host(r["grads"]), host(r["encoding_grads"])], 1)
            j = int(np.argmax(np.abs(g - gr) / np.maximum(np.abs(gr), 1e-2 * np.abs(gr).max())))
            print(f"   {name:16s} A2 {a2(g, gr):.2e}  worst entry {j} (|g_ref| {abs(gr.flat[j]):.1e}, abs err {abs(g.flat[j] - gr.flat[j]):.1e}, "
                  f"{'trainable' if j % gr.shape[1] < ref['grads'].shape[1] else 'encoding'})")
        finally:
            for k, v in saved.items():
                setattr(codegen, k, v)
