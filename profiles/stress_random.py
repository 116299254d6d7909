"""GPU stress run over random circuits of ALL 17 gate kinds, patterns and roles (the generator of
tests/circuit_helpers.py) at random widths and tilings; the numpy oracle is the checker. Bound per
case: <Z_q> 1e-5 absolute; gradients A2 at 1e-4, or twice the A2 error of the reference algorithm
run in complex64 where that precision model itself breaks 1e-4 (the rule of
tests/test_gpu_parity.py::test_random_circuits_multipass); structurally zero gradients absolutely
(1e-6, or twice the complex64 model's own noise on them).
usage: python profiles/stress_random.py [CASES] [SEED] [NMIN NMAX [MMIN]]   (n in [NMIN, NMAX), M in [MMIN, min(n, 13)])"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from circuit_helpers import random_circuit  # noqa: E402
from oracle import layersim_oracle as orc  # noqa: E402


def a2(g, gr):
    if gr.size == 0:
        return 0.0
    return float(np.max(np.abs(g - gr) / np.maximum(np.abs(gr), 1e-2 * np.abs(gr).max())))


def main(cases, seed, n_range=(6, 13), m_min=5):
    from paper_2506_04891_b200.engine import Engine

    rng = np.random.default_rng(seed)
    bad, worst, t0 = 0, 0.0, time.time()
    for c in range(cases):
        n = int(rng.integers(*n_range))
        M = int(rng.integers(m_min, min(n, 13) + 1))
        circ = random_circuit(rng, n, int(rng.integers(6, 18)))
        B = int(rng.integers(1, 4))
        theta = rng.uniform(-3, 3, circ.trainable_count)
        x = rng.uniform(0, 3, (B, circ.encoding_count))
        w = rng.normal(size=n)
        eng = Engine(circ, M=M)
        r = eng.fwd_bwd(theta, x, batch=B, weights=w)
        ref = orc.gradient(circ, theta, x, batch=B, weights=w)
        host = lambda t: np.zeros((B, 0)) if t is None else t.cpu().numpy()  # noqa: E731
        g = np.concatenate([host(r["grads"]), host(r["encoding_grads"])], 1)
        gr = np.concatenate([ref["grads"], ref["encoding_grads"]], 1)
        zerr = float(np.abs(r["zq"].cpu().numpy() - ref["zq"]).max())
        if gr.size and np.abs(gr).max() < 1e-12:
            # structurally zero gradients: absolute, against the complex64 model's own noise
            err, tol = float(np.abs(g).max()), 1e-6
            if err > tol:
                r32 = orc.gradient(circ, theta, x, batch=B, weights=w, dtype=np.complex64)
                tol = max(tol, 2 * float(np.abs(np.concatenate([r32["grads"], r32["encoding_grads"]], 1)).max()))
        else:
            err, tol = a2(g, gr), 1e-4
            if err > tol:  # the precision model decides
                r32 = orc.gradient(circ, theta, x, batch=B, weights=w, dtype=np.complex64)
                tol = max(tol, 2 * a2(np.concatenate([r32["grads"], r32["encoding_grads"]], 1), gr))
        ok = zerr <= 1e-5 and err <= tol
        bad += not ok
        worst = max(worst, err / tol)
        print(f"case {c:3d} n={n:2d} M={M:2d} B={B} layers={len(circ.layers):2d} passes={len(eng.program.passes):2d} "
              f"zq_err={zerr:.1e} grad_err={err:.1e} tol={tol:.1e} {'ok' if ok else 'FAIL'}", flush=True)
        del eng
    print(f"{cases} cases, {bad} failures, worst error / bound {worst:.2f}, {time.time() - t0:.0f} s")
    return 1 if bad else 0


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:]]
    sys.exit(main(a[0] if a else 40, a[1] if len(a) > 1 else 0, (a[2], a[3]) if len(a) > 3 else (6, 13),
                  a[4] if len(a) > 4 else 5))
