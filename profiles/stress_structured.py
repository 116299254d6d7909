"""GPU stress run of the compiler searches and the Euler-form kernels on randomised hardware-style
circuits (not a pytest: a few minutes of B200 time, run by a box script; the oracle is the checker).

Each case draws n, the tile exponent M, a native gate family (IBM: RZ.SX.RZ layers + ECR pairs; IonQ:
GPI2.GPI layers + MS(0,0,1/4) pairs; VQ: RX.RY.RZ + CNOT pairs + ZZ), the number of blocks, the
entangler pattern (even / odd ladders, ring, chain, random explicit pairs) and the role of every
parametrised layer (trainable / encoding / fixed), runs forward + adjoint through the engine at that
tiling and compares <Z_q> (1e-5 absolute) and all angle gradients (A2, 1e-4) with the numpy oracle.
usage: python profiles/stress_structured.py [CASES] [SEED] [NMIN NMAX [MMIN MMAX]]   (half-open ranges)"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import layersim_oracle as orc  # noqa: E402
from paper_2506_04891_b200.circuits import Circuit, Layer, Role, all_qubits, chain_pairs, explicit, ring_pairs  # noqa: E402
from paper_2506_04891_b200.gates import GATE_TRAITS, GateKind  # noqa: E402

rng = np.random.default_rng(0)  # reseeded by main() / the CPU test that imports build()


def npos(pat, n):
    k = pat.kind.value
    return n if k in ("all", "ring") else n - 1 if k == "chain" else len(pat.wires)


def layer(kind, pat, n, role=None):
    g = GateKind(kind)
    k = GATE_TRAITS[g].param_count
    if k == 0:
        return Layer(g, pat)
    if role is None:
        role = [Role.TRAINABLE, Role.TRAINABLE, Role.ENCODING, Role.FIXED][rng.integers(4)]
    if role is Role.FIXED:
        return Layer(g, pat, role, rng.uniform(-3, 3, (npos(pat, n), k)).tolist())
    return Layer(g, pat, role)


def entangler(n):
    r = rng.random()
    if r < 0.4:
        ev = explicit(*[(q, q + 1) for q in range(0, n - 1, 2)])
        od = explicit(*[(q, q + 1) for q in range(1, n - 1, 2)])
        return [ev, od]
    if r < 0.55:
        return [ring_pairs()]
    if r < 0.7:
        return [chain_pairs()]
    pairs = [tuple(int(w) for w in rng.choice(n, 2, replace=False)) for _ in range(int(rng.integers(2, n)))]
    return [explicit(*pairs)]


def build(n):
    fam = ["ibm", "ionq", "vq"][rng.integers(3)]
    layers = []
    if fam == "ibm":
        layers += [layer("sx", all_qubits(), n), layer("rz", all_qubits(), n, Role.ENCODING)]
    else:
        layers += [layer("ry", all_qubits(), n, Role.ENCODING)]
    for _ in range(int(rng.integers(1, 4))):
        if fam == "ibm":
            layers += [layer("rz", all_qubits(), n), layer("sx", all_qubits(), n), layer("rz", all_qubits(), n)]
            two = "ecr"
        elif fam == "ionq":
            layers += [layer("gpi2", all_qubits(), n), layer("gpi", all_qubits(), n)]
            two = "ms"
        else:
            layers += [layer(g, all_qubits(), n) for g in ("rx", "ry", "rz")]
            two = "cnot"
        for pat in entangler(n):
            if two == "ms":
                layers.append(Layer(GateKind("ms"), pat, Role.FIXED, [[0.0, 0.0, 0.25]] * npos(pat, n)))
            else:
                layers.append(layer(two, pat, n))
        if fam == "vq" and rng.random() < 0.5:
            layers.append(layer("rzz", chain_pairs(), n))
    return fam, Circuit(n, layers)


N_RANGE, M_RANGE = (9, 15), (7, 12)  # n in [9, 15), M in [7, min(n, 12)); main() may widen them


def draw_case():
    """(family, circuit, n, tile exponent M, batch) of the next random case"""
    n = int(rng.integers(*N_RANGE))
    M = int(rng.integers(M_RANGE[0], min(n, M_RANGE[1])))
    fam, circ = build(n)
    return fam, circ, n, M, int(rng.integers(1, 4))


def main(cases, seed, n_range=None, m_range=None):
    global rng, N_RANGE, M_RANGE
    from paper_2506_04891_b200.engine import Engine

    N_RANGE, M_RANGE = n_range or N_RANGE, m_range or M_RANGE

    rng = np.random.default_rng(seed)
    worst, bad, t0 = 0.0, 0, time.time()
    for c in range(cases):
        fam, circ, n, M, B = draw_case()
        theta = rng.uniform(-3, 3, circ.trainable_count)
        x = rng.uniform(0, 3, (B, circ.encoding_count))
        w = rng.normal(size=n)
        eng = Engine(circ, M=M)
        r = eng.fwd_bwd(theta, x, batch=B, weights=w)
        ref = orc.gradient(circ, theta, x, batch=B, weights=w)
        zerr = float(np.abs(r["zq"].cpu().numpy() - ref["zq"]).max())
        host = lambda t: np.zeros((B, 0)) if t is None else t.cpu().numpy()  # noqa: E731 (no such angles)
        g = np.concatenate([host(r["grads"]), host(r["encoding_grads"])], 1)
        gr = np.concatenate([ref["grads"], ref["encoding_grads"]], 1)
        if gr.size == 0:
            a2 = 0.0
        elif np.abs(gr).max() > 1e-9:
            a2 = float(np.max(np.abs(g - gr) / np.maximum(np.abs(gr), 1e-2 * np.abs(gr).max())))
        else:  # structurally zero gradients: absolute
            a2 = float(np.abs(g).max())
        tol = 1e-4
        if a2 > tol and gr.size and np.abs(gr).max() > 1e-9:
            # the rule of the random-circuit tests: twice the A2 error of the reference algorithm
            # run in complex64 where that precision model itself breaks 1e-4 (tiny gradients)
            r32 = orc.gradient(circ, theta, x, batch=B, weights=w, dtype=np.complex64)
            g32 = np.concatenate([r32["grads"], r32["encoding_grads"]], 1)
            tol = max(tol, 2 * float(np.max(np.abs(g32 - gr) / np.maximum(np.abs(gr), 1e-2 * np.abs(gr).max()))))
        ok = zerr <= 1e-5 and a2 <= tol
        worst = max(worst, a2)
        bad += not ok
        print(f"case {c:3d} {fam:4s} n={n:2d} M={M:2d} B={B} layers={len(circ.layers):2d} passes={len(eng.program.passes):2d} "
              f"phases={sum(len(p.phases) for p in eng.program.passes):3d} zq_err={zerr:.1e} a2={a2:.1e} tol={tol:.1e} {'ok' if ok else 'FAIL'}",
              flush=True)
        del eng
    print(f"{cases} cases, {bad} failures, worst A2 {worst:.2e}, {time.time() - t0:.0f} s")
    return 1 if bad else 0


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:]]
    sys.exit(main(a[0] if a else 40, a[1] if len(a) > 1 else 0,
                  (a[2], a[3]) if len(a) > 3 else None, (a[4], a[5]) if len(a) > 5 else None))
