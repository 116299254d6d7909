"""Generate the golden fixtures by running the REFERENCE itself (not the oracle).

Run in the authoring container, where the read-only reference exists:

    PYTHONPATH=/root/repo python tests/golden/make_golden.py [--big]

`LAYERSIM_REF_SRC` may point at a writable copy whose Cython backend was built with
`python setup.py build_ext --inplace` (e.g. /tmp/refbuild/src); otherwise the reference's
numpy backend under /root/reference/pkg/src is used (identical math, slower).

Adapters (none modifies a reference file):
* weighted loss  -- `layersim.grad.z_weights` / `layersim.states.z_weights` are rebound
  to d(i) = sum_q w_q (1 - 2 bit_q(i));
* per-qubit <Z_q> -- the reference primitive `ops().zsum(amps, 1 - 2 J[:, q])`;
* capacity        -- rows are run in chunks under the 2^27-element budget
  (batch independence is a reference invariant, tests/test_core.py:198-209).

Outputs (all small): tests/golden/*.npz. The GPU box never reads /root/reference.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, os.environ.get("LAYERSIM_REF_SRC", "/root/reference/pkg/src"))

import layersim as ref  # noqa: E402  (the reference package)
import layersim.grad as ref_grad  # noqa: E402
import layersim.states as ref_states  # noqa: E402
from layersim.backend import ops as ref_ops  # noqa: E402
from layersim.kernels import build_k_matrix, compose_permutation  # noqa: E402
from layersim.oracle import layer_unitary  # noqa: E402

from paper_2506_04891_b200.configs import make_workload  # noqa: E402


def to_ref_circuit(circ):
    layers = []
    for layer in circ.layers:
        pk = layer.pattern.kind.value
        pat = ref.WirePattern(ref.PatternKind(pk), layer.pattern.wires)
        role = None if layer.role is None else ref.Role(layer.role.value)
        layers.append(ref.Layer(ref.GateKind(layer.gate.value), pat, role, layer.values))
    return ref.Circuit(circ.n, layers)


def weighted(n, w):
    idx = np.arange(1 << n)
    d = np.zeros(1 << n)
    for q in range(n):
        d += w[q] * (1.0 - 2.0 * ((idx >> (n - 1 - q)) & 1))
    d.setflags(write=False)
    return d


def run_reference(circ, theta, x, w, rows_per_chunk):
    """Reference gradient() on chunks of rows, weighted loss, per-qubit <Z_q>."""
    n = circ.n
    rc = to_ref_circuit(circ)
    d = weighted(n, w)
    saved = (ref_grad.z_weights, ref_states.z_weights)
    ref_grad.z_weights = ref_states.z_weights = lambda m: d if m == n else saved[0](m)
    try:
        outs = {"value": [], "grads": [], "encoding_grads": [], "zq": []}
        B = x.shape[0]
        idx = np.arange(1 << n)
        for s in range(0, B, rows_per_chunk):
            xb = x[s : s + rows_per_chunk]
            b = xb.shape[0]
            final = ref.apply_circuit(
                rc, theta if rc.trainable_count else None, xb if rc.encoding_count else None,
                state=ref.zero_state(n, b),
            )
            res = ref.backward_sweep(
                rc, theta if rc.trainable_count else None, xb if rc.encoding_count else None, final
            )
            zq = np.stack(
                [ref_ops().zsum(final.amplitudes, 1.0 - 2.0 * ((idx >> (n - 1 - q)) & 1)) for q in range(n)],
                axis=1,
            )
            outs["value"].append(res.value)
            outs["grads"].append(res.grads)
            outs["encoding_grads"].append(res.encoding_grads)
            outs["zq"].append(zq)
        return {k: np.concatenate(v, axis=0) for k, v in outs.items()}
    finally:
        ref_grad.z_weights, ref_states.z_weights = saved


def save_config(tag, cfg, n, batch, rows_per_chunk):
    t0 = time.time()
    wl = make_workload(cfg, n=n, batch=batch)
    out = run_reference(wl.circuit, wl.theta, wl.x, wl.weights, rows_per_chunk)
    path = os.path.join(HERE, f"{tag}.npz")
    np.savez_compressed(
        path, cfg=cfg, n=wl.n, batch=wl.batch, x=wl.x, theta=wl.theta, weights=wl.weights, **out
    )
    print(f"{tag}: cfg{cfg} n={wl.n} B={wl.batch} in {time.time() - t0:.1f}s -> {path}", flush=True)


def save_known_answers():
    """Known-answer vectors straight from the reference (pins conventions)."""
    kv = {}
    rng = np.random.default_rng(5)
    for g in ref.GateKind:
        cnt = ref.GATE_TRAITS[g].param_count
        if cnt == 0:
            kv[f"gate_{g.value}"] = ref.gate_matrix(g)
        else:
            p = rng.uniform(-np.pi, np.pi, (3, cnt))
            kv[f"gate_{g.value}_params"] = p
            kv[f"gate_{g.value}"] = ref.gate_matrix(g, p)
            for k in range(cnt):
                kv[f"dgate_{g.value}_{k}"] = ref_grad.gate_matrix_derivative(g, p, k)
    for n in (2, 3, 4, 5, 8):
        kv[f"sigma_cnot_ring_{n}"] = compose_permutation(
            ref.Layer(ref.GateKind.CNOT, ref.ring_pairs()), n
        ).sigma
    kv["sigma_x_all_2"] = compose_permutation(ref.Layer(ref.GateKind.X, ref.all_qubits()), 2).sigma
    kv["sigma_swap_02_3"] = compose_permutation(
        ref.Layer(ref.GateKind.SWAP, ref.explicit((0, 2))), 3
    ).sigma
    kv["k_rz_3"] = build_k_matrix(ref.GateKind.RZ, 3).k
    kv["z_weights_3"] = np.asarray(ref.z_weights(3))
    # dense layer unitaries for a handful of layers at n=4 (ordering conventions)
    layers = {
        "rzz_ring": (ref.Layer(ref.GateKind.RZZ, ref.ring_pairs(), ref.Role.TRAINABLE), 1),
        "ms_chain": (ref.Layer(ref.GateKind.MS, ref.chain_pairs(), ref.Role.TRAINABLE), 3),
        "ecr_explicit": (ref.Layer(ref.GateKind.ECR, ref.explicit((2, 0), (1, 3))), 0),
        "cnot_ring": (ref.Layer(ref.GateKind.CNOT, ref.ring_pairs()), 0),
        "rot_all": (ref.Layer(ref.GateKind.ROT, ref.all_qubits(), ref.Role.TRAINABLE), 3),
    }
    for name, (layer, k) in layers.items():
        pos = ref.positions(layer, 4)
        p = rng.uniform(-1.5, 1.5, (len(pos), k)) if k else None
        kv[f"layer_{name}_params"] = p if p is not None else np.zeros((0,))
        kv[f"layer_{name}"] = layer_unitary(layer, 4, p)
    # X layers and GPI xor-flips (permutation/antidiagonal index maps, bit-exact tests);
    # fixed angles so these keys do not consume the rng stream above
    from layersim.kernels import _flip_mask

    for n in (3, 5):
        kv[f"sigma_x_all_{n}"] = compose_permutation(ref.Layer(ref.GateKind.X, ref.all_qubits()), n).sigma
    kv["sigma_x_explicit_0_2_4"] = compose_permutation(
        ref.Layer(ref.GateKind.X, ref.explicit((0,), (2,))), 4).sigma
    gpi = {"all_4": (ref.all_qubits(), 4), "explicit_1_3_5": (ref.explicit((1,), (3,)), 5)}
    for name, (pat, n) in gpi.items():
        layer = ref.Layer(ref.GateKind.GPI, pat, ref.Role.TRAINABLE)
        pos = ref.positions(layer, n)
        kv[f"gpi_flip_mask_{name}"] = np.int64(_flip_mask(pos, n))
        for tag, p in (("zero", np.zeros((len(pos), 1))), ("phase", np.linspace(0.05, 0.4, len(pos))[:, None])):
            kv[f"layer_gpi_{name}_{tag}_params"] = p
            kv[f"layer_gpi_{name}_{tag}"] = layer_unitary(layer, n, p)
    path = os.path.join(HERE, "known_answers.npz")
    np.savez_compressed(path, **kv)
    print("known answers ->", path)


def save_random_circuits():
    """Mixed random circuits over every gate and pattern (reference test_grad.py:70-89 style),
    n=5, batch=3, run through the reference gradient."""
    rng = np.random.default_rng(20260101)
    G, P, R = ref.GateKind, ref.PatternKind, ref.Role
    one = [G.RY, G.RX, G.RZ, G.ROT, G.GPI, G.GPI2, G.H, G.S, G.Z, G.X, G.SX]
    two = [G.CNOT, G.CZ, G.RZZ, G.MS, G.ECR, G.SWAP]
    out = {}
    for c in range(6):
        n = 5
        layers = []
        for _ in range(10):
            if rng.random() < 0.55:
                g = one[rng.integers(len(one))]
                pat = ref.all_qubits() if rng.random() < 0.7 else ref.explicit(
                    *[(int(q),) for q in rng.permutation(n)[: rng.integers(1, n)]]
                )
            else:
                g = two[rng.integers(len(two))]
                r = rng.random()
                if r < 0.35:
                    pat = ref.ring_pairs()
                elif r < 0.7:
                    pat = ref.chain_pairs()
                else:
                    prs = [tuple(int(v) for v in rng.permutation(n)[:2]) for _ in range(rng.integers(1, 4))]
                    pat = ref.explicit(*prs)
            cnt = ref.GATE_TRAITS[g].param_count
            if cnt == 0:
                layers.append(ref.Layer(g, pat))
            else:
                role = [R.TRAINABLE, R.ENCODING, R.FIXED][rng.integers(3)]
                vals = None
                if role is R.FIXED:
                    npos = len(ref.positions(ref.Layer(g, pat, R.TRAINABLE), n))
                    vals = tuple(tuple(float(v) for v in rng.uniform(-1, 1, cnt)) for _ in range(npos))
                layers.append(ref.Layer(g, pat, role, vals))
        circ = ref.Circuit(n, layers)
        theta = rng.uniform(-np.pi, np.pi, circ.trainable_count)
        x = rng.uniform(-np.pi, np.pi, (3, circ.encoding_count))
        w = rng.standard_normal(n)
        res = run_reference(circ, theta, x, w, 3)
        spec = [
            (l.gate.value, l.pattern.kind.value, l.pattern.wires, None if l.role is None else l.role.value, l.values)
            for l in layers
        ]
        out[f"c{c}_spec"] = np.array(repr(spec))
        out[f"c{c}_theta"], out[f"c{c}_x"], out[f"c{c}_w"] = theta, x, w
        for k, v in res.items():
            out[f"c{c}_{k}"] = v
    path = os.path.join(HERE, "random_circuits.npz")
    np.savez_compressed(path, **out)
    print("random circuits ->", path)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also the full-width cfg2..cfg5 row subsets")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    print("reference backend:", ref.active_backend())
    jobs = [("known", None), ("random", None)]
    jobs += [(f"small_cfg{c}", (c, 6, 3, 3)) for c in range(1, 6)]
    jobs += [("cfg1_full", (1, None, None, 64))]
    if args.big:
        jobs += [
            ("cfg2_rows4", (2, None, 4, 4)),
            ("cfg3_rows2", (3, None, 2, 2)),
            ("cfg4_rows1", (4, None, 1, 1)),
            ("cfg5_rows1", (5, None, 1, 1)),
        ]
    for tag, spec in jobs:
        if args.only and tag not in args.only.split(","):
            continue
        if tag == "known":
            save_known_answers()
        elif tag == "random":
            save_random_circuits()
        else:
            save_config(tag, *spec)


if __name__ == "__main__":
    main()
