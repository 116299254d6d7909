"""CPU ORACLE -- test infrastructure only, never the product path.

A numpy (complex128) restatement of the reference's batched forward + adjoint backward
path, used as the parity checker by `tests/`, by `__graft_entry__.smoke()` and as the
CPU baseline leg of `bench.py` ("kind": "port"). Nothing under `paper_2506_04891_b200/`
imports this module; the product path fails loudly when its CUDA library is missing.

What it restates (reference files under /root/reference/pkg/src/layersim/):

* gate matrices and derivatives ............ gates.py:144-312
* wire positions / slot layout ............. circuits.py:95-214
* einsum kernel: one pass per position ..... kernels.py:579-637, _pyops.py:73-138
* apply_circuit (copy, then layer loop) .... core.py:46-72
* z_weights / expectation_z_sum ............ states.py:88-102 (+ the weighted-loss adapter
  of SURVEY §0.2: d(i) = sum_q w_q (1 - 2 bit_q(i)); w = ones reproduces sum_k Z_k)
* backward_sweep / layer_backward .......... grad.py:143-204
  - commuting rule (diagonal or disjoint layers) grad.py:102-119
  - descending rule (overlapping non-commuting) grad.py:122-140
  - couplings / contraction ................ grad.py:40-73
* gradient ................................. grad.py:207-218

Parity pinning: `tests/test_oracle.py` checks this module against golden vectors produced
by the reference itself (`tests/golden/make_golden.py`, run in the authoring container
where /root/reference exists) and against the reference test-suite's known answers.
"""

from __future__ import annotations

import numpy as np

_R2 = np.sqrt(0.5)
_TWO_PI = 2.0 * np.pi

# (arity, param_count, diagonal) per gate name -- reference gates.py:60-78
_TRAITS = {
    "z": (1, 0, True), "cz": (2, 0, True), "rz": (1, 1, True), "rzz": (2, 1, True),
    "gpi": (1, 1, False), "s": (1, 0, True), "cnot": (2, 0, False), "x": (1, 0, False),
    "h": (1, 0, False), "ry": (1, 1, False), "rx": (1, 1, False), "rot": (1, 3, False),
    "gpi2": (1, 1, False), "ms": (2, 3, False), "sx": (1, 0, False), "ecr": (2, 0, False),
    "swap": (2, 0, False),
}


def _name(layer) -> str:
    return layer.gate.value


# ----------------------------------------------------------------------------- gates


def _m2(a, b, c, d):
    a, b, c, d = np.broadcast_arrays(*(np.asarray(v, dtype=complex) for v in (a, b, c, d)))
    return np.stack([np.stack([a, b], -1), np.stack([c, d], -1)], -2)


def _rz(t):
    e = np.exp(-0.5j * t)
    return _m2(e, 0 * e, 0 * e, np.conj(e))


def _ry(t):
    c, s = np.cos(t / 2), np.sin(t / 2)
    return _m2(c, -s, s, c)


def _rx(t):
    c, s = np.cos(t / 2), np.sin(t / 2)
    return _m2(c, -1j * s, -1j * s, c)


def _const(name):
    table = {
        "z": np.diag([1, -1]), "s": np.diag([1, 1j]), "x": [[0, 1], [1, 0]],
        "h": _R2 * np.array([[1, 1], [1, -1]]), "sx": 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]]),
        "cz": np.diag([1, 1, 1, -1]), "cnot": np.eye(4)[[0, 1, 3, 2]], "swap": np.eye(4)[[0, 2, 1, 3]],
        "ecr": _R2 * np.array([[0, 1, 0, 1j], [1, 0, -1j, 0], [0, 1j, 0, 1], [-1j, 0, 1, 0]]),
    }
    return np.asarray(table[name], dtype=complex)


def gate_matrix(name: str, p=None) -> np.ndarray:
    """Unitary, broadcast over leading axes of p[..., k] (reference gates.py:144-236)."""
    if _TRAITS[name][1] == 0:
        return _const(name)
    p = np.asarray(p, dtype=float)
    if name == "rz":
        return _rz(p[..., 0])
    if name == "ry":
        return _ry(p[..., 0])
    if name == "rx":
        return _rx(p[..., 0])
    if name == "rot":
        return _rz(p[..., 2]) @ _ry(p[..., 1]) @ _rz(p[..., 0])
    if name == "gpi":
        e = np.exp(1j * _TWO_PI * p[..., 0])
        return _m2(0 * e, np.conj(e), e, 0 * e)
    if name == "gpi2":
        e = np.exp(1j * _TWO_PI * p[..., 0])
        one = np.full(e.shape, _R2, dtype=complex)
        return _m2(one, -1j * _R2 * np.conj(e), -1j * _R2 * e, one)
    if name == "rzz":
        e = np.exp(-0.5j * p[..., 0])
        out = np.zeros(e.shape + (4, 4), dtype=complex)
        out[..., 0, 0] = out[..., 3, 3] = e
        out[..., 1, 1] = out[..., 2, 2] = np.conj(e)
        return out
    if name == "ms":
        c, s = np.cos(np.pi * p[..., 2]), np.sin(np.pi * p[..., 2])
        es = np.exp(1j * _TWO_PI * (p[..., 0] + p[..., 1]))
        ed = np.exp(1j * _TWO_PI * (p[..., 0] - p[..., 1]))
        out = np.zeros(c.shape + (4, 4), dtype=complex)
        for i in range(4):
            out[..., i, i] = c
        out[..., 0, 3] = -1j * s * np.conj(es)
        out[..., 3, 0] = -1j * s * es
        out[..., 1, 2] = -1j * s * ed
        out[..., 2, 1] = -1j * s * np.conj(ed)
        return out
    raise ValueError(name)


def gate_derivative(name: str, p, k: int) -> np.ndarray:
    """d U / d p[..., k] (reference gates.py:239-312)."""
    p = np.asarray(p, dtype=float)
    gen = {"rz": np.diag([1, -1]), "ry": [[0, -1j], [1j, 0]], "rx": [[0, 1], [1, 0]],
           "rzz": np.diag([1, -1, -1, 1])}
    if name in gen:
        return -0.5j * (np.asarray(gen[name], dtype=complex) @ gate_matrix(name, p))
    if name == "rot":
        a, b, c = p[..., 0], p[..., 1], p[..., 2]
        Z = np.diag([1, -1]).astype(complex)
        Y = np.array([[0, -1j], [1j, 0]])
        if k == 0:
            return _rz(c) @ _ry(b) @ (-0.5j * (Z @ _rz(a)))
        if k == 1:
            return _rz(c) @ (-0.5j * (Y @ _ry(b))) @ _rz(a)
        return (-0.5j * (Z @ _rz(c))) @ _ry(b) @ _rz(a)
    if name == "gpi":
        e = np.exp(1j * _TWO_PI * p[..., 0])
        return _m2(0 * e, -1j * _TWO_PI * np.conj(e), 1j * _TWO_PI * e, 0 * e)
    if name == "gpi2":
        e = np.exp(1j * _TWO_PI * p[..., 0])
        return _m2(0 * e, -_TWO_PI * _R2 * np.conj(e), _TWO_PI * _R2 * e, 0 * e)
    if name == "ms":
        c, s = np.cos(np.pi * p[..., 2]), np.sin(np.pi * p[..., 2])
        es = np.exp(1j * _TWO_PI * (p[..., 0] + p[..., 1]))
        ed = np.exp(1j * _TWO_PI * (p[..., 0] - p[..., 1]))
        out = np.zeros(c.shape + (4, 4), dtype=complex)
        if k == 2:
            for i in range(4):
                out[..., i, i] = -np.pi * s
            out[..., 0, 3] = -1j * np.pi * c * np.conj(es)
            out[..., 3, 0] = -1j * np.pi * c * es
            out[..., 1, 2] = -1j * np.pi * c * ed
            out[..., 2, 1] = -1j * np.pi * c * np.conj(ed)
            return out
        sg = 1.0 if k == 0 else -1.0
        out[..., 0, 3] = -_TWO_PI * s * np.conj(es)
        out[..., 3, 0] = _TWO_PI * s * es
        out[..., 1, 2] = sg * _TWO_PI * s * ed
        out[..., 2, 1] = -sg * _TWO_PI * s * np.conj(ed)
        return out
    raise ValueError(name)


# ----------------------------------------------------------------------------- IR helpers


def positions(layer, n: int):
    """reference circuits.py:95-126"""
    kind = layer.pattern.kind.value
    if kind == "all":
        return [(q,) for q in range(n)]
    if kind == "chain":
        return [(q, q + 1) for q in range(n - 1)]
    if kind == "ring":
        return [(0, 1)] if n == 2 else [(q, (q + 1) % n) for q in range(n)]
    return [tuple(w) for w in layer.pattern.wires]


def slots(circuit):
    """(role, start, count) per layer -- reference circuits.py:143-174"""
    out, t, e = [], 0, 0
    for layer in circuit.layers:
        arity, k, _ = _TRAITS[_name(layer)]
        cnt = len(positions(layer, circuit.n)) * k
        role = None if layer.role is None else layer.role.value
        if cnt == 0 or role is None:
            out.append(None)
        elif role == "fixed":
            out.append(("fixed", 0, cnt))
        elif role == "trainable":
            out.append(("trainable", t, cnt))
            t += cnt
        else:
            out.append(("encoding", e, cnt))
            e += cnt
    return out, t, e


def layer_params(circuit, i, sl, trainable, encoding):
    """reference circuits.py:189-214"""
    layer = circuit.layers[i]
    s = sl[i]
    if s is None:
        return None
    k = _TRAITS[_name(layer)][1]
    npos = len(positions(layer, circuit.n))
    if s[0] == "fixed":
        return np.asarray(layer.values, dtype=float).reshape(npos, k)
    if s[0] == "trainable":
        return np.asarray(trainable, dtype=float)[s[1] : s[1] + s[2]].reshape(npos, k)
    return np.asarray(encoding, dtype=float)[:, s[1] : s[1] + s[2]].reshape(-1, npos, k)


# ----------------------------------------------------------------------------- primitives


def _split1(psi, bit):
    b, dim = psi.shape
    lo = 1 << bit
    return psi.reshape(b, dim // (2 * lo), 2, lo)


def _split2(psi, ba, bb):
    """View with axes (b, w, A, y, B, z) where A is bit ba and B is bit bb (ba > bb) or
    swapped; returns (view, first_is_hi)."""
    hi, lo = (ba, bb) if ba > bb else (bb, ba)
    b, dim = psi.shape
    v = psi.reshape(b, dim >> (hi + 1), 2, 1 << (hi - lo - 1), 2, 1 << lo)
    return v, ba > bb


def apply_1q(psi, u, bit):
    """psi <- (u on bit) psi; u is (2,2) or per-row (B,2,2). reference _pyops.py:73-91"""
    v = _split1(psi, bit)
    a = v[:, :, 0, :].copy()
    b = v[:, :, 1, :]
    if u.ndim == 2:
        v[:, :, 0, :] = u[0, 0] * a + u[0, 1] * b
        v[:, :, 1, :] = u[1, 0] * a + u[1, 1] * b
    else:
        uu = u[:, None, None, :, :]
        n0 = uu[..., 0, 0] * a + uu[..., 0, 1] * b
        v[:, :, 1, :] = uu[..., 1, 0] * a + uu[..., 1, 1] * b
        v[:, :, 0, :] = n0


def apply_2q(psi, u, ba, bb):
    """4x4 u on (bit ba = first wire, bit bb); u (4,4) or (B,4,4). reference _pyops.py:94-138"""
    v, first_hi = _split2(psi, ba, bb)
    if not first_hi:  # reorder the local basis so the high bit comes first
        perm = [0, 2, 1, 3]
        u = u[..., perm, :][..., :, perm]
    blocks = [v[:, :, i, :, j, :].copy() for i in (0, 1) for j in (0, 1)]
    for r in range(4):
        i, j = divmod(r, 2)
        acc = 0
        for c in range(4):
            coef = u[r, c] if u.ndim == 2 else u[:, r, c][:, None, None, None]
            acc = acc + coef * blocks[c]
        v[:, :, i, :, j, :] = acc


def apply_gate(psi, mat, bits):
    if len(bits) == 1:
        apply_1q(psi, mat, bits[0])
    else:
        apply_2q(psi, mat, bits[0], bits[1])


def dagger(u):
    return np.conj(np.swapaxes(u, -1, -2))


def coupling(lam, psi, bits):
    """M[b, i, j] = sum conj(lam_i) psi_j over the local sub-blocks (reference grad.py:49-61)."""
    if len(bits) == 1:
        lv, pv = _split1(lam, bits[0]), _split1(psi, bits[0])
        return np.einsum("bxiy,bxjy->bij", lv.conj(), pv)
    lv, first_hi = _split2(lam, bits[0], bits[1])
    pv, _ = _split2(psi, bits[0], bits[1])
    m = np.einsum("bwiyjz,bwkylz->bijkl", lv.conj(), pv)
    if not first_hi:
        m = m.transpose(0, 2, 1, 4, 3)
    return m.reshape(m.shape[0], 4, 4)


# ----------------------------------------------------------------------------- observable


def z_diag(n: int, weights=None) -> np.ndarray:
    """d(i) = sum_q w_q (1 - 2 bit_{n-1-q}(i)); w=None -> n - 2 popcount (states.py:88-97)."""
    w = np.ones(n) if weights is None else np.asarray(weights, dtype=float)
    idx = np.arange(1 << n)
    d = np.zeros(1 << n)
    for q in range(n):
        d += w[q] * (1.0 - 2.0 * ((idx >> (n - 1 - q)) & 1))
    return d


def expectation_z(psi: np.ndarray, n: int) -> np.ndarray:
    """<Z_q> per row, shape (B, n)."""
    p = np.abs(psi) ** 2
    idx = np.arange(1 << n)
    out = np.empty((psi.shape[0], n))
    for q in range(n):
        s = 1.0 - 2.0 * ((idx >> (n - 1 - q)) & 1)
        out[:, q] = p @ s
    return out


# ----------------------------------------------------------------------------- forward


def _layer_mats(circuit, i, sl, trainable, encoding, dtype=complex):
    layer = circuit.layers[i]
    name = _name(layer)
    pos = positions(layer, circuit.n)
    par = layer_params(circuit, i, sl, trainable, encoding)
    if par is None:
        m = gate_matrix(name).astype(dtype)
        return [m] * len(pos)
    if par.ndim == 2:
        return [gate_matrix(name, par[j]).astype(dtype) for j in range(len(pos))]
    return [gate_matrix(name, par[:, j]).astype(dtype) for j in range(len(pos))]


def apply_circuit(circuit, trainable=None, encoding=None, state=None, batch=1, dtype=complex):
    """Forward pass on a copy of `state` (default |0..0>), one pass per gate position
    (the reference's einsum kernel, kernels.py:611-622).

    `dtype=np.complex64` runs the same algorithm with complex64 states, matrices and einsum
    accumulation: a precision model of a single-precision engine (test-only, used to show
    which deviations are the complex64 rounding floor rather than a kernel defect)."""
    n = circuit.n
    if state is None:
        psi = np.zeros((batch, 1 << n), dtype=dtype)
        psi[:, 0] = 1.0
    else:
        psi = np.array(state, dtype=dtype, copy=True)
    sl, _, _ = slots(circuit)
    for i, layer in enumerate(circuit.layers):
        mats = _layer_mats(circuit, i, sl, trainable, encoding, dtype)
        for ws, m in zip(positions(layer, n), mats):
            apply_gate(psi, m, [n - 1 - w for w in ws])
    return psi


# ----------------------------------------------------------------------------- backward


def _inverse_layer(psi, circuit, i, mats):
    n = circuit.n
    pos = positions(circuit.layers[i], n)
    for j in range(len(pos) - 1, -1, -1):
        apply_gate(psi, dagger(mats[j]), [n - 1 - w for w in pos[j]])


def _contract(v, m):
    """2 Re sum_ij v_ij M_bij; v shared (d,d) or per row (B,d,d) -- reference grad.py:70-73"""
    sub = "ij,bij->b" if v.ndim == 2 else "bij,bij->b"
    return 2.0 * np.real(np.einsum(sub, v, m))


def _disjoint(pos):
    seen = set()
    for p in pos:
        if seen & set(p):
            return False
        seen |= set(p)
    return True


def backward_sweep(circuit, trainable, encoding, final, weights=None, need_encoding=True,
                   dtype=complex):
    """Adjoint reverse sweep (reference grad.py:169-204) with the weighted observable.

    Returns (value (B,), grads (B,T), encoding_grads (B,E)).
    """
    n = circuit.n
    sl, T, E = slots(circuit)
    psi = np.array(final, dtype=dtype, copy=True)
    real = np.float32 if np.dtype(dtype) == np.complex64 else float
    d = z_diag(n, weights).astype(real)
    lam = psi * d[None, :]
    batch = psi.shape[0]
    grads = np.zeros((batch, T))
    egrads = np.zeros((batch, E))
    last_needed = 0
    if not need_encoding:
        last_needed = min([i for i, s in enumerate(sl) if s and s[0] == "trainable"], default=0)
    for i in range(len(circuit.layers) - 1, last_needed - 1, -1):
        layer = circuit.layers[i]
        name = _name(layer)
        s = sl[i]
        mats = _layer_mats(circuit, i, sl, trainable, encoding, dtype)
        pos = positions(layer, n)
        need = s is not None and s[0] in ("trainable", "encoding")
        if not need:
            _inverse_layer(psi, circuit, i, mats)
            _inverse_layer(lam, circuit, i, mats)
            continue
        par = layer_params(circuit, i, sl, trainable, encoding)
        k = _TRAITS[name][1]
        out = np.zeros((batch, len(pos), k))
        bits = [[n - 1 - w for w in ws] for ws in pos]
        if _TRAITS[name][2] or _disjoint(pos):
            # commuting rule: step both down, then contract E^dag dE per position
            _inverse_layer(psi, circuit, i, mats)
            _inverse_layer(lam, circuit, i, mats)
            for j in range(len(pos)):
                pj = par[j] if par.ndim == 2 else par[:, j]
                m = coupling(lam, psi, bits[j])
                for kk in range(k):
                    v = dagger(mats[j]) @ gate_derivative(name, pj, kk).astype(dtype)
                    out[:, j, kk] = _contract(v, m)
        else:
            # descending rule: peel gate by gate
            for j in range(len(pos) - 1, -1, -1):
                pj = par[j] if par.ndim == 2 else par[:, j]
                apply_gate(psi, dagger(mats[j]), bits[j])
                m = coupling(lam, psi, bits[j])
                for kk in range(k):
                    dv = gate_derivative(name, pj, kk).astype(dtype)
                    out[:, j, kk] = _contract(dv, m)
                apply_gate(lam, dagger(mats[j]), bits[j])
        flat = out.reshape(batch, -1)
        if s[0] == "trainable":
            grads[:, s[1] : s[1] + s[2]] = flat
        else:
            egrads[:, s[1] : s[1] + s[2]] = flat
    value = (np.abs(final) ** 2) @ d
    return value, grads, egrads


def gradient(circuit, trainable=None, encoding=None, batch=1, weights=None, need_encoding=True,
             dtype=complex):
    """Forward from |0..0> then the adjoint sweep (reference grad.py:207-218).

    Returns dict(value (B,), zq (B,n), grads (B,T), encoding_grads (B,E))."""
    final = apply_circuit(circuit, trainable, encoding, batch=batch, dtype=dtype)
    value, g, eg = backward_sweep(circuit, trainable, encoding, final, weights, need_encoding, dtype)
    return {"value": value, "zq": expectation_z(final, circuit.n), "grads": g, "encoding_grads": eg}
