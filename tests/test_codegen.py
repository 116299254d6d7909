"""Host-side pieces of the specialised-kernel generator (codegen.py) that can be checked
without a GPU: the Walsh-component form of diagonal couplings, the shared-memory swizzle and
lane order, and that every config's kernels are generated."""

import numpy as np
import pytest

from paper_2506_04891_b200 import codegen, schedule as S
from paper_2506_04891_b200.configs import make_workload
from paper_2506_04891_b200.gates import gate_matrix, gate_matrix_derivative


def _diag_groups(cfg):
    wl = make_workload(cfg)
    prog = S.compile_circuit(wl.circuit, M=12 if wl.n > 12 else wl.n, R=4, prefix=True, fold=True, split=True)
    return [g for g in prog.groups if g.diag and g.needs_grad]


def _walsh(c, ar):
    return np.array([(-1) ** bin(c & e).count("1") for e in range(1 << ar)], float)


@pytest.mark.parametrize("cfg", [2, 5])
def test_diag_components_reproduce_gradients(cfg):
    """g_p = -2 sum_e a'_pe S_e computed from the kept Walsh components (constant component
    dropped, S' = 2^-ar sum_c V_c w_c) equals the class-sum form whenever sum_e S_e = 0
    (Im<lam|psi> = 0 over a row)."""
    rng = np.random.default_rng(7)
    groups = _diag_groups(cfg)
    assert groups
    for g in groups:
        comps = codegen.diag_components(g)
        ar = g.arity
        d = 1 << ar
        assert comps and 0 not in comps
        for _ in range(3):
            S_e = rng.normal(size=d)
            S_e -= S_e.mean()  # zero total: the row invariant
            V = {c: _walsh(c, ar) @ S_e for c in comps}
            S_p = sum(V[c] * _walsh(c, ar) for c in comps) / d
            prm = [float(rng.uniform(-3, 3)) for _ in g.gates[0][0].src]
            for gate, _ in g.gates:
                k = len(gate.src)
                p = prm[:k]
                G = np.diag(gate_matrix(gate.kind, p))
                for j in range(k):
                    dG = np.diag(gate_matrix_derivative(gate.kind, p, j))
                    ap = np.imag(dG / G)
                    np.testing.assert_allclose(-2 * ap @ S_p, -2 * ap @ S_e, atol=1e-12)


def test_diag_components_known_gates():
    comp = {}
    for cfg in (2, 5):
        for g in _diag_groups(cfg):
            comp[tuple(x.kind.value for x, _ in g.gates)] = codegen.diag_components(g)
    assert comp[("rz",)] == (1,)
    assert comp[("rzz",)] == (3,)


def test_swizzle_keeps_bit0_and_lanes_conflict_free():
    assert all(v % 2 == 0 and 0 < v < 16 for v in S.SWZ_H)
    for cfg, M in ((2, 11), (3, 12), (4, 12), (5, 12)):
        wl = make_workload(cfg)
        prog = S.compile_circuit(wl.circuit, M=M, R=4, prefix=True, fold=True, split=True)
        for pp in prog.passes:
            for ph in pp.phases:
                lanes = ph.threads[:4]
                if 0 in ph.regs:  # 16-byte pairs: 8 lanes per wavefront need 8 distinct slots
                    vec = [S.swz_vec(b) & 14 for b in lanes[:3]]
                else:  # 8-byte accesses: 16 lanes need 16 distinct slots
                    vec = [S.swz_vec(b) for b in lanes]
                slots = {np.bitwise_xor.reduce([v for j, v in enumerate(vec) if (m >> j) & 1] or [0])
                         for m in range(1 << len(vec))}
                assert len(slots) == 1 << len(vec), (cfg, ph)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_kernels_generate(cfg):
    wl = make_workload(cfg)
    M = 12 if wl.n > 12 else None
    prog = S.compile_circuit(wl.circuit, M=M, R=4 if M else None, prefix=True, fold=True, split=True)
    ks = codegen.generate_kernels(prog)
    names = {k[2] for k in ks}
    L = len(prog.passes)
    assert len(names) == 2 * L  # forward per pass, adjoint per pass but the last, turnaround
    for _, _, name, src, _ in ks:
        assert f"void __launch_bounds__" in src and name in src
