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


_HOST_PRELUDE = r"""
#include <cstdio>
#include <cstdlib>
struct float2 { float x, y; };
static inline float2 make_float2(float x, float y) { float2 r; r.x = x; r.y = y; return r; }
static inline float2 fx(float2 x, float s, float2 a) { return make_float2(a.x + s * x.x, a.y + s * x.y); }
static inline float2 mx(float2 x, float s) { return make_float2(s * x.x, s * x.y); }
static inline float2 fix(float2 x, float s, float2 a) { return make_float2(a.x - s * x.y, a.y + s * x.x); }
static inline float2 cm(float ar, float ai, float2 x) { return fix(x, ai, mx(x, ar)); }
"""


def _euler_entry(U):
    """floats 8..13 of a one-qubit group-table entry (csrc/lsq_common.cuh group_table_entry)"""
    c = abs(U[0, 0])
    ea = U[1, 0] * np.conj(U[0, 0])
    ea /= abs(ea)
    eg = U[1, 1] * np.conj(U[0, 0]) / c**2 * np.conj(ea)
    return [c, abs(U[1, 0]) / c, ea.real, ea.imag, eg.real, eg.imag]


@pytest.mark.parametrize("dagger", [False, True])
@pytest.mark.parametrize("bits", [(0, 1, 2, 3), (2, 0), (3, 1, 0)])
def test_euler_merged_block_on_host(tmp_path, bits, dagger):
    """The emitted merged Euler block (codegen._emit_euler_merged), compiled as host C++ with
    scalar stand-ins of the packed primitives, equals the product of the groups' unitaries
    (global phases dropped, deferred scale P.sc) on random vectors."""
    import shutil
    import subprocess
    import types

    if shutil.which("g++") is None:
        pytest.skip("no host compiler")
    wl = make_workload(4)
    prog = S.compile_circuit(wl.circuit, M=12, R=4, prefix=True, fold=True, split=True)
    cand = [g for g in prog.groups if g.arity == 1 and not g.diag and not g.prefix
            and codegen.u00_const_mag(g) is not None and len(g.gates) == 3]
    grps = cand[: len(bits)]
    assert len(grps) == len(bits)
    rng = np.random.default_rng(5)
    R, nvec = 4, 2
    P = types.SimpleNamespace(NR=1 << R, R=R, sc=[1.0, 1.0], prog=prog)
    run = [[S.OP_U1, b, -1, g.gid, -1, 16 * gi, 0, 0] for gi, (b, g) in enumerate(zip(bits, grps))]
    w = codegen._W()
    codegen._emit_euler_merged(w, P, run, nvec, dagger)
    # group tables from random parameters
    smat, Us = [], []
    for g in grps:
        U = np.eye(2, dtype=complex)
        for gate, _ in g.gates:
            k = len(gate.src)
            U = (gate_matrix(gate.kind, [float(rng.uniform(-3, 3)) for _ in range(k)]) if k
                 else gate_matrix(gate.kind)) @ U
        ent = [0.0] * 16
        for e in range(4):
            ent[2 * e], ent[2 * e + 1] = U.flat[e].real, U.flat[e].imag
        ent[8:14] = _euler_entry(U)
        smat += ent
        Us.append(U * np.exp(-1j * np.angle(U[0, 0])))  # global phase dropped
    v = rng.normal(size=(nvec, 1 << R)) + 1j * rng.normal(size=(nvec, 1 << R))
    init = "\n".join(f"v[{q}][{i}] = make_float2({float(v[q, i].real)!r}f, {float(v[q, i].imag)!r}f);"
                     for q in range(nvec) for i in range(1 << R))
    src = (_HOST_PRELUDE + f"int main() {{ float s_mat[{len(smat)}] = {{{', '.join(repr(float(np.float32(x))) + 'f' for x in smat)}}};\n"
           f"float2 v[{nvec}][{1 << R}];\n{init}\n" + "\n".join(w.lines) +
           f"\nfor (int q = 0; q < {nvec}; ++q) for (int i = 0; i < {1 << R}; ++i) printf(\"%.9g %.9g\\n\", v[q][i].x, v[q][i].y);\nreturn 0; }}\n")
    (tmp_path / "m.cpp").write_text(src)
    subprocess.run(["g++", "-O1", "-o", str(tmp_path / "m"), str(tmp_path / "m.cpp")], check=True)
    out = subprocess.run([str(tmp_path / "m")], check=True, capture_output=True, text=True).stdout.split()
    got = np.array(out, float).reshape(nvec, 1 << R, 2)
    got = got[..., 0] + 1j * got[..., 1]
    ref = v.copy()
    for b, U in zip(bits, Us):
        A = np.conj(U.T) if dagger else U
        t = ref.reshape(nvec, 1 << (R - 1 - b), 2, 1 << b)  # register bit b of the index
        ref = np.einsum("ij,qxjy->qxiy", A, t).reshape(nvec, 1 << R)
    for q in range(nvec):
        np.testing.assert_allclose(got[q] / P.sc[q], ref[q], atol=2e-5)


@pytest.mark.parametrize("seed", [3, 7])
def test_kernels_generate_for_random_hardware_style_circuits(seed):
    """Kernel generation (no compile) over the randomised IBM / IonQ / VQ-style circuits of the
    GPU stress run (profiles/stress_structured.py), with the engine's compile settings. Seed 3
    holds the case that broke the merged Euler runs on the GPU box: ECR applied twice on one pair
    is an identity permutation that emits no op, so two groups of one wire become neighbours."""
    import importlib.util
    import os

    from paper_2506_04891_b200.engine import forward_program

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "stress_structured.py")
    spec = importlib.util.spec_from_file_location("stress_structured", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.rng = np.random.default_rng(seed)
    kw = dict(prefix=True, fold=True, split=True)
    for _ in range(14):
        fam, circ, n, M, B = mod.draw_case()
        mod.rng.uniform(-3, 3, circ.trainable_count)  # keep the stress run's draw order
        mod.rng.uniform(0, 3, (B, circ.encoding_count))
        mod.rng.normal(size=n)
        prog = S.compile_circuit(circ, M=M, R=S.DEFAULT_R_SPECIALISED if M >= 9 else S.default_r(M), **kw)
        pf = forward_program(circ, prog, M=M, isolate=(), direct=(), split_layers=(), **kw)
        ks = codegen.kernel_set(prog, pf)
        assert len(ks) == 2 * len(prog.passes)
