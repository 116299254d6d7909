"""Per-circuit CUDA code generation: one straight-line sm_100a kernel per (pass, mode).

A kernel that interprets the op words at run time (round 1's generic kernel, since removed)
dispatches over run-time register indices, which makes the compiler copy the whole
64-register amplitude tile at every op (ncu: 54% of executed instructions were MOVs). Here
the schedule is emitted as straight-line code compiled by NVRTC for sm_100a at program
creation, so that

* register-bit indices, tile layouts and global/shared offsets are compile-time constants;
* permutation groups (CNOT, SWAP, X chains) become pure register renames (zero
  instructions);
* parameter-free groups (SX, ECR, MS(0,0,1/4), H, ...) use immediate matrix entries, so
  structural zeros cost nothing;
* a diagonal run accumulates fixed-point phases with compile-time index selection.

The emitted kernels share one launch contract (PassArgs, modes, flags, partial buffers,
csrc/lsq_prims.cuh) with the C-ABI drivers; the CPU emulator (tests/emulator.py) interprets
the same program words.
"""

from __future__ import annotations

import os

import numpy as np

from . import schedule as S
from .gates import GATE_TRAITS

_HERE = os.path.dirname(os.path.abspath(__file__))
PRIMS = os.path.join(_HERE, "csrc", "lsq_prims.cuh")

MODE_FWD, MODE_TURN, MODE_BWD = 0, 1, 2


def kernel_name(pi: int, mode: int) -> str:
    return f"lsq_jit_p{pi}_m{mode}"


def _f(x: float) -> str:
    return repr(float(np.float32(x))) + "f"


def _cexpr(coefs, xs):
    """Real/imag expressions of sum_c coefs[c] * xs[c] with constant complex coefs;
    zero terms dropped, +-1 folded."""
    re_terms, im_terms = [], []
    for cf, x in zip(coefs, xs):
        a, b = float(np.real(cf)), float(np.imag(cf))
        if abs(a) > 1e-15:
            re_terms.append(_term(a, f"{x}.x"))
            im_terms.append(_term(a, f"{x}.y"))
        if abs(b) > 1e-15:
            re_terms.append(_term(-b, f"{x}.y"))
            im_terms.append(_term(b, f"{x}.x"))
    return _sum(re_terms), _sum(im_terms)


def _term(c, v):
    if abs(c - 1.0) < 1e-15:
        return ("+", v)
    if abs(c + 1.0) < 1e-15:
        return ("-", v)
    return ("+", f"{_f(c)}*{v}")


def _sum(terms):
    if not terms:
        return "0.f"
    out = ""
    for i, (sg, t) in enumerate(terms):
        if i == 0:
            out = t if sg == "+" else f"-{t}"
        else:
            out += f" {sg} {t}"
    return out


class _Pass:
    """Compile-time view of one pass for code emission."""

    def __init__(self, prog, pi):
        self.prog = prog
        self.pi = pi
        self.pp = prog.passes[pi]
        self.M = self.pp.M
        self.R = self.pp.R
        self.NT = 1 << (self.M - self.R)
        self.NR = 1 << self.R
        self.NW = (self.NT + 31) // 32
        self.n = prog.n
        self.pbit = list(self.pp.phys_of_local)
        self.nbit = [p for p in range(self.n) if p not in set(self.pbit)]
        self.enc = prog.enc[pi]

    def goff(self, ph, i):
        regs = self.pp.phases[ph].regs
        return sum(1 << self.pbit[regs[k]] for k in range(self.R) if (i >> k) & 1)

    def soff(self, ph, i):
        regs = self.pp.phases[ph].regs
        loc = sum(1 << regs[k] for k in range(self.R) if (i >> k) & 1)
        return S_swz(loc)


def S_swz(L: int) -> int:
    h = 0
    for j, v in enumerate(S.SWZ_H):
        if (L >> (4 + j)) & 1:
            h ^= v
    return L ^ h


# ----------------------------------------------------------------------------------------- emit


class _W:
    def __init__(self):
        self.lines = []
        self.ind = 1

    def __call__(self, s=""):
        self.lines.append("  " * self.ind + s if s else "")

    def block(self, head):
        self(head + " {")
        self.ind += 1

    def end(self, tail=""):
        self.ind -= 1
        self("}" + tail)


def phase_normalized(U):
    """U times the global phase that makes its largest entry real positive (SX -> X90 with
    real diagonal and imaginary off-diagonal entries)."""
    k = np.unravel_index(np.argmax(np.abs(U)), U.shape)
    return U * np.exp(-1j * np.angle(U[k]))


def _group_const_matrix(grp, drop_phase=False):
    """Compile-time matrix of a group whose parameters are all FIXED (or absent). Gradient
    programs (folded observable, no state returned) drop its global phase: <Z_q> and every
    coupling conj(lam) psi are invariant under a common phase of psi and lam = O psi."""
    if any(s != S.FIXED_SRC for g, _ in grp.gates for s in g.src):
        return None
    U = S.group_matrix_host(grp)
    return phase_normalized(U) if drop_phase else U


def _emit_const_u(w, P, v, U, regs_bits, dagger):
    """Constant-matrix group on register bits (list of reg indices, first = MSB)."""
    if dagger:
        U = np.conj(U.T)
    d = U.shape[0]
    R = P.R
    if d == 2:
        (k,) = regs_bits
        for i in range(1 << R):
            if (i >> k) & 1:
                continue
            q = [i, i | (1 << k)]
            _emit_small(w, v, U, q)
    else:
        ka, kb = regs_bits
        for i in range(1 << R):
            if ((i >> ka) & 1) or ((i >> kb) & 1):
                continue
            q = [i, i | (1 << kb), i | (1 << ka), i | (1 << ka) | (1 << kb)]
            _emit_small(w, v, U, q)


_PAULI = {
    "I": np.eye(2, dtype=complex),
    "X": np.array([[0, 1], [1, 0]], dtype=complex),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=complex),
    "Z": np.array([[1, 0], [0, -1]], dtype=complex),
}
_STRUCT_CACHE: dict = {}


def u1_structure(grp, samples: int = 4):
    """Structure of a one-qubit group over its parameters (drawn at random; FIXED ones kept):

    * classes[a][b] of U: '0' (always zero), 'r' (real), 'i' (imaginary) or 'c' (complex);
    * comps: Pauli components P of K = i W that are nonzero for some parameter, W = the
      anti-Hermitian derivative weight (G_s..G_j+1) dG_j (G_j-1..G_1) U^+ of any free parameter.
    Only these entries are multiplied and only these components are accumulated."""
    from .gates import gate_matrix, gate_matrix_derivative

    key = tuple((g.kind, tuple(g.src), tuple(g.fixed)) for g, _ in grp.gates)
    if key in _STRUCT_CACHE:
        return _STRUCT_CACHE[key]
    rng = np.random.default_rng(12345)
    re_nz = np.zeros((2, 2), bool)
    im_nz = np.zeros((2, 2), bool)
    comps = set()
    for _ in range(samples):
        mats, ders = [], []
        for g, _rev in grp.gates:
            k = GATE_TRAITS[g.kind].param_count
            if k == 0:
                mats.append(gate_matrix(g.kind))
                ders.append([])
                continue
            prm = [g.fixed[j] if g.src[j] == S.FIXED_SRC else float(rng.uniform(-3.0, 3.0)) for j in range(k)]
            mats.append(gate_matrix(g.kind, prm))
            ders.append([gate_matrix_derivative(g.kind, prm, j) for j in range(k) if g.src[j] != S.FIXED_SRC])
        U = np.eye(2, dtype=complex)
        for G in mats:
            U = G @ U
        tol = 1e-12 * max(1.0, np.abs(U).max())
        re_nz |= np.abs(U.real) > tol
        im_nz |= np.abs(U.imag) > tol
        for j, dl in enumerate(ders):
            before = np.eye(2, dtype=complex)
            for G in mats[:j]:
                before = G @ before
            after = np.eye(2, dtype=complex)
            for G in mats[j + 1:]:
                after = G @ after
            for dG in dl:
                K = 1j * (after @ dG @ before @ U.conj().T)
                for nm, Pm in _PAULI.items():
                    if abs(np.trace(Pm @ K)) / 2 > 1e-9:
                        comps.add(nm)
    classes = [["0" if not (re_nz[a, b] or im_nz[a, b]) else
                "c" if (re_nz[a, b] and im_nz[a, b]) else ("r" if re_nz[a, b] else "i")
                for b in range(2)] for a in range(2)]
    out = (classes, frozenset(comps))
    _STRUCT_CACHE[key] = out
    return out


def coupling_layout(comps):
    """[(component, slot position)] of the anti-Hermitian projected coupling M' (see
    u1_coupling_h): Z -> M'00.y, X -> M'01.y, Y -> M'10.x; with a trace component the diagonal
    is kept as A = Im c00 -> M'00.y and B = Im c11 -> M'11.y."""
    lay = []
    if "I" in comps:
        lay += [("A", 1), ("B", 7)]
    elif "Z" in comps:
        lay.append(("Z", 1))
    if "X" in comps:
        lay.append(("X", 3))
    if "Y" in comps:
        lay.append(("Y", 4))
    return lay


# (function, l index, p index) pairs per component: value = sum_pairs (acc.x + acc.y)
_COMP_TERMS = {
    "Z": (("_mj", "i", "i"), ("_j", "j", "j")),
    "X": (("_mj", "i", "j"), ("_mj", "j", "i")),
    "Y": (("_p", "j", "i"), ("_n", "i", "j")),
    "A": (("_mj", "i", "i"),),
    "B": (("_mj", "j", "j"),),
}


def _tree_sum(terms):
    """Balanced addition tree (fp adds are not reassociated by the compiler: a left-leaning
    chain of 15 adds is 15 dependent latencies, the tree 4)."""
    terms = list(terms)
    if not terms:
        return "0.f"
    while len(terms) > 1:
        nxt = [f"({terms[q]} + {terms[q + 1]})" for q in range(0, len(terms) - 1, 2)]
        if len(terms) % 2:
            nxt.append(terms[-1])
        terms = nxt
    return terms[0]


COUPLING_CHAINS = int(os.environ.get("LSQ_COUPLING_CHAINS", "1"))  # partial sums per component: 1 measured best (registers beat ILP)


def _emit_u1_coupling(w, P, k, slot, comps):
    lay = coupling_layout(comps)
    if not lay:
        return
    names = [P.coup.new(w) for _ in lay]
    w("{")
    w.ind += 1
    pairs = [(i, i | (1 << k)) for i in range(1 << P.R) if not (i >> k) & 1]
    nch = max(1, min(COUPLING_CHAINS, len(pairs)))
    for ci, (nm, _pos) in enumerate(lay):
        accs = [None] * nch
        for pi, (i, j) in enumerate(pairs):
            idx = {"i": i, "j": j}
            c = pi % nch
            for fn, li, pi_ in _COMP_TERMS[nm]:
                a, b = f"v[1][{idx[li]}]", f"v[0][{idx[pi_]}]"
                accs[c] = f"vm{fn}({a}, {b})" if accs[c] is None else f"vf{fn}({a}, {b}, {accs[c]})"
        for c in range(nch):
            w(f"const float2 t{ci}_{c} = {accs[c]};")
        w(f"{names[ci]} = {_scaled(P, _tree_sum([f't{ci}_{c}.x' for c in range(nch)] + [f't{ci}_{c}.y' for c in range(nch)]))};")
    w.ind -= 1
    w("}")
    used = {pos for _, pos in lay}
    free = [slot + q for q in range(8) if q not in used]
    for ci, (nm, pos) in enumerate(lay):
        P.coup.add(w, names[ci], slot + pos, free)


EULER_COUP = os.environ.get("LSQ_EULER_COUP", "1") != "0"


def _pi1_chain(P, k):
    """Packed chain whose .x + .y is sum over the pairs of register bit k of
    Im(conj(lam_j) psi_j), j the member with the bit set: one FFMA2 per pair."""
    acc = None
    for i in range(1 << P.R):
        if (i >> k) & 1:
            continue
        j = i | (1 << k)
        a, b = f"v[1][{j}]", f"v[0][{j}]"
        acc = f"vm_mj({a}, {b})" if acc is None else f"vf_mj({a}, {b}, {acc})"
    return acc


def _emit_euler_coupling_post(w, P, k):
    """Couplings of a one-qubit group U = e^{id} D(a) R D(g) (D(x) = diag(1, e^{ix}), R a fixed
    rotation: |U00| the same for every parameter value) taken at the Euler points instead of as
    three Pauli components at the post-group point. Every derivative weight is
    W = i (d' I + a' Pi1 + g' U Pi1 U^+), Pi1 = |1><1|, so the gradient only needs
    P1 = Im <lam|Pi1|psi> after the group and Q1 = the same before it (where U Pi1 U^+ is Pi1
    again): one FFMA2 per amplitude pair each, against six for the X, Y, Z components. This
    part takes P1 (before the group is un-applied); _emit_euler_coupling_pre finishes."""
    names = [P.coup.new(w) for _ in range(3)]
    w(f"{{ const float2 t_ = {_pi1_chain(P, k)}; {names[0]} = {_scaled(P, '(t_.x + t_.y)')}; }}")
    return names


def _emit_euler_coupling_pre(w, P, k, slot, names, g, cmag):
    """Q1 at the pre-group point, then the equivalent M' = [[i Z', i s], [t, 0]] the contraction
    reads (slot floats 1, 3, 4, the layout of the X, Y, Z components): Z' = -2 P1 (Im<lam|psi>
    = 0 over the row), (s, t) = mu (Re z, -Im z) with z = U01 conj(U11) and
    mu = (Q1 - (|U11|^2 - |U01|^2) P1) / |z|^2, which reproduces 2 Re sum W_ab M_ab =
    -2 (a' P1 + g' Q1) for every weight of the form above. |U11| = |U00| = cmag."""
    c2 = float(cmag) ** 2
    dz, zz = c2 - (1.0 - c2), c2 * (1.0 - c2)
    w(f"{{ const float2 t_ = {_pi1_chain(P, k)}; const float q_ = {_scaled(P, '(t_.x + t_.y)')};")
    q = "q_" if abs(dz) < 1e-12 else f"(q_ - {_f(dz)} * {names[0]})"
    w(f"  const float mu_ = {q} * {_f(1.0 / zz)};")
    w(f"  {names[1]} = mu_ * ({g}[2] * {g}[6] + {g}[3] * {g}[7]);")
    w(f"  {names[2]} = mu_ * ({g}[2] * {g}[7] - {g}[3] * {g}[6]);")
    w(f"  {names[0]} *= -2.f; }}")
    free = [slot + q_ for q_ in range(8) if q_ not in (1, 3, 4)]
    for nm, pos in zip(names, (1, 3, 4)):
        P.coup.add(w, nm, slot + pos, free)


def _emit_u1_struct(w, v, k, R, classes, g, dagger):
    """U (or U^+) from the table entry g (row-major re, im) on register bit k, emitting only
    the terms the structure allows: real entry -> one FFMA2, imaginary -> one FFMA2 on i x,
    complex -> two, zero -> none."""
    for i in range(1 << R):
        if (i >> k) & 1:
            continue
        j = i | (1 << k)
        w(f"{{ const float2 x0 = {v}[{i}], x1 = {v}[{j}];")
        for a, dst in ((0, i), (1, j)):
            expr = None
            for b in (0, 1):
                ra, cb = (b, a) if dagger else (a, b)  # U^+_ab = conj(U_ba)
                cls = classes[ra][cb]
                e = 2 * ra + cb
                re, im = f"{g}[{2 * e}]", f"{g}[{2 * e + 1}]"
                if cls in ("r", "c"):
                    expr = f"mx(x{b}, {re})" if expr is None else f"fx(x{b}, {re}, {expr})"
                if cls in ("i", "c"):
                    if dagger:
                        expr = f"mulmix(x{b}, {im})" if expr is None else f"fmix(x{b}, {im}, {expr})"
                    else:
                        expr = f"mulix(x{b}, {im})" if expr is None else f"fix(x{b}, {im}, {expr})"
            w(f"  {v}[{dst}] = {expr if expr else 'make_float2(0.f, 0.f)'};")
        w("}")


def _emit_small(w, v, U, q):
    """Constant complex matrix on packed f32x2: per nonzero coefficient at most two FFMA2
    (real part times x, imaginary part times i*x); zero halves are skipped."""
    d = len(q)
    w("{ " + " ".join(f"const float2 x{c} = {v}[{q[c]}];" for c in range(d)))
    for r in range(d):
        expr = None
        for c in range(d):
            a, b = float(np.real(U[r, c])), float(np.imag(U[r, c]))
            for coef, kind in ((a, "x"), (b, "ix")):
                if abs(coef) < 1e-15:
                    continue
                if expr is None:
                    expr = f"{'mx' if kind == 'x' else 'mulix'}(x{c}, {_f(coef)})"
                else:
                    expr = f"{'fx' if kind == 'x' else 'fix'}(x{c}, {_f(coef)}, {expr})"
        w(f"  {v}[{q[r]}] = {expr if expr else 'make_float2(0.f, 0.f)'};")
    w("}")


UNIT_CONST = os.environ.get("LSQ_UNIT_CONST", "1") != "0"


def unit_form(U):
    """(kappa, U / kappa) when every nonzero entry of the constant matrix U has modulus kappa
    and U / kappa has entries in {0, +-1, +-i} (MS(0,0), ECR, H, X90 ...); else None."""
    mags = np.abs(U[np.abs(U) > 1e-12])
    if mags.size == 0:
        return None
    kappa = float(mags.max())
    if np.any(np.abs(mags - kappa) > 1e-9 * kappa):
        return None
    V = U / kappa
    ok = (np.abs(V) < 1e-12) | (np.abs(V - 1) < 1e-9) | (np.abs(V + 1) < 1e-9) | \
         (np.abs(V - 1j) < 1e-9) | (np.abs(V + 1j) < 1e-9)
    if not ok.all() or abs(kappa - 1.0) < 1e-12:
        return None
    return kappa, np.round(V.real) + 1j * np.round(V.imag)


def _emit_unit_small(w, v, V, q):
    """Constant matrix with entries in {0, +-1, +-i} (the scale is deferred): an output row with
    a +1 entry starts from that amplitude (no multiply) and adds the others with one FFMA2 each
    (coefficient +-1 on x or on i x); rows without a +1 entry fall back to one multiply."""
    d = len(q)
    w("{ " + " ".join(f"const float2 x{c} = {v}[{q[c]}];" for c in range(d)))
    for r in range(d):
        terms = [(c, complex(V[r, c])) for c in range(d) if abs(V[r, c]) > 0.5]
        first = next((t for t in terms if abs(t[1] - 1) < 1e-9), None)
        if first is not None:
            expr = f"x{first[0]}"
            rest = [t for t in terms if t is not first]
        else:
            c0, a = terms[0]
            expr = f"mx(x{c0}, {_f(a.real)})" if abs(a.imag) < 0.5 else f"mulix(x{c0}, {_f(a.imag)})"
            rest = terms[1:]
        for c, a in rest:
            if abs(a.imag) < 0.5:
                expr = f"fx(x{c}, {_f(a.real)}, {expr})"
            else:
                expr = f"fix(x{c}, {_f(a.imag)}, {expr})"
        w(f"  {v}[{q[r]}] = {expr if terms else 'make_float2(0.f, 0.f)'};")
    w("}")


def _emit_unit_const(w, P, v, V, regs_bits, dagger):
    if dagger:
        V = np.conj(V.T)
    R = P.R
    if V.shape[0] == 2:
        (k,) = regs_bits
        for i in range(1 << R):
            if not (i >> k) & 1:
                _emit_unit_small(w, v, V, [i, i | (1 << k)])
    else:
        ka, kb = regs_bits
        for i in range(1 << R):
            if not ((i >> ka) & 1) and not ((i >> kb) & 1):
                _emit_unit_small(w, v, V, [i, i | (1 << kb), i | (1 << ka), i | (1 << ka) | (1 << kb)])


def _scaled(P, expr, q=(0, 1)):
    """expr times the deferred scales of the vectors in q: the compile-time 1/sc of unit-form
    constant gates and the run-time rho_ of tangent-form rotations (true = computed x rho_)."""
    c = 1.0
    for i in q:
        c /= P.sc[i]
    nr = sum(1 for i in q if P.rho_live)
    out = expr
    if abs(c - 1.0) >= 1e-15:
        out = f"(({out}) * {_f(c)})"
    if nr:
        out = f"(({out}) * {' * '.join(['rho_'] * nr)})"
    return out


TAN_ROT = os.environ.get("LSQ_TAN_ROT", "1") != "0"
TAN_TH = 0.01  # |cos| below this: the rotation takes the two-op form
TAN_RENORM = 8  # tangent-form rotations between forced renormalisations (range guard)
_ROT_CACHE: dict = {}


def is_rotation(grp) -> bool:
    """One-qubit group whose matrix is a real rotation [[c, -s], [s, c]] for all parameters
    (RY and products of RY): applied in tangent form (see _emit_tan_rot)."""
    from .gates import gate_matrix

    if grp.arity != 1:
        return False
    key = tuple((g.kind, tuple(g.src), tuple(g.fixed)) for g, _ in grp.gates)
    if key in _ROT_CACHE:
        return _ROT_CACHE[key]
    rng = np.random.default_rng(99)
    ok = True
    for _ in range(3):
        U = np.eye(2, dtype=complex)
        for g, _r in grp.gates:
            k = GATE_TRAITS[g.kind].param_count
            prm = [g.fixed[j] if g.src[j] == S.FIXED_SRC else float(rng.uniform(-3.0, 3.0)) for j in range(k)]
            U = (gate_matrix(g.kind, prm) if k else gate_matrix(g.kind)) @ U
        if np.abs(U.imag).max() > 1e-12 or abs(U[0, 0] - U[1, 1]) > 1e-12 or abs(U[0, 1] + U[1, 0]) > 1e-12:
            ok = False
    _ROT_CACHE[key] = ok
    return ok


def _emit_tan_rot(w, P, k, g, nvec, dagger, classes):
    """Rotation R = [[c, -s], [s, c]] on register bit k as R / c = [[1, -t], [t, 1]]: one FFMA2
    per output amplitude instead of two; the vectors carry the run-time scale rho_ *= c
    (uniform over the block: the angle is shared or per row). |c| < TAN_TH keeps the two-op
    form (uniform branch)."""
    w(f"{{ const float c_ = {g}[0], t_ = __fdividef({g}[4], {g}[0]), nt_ = -t_;")
    w(f"if (fabsf(c_) >= {TAN_TH}f) {{")
    a0, a1 = ("t_", "nt_") if dagger else ("nt_", "t_")  # R^+/c = [[1, t], [-t, 1]]
    for q in range(nvec):
        for i in range(1 << P.R):
            if (i >> k) & 1:
                continue
            j = i | (1 << k)
            w(f"  {{ const float2 x0 = v[{q}][{i}], x1 = v[{q}][{j}]; "
              f"v[{q}][{i}] = fx(x1, {a0}, x0); v[{q}][{j}] = fx(x0, {a1}, x1); }}")
    w("  rho_ *= c_;")
    w("} else {")
    for q in range(nvec):
        _emit_u1_struct(w, f"v[{q}]", k, P.R, classes, g, dagger)
    w("} }")
    P.rho_live = True
    P.tan_count += 1


EULER_TAN = os.environ.get("LSQ_EULER_TAN", "1") != "0"
# groups whose |U00| varies with the parameters need the uniform fallback branch (adjoint only)
EULER_BRANCH = os.environ.get("LSQ_EULER_BRANCH", "0") == "1"  # measured: cfg5 277 vs 279 evals/s with it
_MAG_CACHE: dict = {}


def u00_const_mag(grp, samples: int = 6):
    """|U00| of a one-qubit group when it is the same for every parameter value (RZ.SX.RZ,
    GPI2.GPI: 1/sqrt2), else None. Such groups take the Euler tangent form without a branch."""
    from .gates import gate_matrix

    key = tuple((g.kind, tuple(g.src), tuple(g.fixed)) for g, _ in grp.gates)
    if key in _MAG_CACHE:
        return _MAG_CACHE[key]
    rng = np.random.default_rng(4321)
    mags = []
    for _ in range(samples):
        U = np.eye(2, dtype=complex)
        for g, _r in grp.gates:
            k = GATE_TRAITS[g.kind].param_count
            prm = [g.fixed[j] if g.src[j] == S.FIXED_SRC else float(rng.uniform(-3.0, 3.0)) for j in range(k)]
            U = (gate_matrix(g.kind, prm) if k else gate_matrix(g.kind)) @ U
        mags.append(abs(U[0, 0]))
    m = mags[0] if (max(mags) - min(mags) < 1e-9 and mags[0] >= 0.1) else None
    _MAG_CACHE[key] = m
    return m


def _emit_euler_tan(w, P, k, g, nvec, dagger, classes, branch):
    """General one-qubit group U = e^{i d} diag(1, e^{ia}) R(b) diag(1, e^{ig}) (R = [[c, -s],
    [s, c]], global phase dropped: gradient programs only) on register bit k, with the rotation
    in tangent form R / c = [[1, -t], [t, 1]]: per pair a phase on one member, two single-FFMA2
    outputs and a phase on one output -- 6 packed ops instead of 8; the vectors carry the
    run-time scale rho_ *= c = |U00|. Adjoint: U^+ = diag(1, e^{-ig}) R(-b) diag(1, e^{-ia}).
    The group table entry holds U (floats 0..7, row-major re, im) and, from the fp64 group-table
    kernel (lsq_common.cuh group_table_entry), c, t, e^{ia}, e^{ig} (floats 8..13). `branch`:
    |U00| may vanish, so c < TAN_TH takes the direct form (uniform branch)."""
    w(f"{{ const float c_ = {g}[8], t_ = {g}[9], nt_ = -t_;")
    w(f"  const float2 ea_ = make_float2({g}[10], {g}[11]), eg_ = make_float2({g}[12], {g}[13]);")
    if branch:
        w(f"  if (c_ >= {TAN_TH}f) {{")
    for q in range(nvec):
        for i in range(1 << P.R):
            if (i >> k) & 1:
                continue
            j = i | (1 << k)
            if not dagger:
                w(f"    {{ const float2 x0 = v[{q}][{i}], x1 = cm(eg_.x, eg_.y, v[{q}][{j}]); "
                  f"v[{q}][{i}] = fx(x1, nt_, x0); v[{q}][{j}] = cm(ea_.x, ea_.y, fx(x0, t_, x1)); }}")
            else:
                w(f"    {{ const float2 x0 = v[{q}][{i}], x1 = cm(ea_.x, -ea_.y, v[{q}][{j}]); "
                  f"v[{q}][{i}] = fx(x1, t_, x0); v[{q}][{j}] = cm(eg_.x, -eg_.y, fx(x0, nt_, x1)); }}")
    w("    rho_ *= c_;")
    if branch:
        # the global phase e^{-i d} dropped here is tracked (phc_): the direct form of the else
        # branch, the forward kernels and the checkpoints keep it, so stored vectors must too
        w(f"    phc_ = cm({g}[14], {'-' if dagger else ''}{g}[15], phc_);")
        P.ph_live = True
        w("  } else {")
        for q in range(nvec):
            _emit_u1_struct(w, f"v[{q}]", k, P.R, classes, g, dagger)
        w("  }")
    w("}")
    P.rho_live = True
    P.tan_count += 1


# consecutive Euler-form one-qubit groups of a phase (a layer of RZ.SX.RZ / GPI2.GPI groups on
# the phase's register wires) applied with MERGED diagonal factors: minimum run length, 0 = off
EULER_MERGE = int(os.environ.get("LSQ_EULER_MERGE", "2"))
SC_GUARD = 1e12  # deferred compile-time scale above which the vectors are renormalised


def _emit_euler_merged(w, P, run, nvec, dagger):
    """A run of k Euler-form groups U_b = D_b(a_b) R_b D_b(g_b) (constant |U00|, see
    _emit_euler_tan) on DISTINCT register bits, applied as three commuting layers instead of k
    separate groups: the product of the pre-phases as ONE diagonal over the 2^k sub-indices of
    the run's bits (one complex multiply per amplitude, none for sub-index 0), the k tangent-form
    rotations (one FFMA2 per output), and the product of the post-phases as one diagonal.
    Separately every group costs a complex multiply on half the amplitudes twice, i.e. k complex
    multiplies per amplitude for the run; merged it is 2 (1 - 2^-k), plus the 2^k - 1 - k table
    products per diagonal, shared by psi and lambda. k = 4: 12 -> 7.75 (+ 1.4) packed ops per
    amplitude per vector. The scale |U00|^k is a compile-time constant (P.sc), so these groups
    need no run-time rho_. Adjoint: conj(post) first, R^+, conj(pre)."""
    k = len(run)
    bits = [int(op[1]) for op in run]
    assert len(set(bits)) == k, "merged Euler run on repeated register bits"
    w("{")
    w.ind += 1
    for gi, op in enumerate(run):
        w(f"const float* g{gi}_ = s_mat + {int(op[5])};")
        w(f"const float t{gi}_ = g{gi}_[9], nt{gi}_ = -t{gi}_;")

    def sub(i):
        return sum(((i >> bits[gi]) & 1) << gi for gi in range(k))

    def diagonal(name, fo, conj):
        """multiply amplitude i of every vector by prod_{b in sub(i)} e_b (conjugated in the
        adjoint); table entries are defined right before their first use, in sub-index order"""
        members = {}
        for i in range(P.NR):
            members.setdefault(sub(i), []).append(i)
        for s_ in range(1, 1 << k):
            top = s_.bit_length() - 1
            rest = s_ ^ (1 << top)
            if rest == 0:
                w(f"const float2 {name}{s_}_ = make_float2(g{top}_[{fo}], g{top}_[{fo + 1}]);")
            else:
                w(f"const float2 {name}{s_}_ = cm({name}{1 << top}_.x, {name}{1 << top}_.y, {name}{rest}_);")
            for q in range(nvec):
                for i in members[s_]:
                    w(f"v[{q}][{i}] = cm({name}{s_}_.x, {'-' if conj else ''}{name}{s_}_.y, v[{q}][{i}]);")

    # forward: pre-phases e^{ig} (floats 12, 13), adjoint: conj of the post-phases e^{ia} (10, 11)
    diagonal("ef", 10 if dagger else 12, dagger)
    for gi in range(k):
        a0, a1 = (f"t{gi}_", f"nt{gi}_") if dagger else (f"nt{gi}_", f"t{gi}_")
        for q in range(nvec):
            for i in range(P.NR):
                if (i >> bits[gi]) & 1:
                    continue
                j = i | (1 << bits[gi])
                w(f"{{ const float2 x0 = v[{q}][{i}], x1 = v[{q}][{j}]; "
                  f"v[{q}][{i}] = fx(x1, {a0}, x0); v[{q}][{j}] = fx(x0, {a1}, x1); }}")
    diagonal("el", 12 if dagger else 10, dagger)
    w.ind -= 1
    w("}")
    for op in run:
        cmag = u00_const_mag(P.prog.groups[int(op[3])])
        for q in range(nvec):
            P.sc[q] /= cmag  # applied U / |U00|: computed = true x sc
    _guard_scale(w, P, nvec)


def _guard_scale(w, P, nvec):
    """Fold a large deferred compile-time scale back into the amplitudes (range guard)."""
    for q in range(nvec):
        if P.sc[q] > SC_GUARD or P.sc[q] < 1.0 / SC_GUARD:
            for i in range(P.NR):
                w(f"v[{q}][{i}] = mx(v[{q}][{i}], {_f(1.0 / P.sc[q])});")
            P.sc[q] = 1.0


def _renorm_rho(w, P, nvec):
    """Multiply the run-time scale back into the amplitudes (range guard, branch merges)."""
    if not P.rho_live:
        return
    for q in range(nvec):
        for i in range(1 << P.R):
            w(f"v[{q}][{i}] = mx(v[{q}][{i}], rho_);")
    w("rho_ = 1.f;")
    P.rho_live = False
    P.tan_count = 0


def _src_expr(sw, P, tp_var):
    """(kind, expr) of a diagonal source: ('reg', k) or ('const', c-expression)."""
    kind, val = int(sw) >> 8, int(sw) & 0xFF
    if kind == S.SRC_REG:
        return "reg", val
    if kind == S.SRC_THREAD:
        return "const", f"(({tp_var} >> {val}) & 1u)"
    if kind == S.SRC_NONLOCAL:
        return "const", f"(int)((tbase >> {val}) & 1ull)"
    return "none", None


class _Coup:
    """Backward coupling values (anti-Hermitian projections, see u1_structure) packed four
    per half-block; two half-blocks share one 8-value warp reduce-scatter
    (warp_accumulate8p). Lane l owns value j = (l >> 2) & 3 of half (l >> 4) & 1 and adds it
    at a per-lane offset: an arithmetic progression o0 + d j when the offsets allow one
    (padding zeros go to free floats of the same slots or to the 8 padding floats after the
    slots), else a select chain."""

    def __init__(self, P):
        self.P = P
        self.n = 0
        self.vals = []  # pending (name, offset, free offsets)
        self.half = None  # pending complete half: (names[4], offsets[4])

    def new(self, w):
        name = f"cv{self.n}_"
        self.n += 1
        w(f"float {name};")
        return name

    def add(self, w, name, off, free):
        self.vals.append((name, off, tuple(free)))
        if len(self.vals) == 4:
            self._close(w)

    def flush(self, w):
        if self.vals:
            self._close(w)
        if self.half is not None:
            h, self.half = self.half, None
            self._emit(w, h, None)

    def _close(self, w):
        vals, self.vals = self.vals, []
        h = self._layout(vals)
        if self.half is None:
            self.half = h
        else:
            a, self.half = self.half, None
            self._emit(w, a, h)

    def _layout(self, vals):
        """(names[4], offsets[4], offset expression) of one half-block."""
        P = self.P
        reals = {off: nm for nm, off, _ in vals}
        nz = 4 - len(vals)
        pad = [P.slotf + q for q in range(8)]
        cand = sorted({f for _, _, fr in vals for f in fr} - set(reals)) + pad
        best = None
        if P.NT >= 32:
            for o0 in sorted(set(reals) | set(cand)):
                for d in (1, 2, 3, 4, 8, -1, -2, -4, -8):
                    offs = [o0 + d * q for q in range(4)]
                    if not set(reals) <= set(offs):
                        continue
                    zs = [o for o in offs if o not in reals]
                    if len(zs) == nz and all(z in cand for z in zs):
                        best = (offs, f"{o0} + {d} * lj_" if d != 1 else f"{o0} + lj_")
                        break
                if best:
                    break
            if best is None:
                for base in sorted({o - p for o in reals for p in (1, 3, 4, 7)}):
                    offs = [base + p for p in (1, 3, 4, 7)]
                    zs = [o for o in offs if o not in reals]
                    if set(reals) <= set(offs) and len(zs) == nz and all(z in cand for z in zs):
                        best = (offs, f"{base} + pu1_")
                        break
        if best is None:
            offs = list(reals) + pad[:nz]
            sel = f"(lj_ & 2 ? (lj_ & 1 ? {offs[3]} : {offs[2]}) : (lj_ & 1 ? {offs[1]} : {offs[0]}))"
            best = (offs, sel)
        offs, expr = best
        names = [reals.get(o, "0.f") for o in offs]
        return names, offs, expr

    def _emit(self, w, a, b):
        P = self.P
        vals = list(a[0]) + (list(b[0]) if b else ["0.f"] * 4)
        init = f"float a8_[8] = {{{', '.join(vals)}}};"
        if P.NT >= 32:
            eb = b[2] if b else f"{P.slotf} + lj_"
            w(f"{{ {init} warp_accumulate8p<NT>(a8_, wacc + (hi16_ ? {eb} : {a[2]})); }}")
        else:
            adds = [f"wacc[{o}] += a8_[{q}];" for q, (nm, o) in enumerate(zip(a[0], a[1])) if nm != "0.f"]
            if b:
                adds += [f"wacc[{o}] += a8_[{4 + q}];" for q, (nm, o) in enumerate(zip(b[0], b[1])) if nm != "0.f"]
            w(f"{{ {init} warp_sum<NT, 8>(a8_); if ((tid & 31) == 0) {{ {' '.join(adds)} }} }}")


_DIAG_COMP_CACHE: dict = {}


def diag_components(grp, samples: int = 3):
    """Nonzero Walsh components of a diagonal group's phase derivatives.

    G = diag(e^{i alpha_e}) over the 2^ar classes e (first wire = MSB). Every free parameter
    p has dalpha_p/dtheta = sum_c a_{p,c} w_c(e) with w_c(e) = (-1)^popc(c & e). The gradient
    is -2 sum_e alpha'_{p,e} S_e, S_e = sum over class e of Im(conj(lam) psi): it only needs
    the component sums V_c = sum_e w_c(e) S_e for the c with a_{p,c} != 0. The constant
    component c = 0 multiplies Im<lam|psi> over the row, which is 0 (lam and psi evolve under
    the same unitaries from lam = O psi with O Hermitian), so it is never accumulated."""
    from .gates import gate_matrix, gate_matrix_derivative

    key = tuple((g.kind, tuple(g.src), tuple(g.fixed), rev) for g, rev in grp.gates)
    if key in _DIAG_COMP_CACHE:
        return _DIAG_COMP_CACHE[key]
    d = 1 << grp.arity
    rng = np.random.default_rng(4321)
    comps = set()
    for _ in range(samples):
        mats, ders = [], []
        for g, rev in grp.gates:
            k = GATE_TRAITS[g.kind].param_count
            prm = [g.fixed[j] if g.src[j] == S.FIXED_SRC else float(rng.uniform(-3.0, 3.0)) for j in range(k)]
            G = np.diag(np.diag(gate_matrix(g.kind, prm) if k else gate_matrix(g.kind)))
            dl = [np.diag(np.diag(gate_matrix_derivative(g.kind, prm, j))) for j in range(k) if g.src[j] != S.FIXED_SRC]
            if rev and d == 4:  # gate given on (b, a): swap the two wires of the class index
                perm = [0, 2, 1, 3]
                G = G[np.ix_(perm, perm)]
                dl = [D[np.ix_(perm, perm)] for D in dl]
            mats.append(G)
            ders.append(dl)
        U = np.eye(d, dtype=complex)
        for G in mats:
            U = G @ U
        for j, dl in enumerate(ders):
            for dG in dl:
                full = np.eye(d, dtype=complex)
                for jj, G in enumerate(mats):
                    full = (dG if jj == j else G) @ full
                ap = np.imag(np.diag(full) / np.diag(U))  # alpha'_e
                for c in range(1, d):
                    wc = np.array([(-1) ** bin(c & e).count("1") for e in range(d)])
                    if abs(ap @ wc) / d > 1e-9:
                        comps.add(c)
    out = tuple(sorted(comps))
    _DIAG_COMP_CACHE[key] = out
    return out


def _emit_drun_walsh(w, P, subs, tp):
    """Diagonal couplings as Walsh component sums (see diag_components): per distinct
    register mask m one packed chain T_m = sum_i (-1)^popc(i & m) lam_i .* (psi_i.y, -psi_i.x),
    V = T.x + T.y; thread and tile bits of a component only flip its sign. Component c of a
    sub goes to slot float 2c - 1; the CTA epilogue (P.walsh) expands the components into the
    per-class values S'_e the contraction kernel reads."""
    R = P.R
    plan = []  # (sub index, slot, ar, comp, regmask, sign expressions)
    for si, s in enumerate(subs):
        slot = int(s[4])
        if slot < 0:
            continue
        grp = P.prog.groups[int(s[2])]
        ar = int(s[5])
        srcs = [_src_expr(s[0], P, tp)] + ([_src_expr(s[1], P, tp)] if ar == 2 else [])
        comps = diag_components(grp)
        for c in comps:
            regmask, signs = 0, []
            for q, (kind, e) in enumerate(srcs):
                bit = (c >> (ar - 1 - q)) & 1  # class index e = 2 a + b: wire a is the MSB
                if not bit:
                    continue
                if kind == "reg":
                    regmask ^= 1 << e
                else:
                    signs.append(e)
            plan.append((si, slot, ar, c, regmask, signs))
        P.walsh.append((slot, ar, comps))
    masks = sorted({pl[4] for pl in plan})
    names = [P.coup.new(w) for _ in plan]
    w("{")
    w.ind += 1
    nch = COUPLING_CHAINS
    for m in masks:
        accs = [None] * nch
        for i in range(P.NR):
            fn = "_j" if bin(i & m).count("1") & 1 else "_mj"
            c = i % nch
            accs[c] = f"vm{fn}(v[1][{i}], v[0][{i}])" if accs[c] is None else f"vf{fn}(v[1][{i}], v[0][{i}], {accs[c]})"
        for c in range(nch):
            w(f"const float2 wt{m}_{c} = {accs[c]};")
        w(f"const float wv{m} = {_scaled(P, _tree_sum([f'wt{m}_{c}.x' for c in range(nch)] + [f'wt{m}_{c}.y' for c in range(nch)]))};")
    for (si, slot, ar, c, regmask, signs), nm in zip(plan, names):
        if signs:
            par = " ^ ".join(f"(int)({e})" for e in signs)
            w(f"{nm} = (({par}) & 1) ? -wv{regmask} : wv{regmask};")
        else:
            w(f"{nm} = wv{regmask};")
    w.ind -= 1
    w("}")
    for (si, slot, ar, c, regmask, signs), nm in zip(plan, names):
        used = {slot + 2 * cc - 1 for cc in diag_components(P.prog.groups[int(subs[si][2])])}
        free = [slot + q for q in range(2 << ar) if slot + q not in used]
        P.coup.add(w, nm, slot + 2 * c - 1, free)

def _emit_drun(w, P, op, ph_idx, mode_bwd, nv, couplings=True, rotate=True):
    subs = P.enc["subs"][op[6] : op[6] + op[7]]
    tp = f"tp{ph_idx}"
    R = P.R
    # couplings (backward, before un-applying: conj(l) p is phase invariant)
    if not couplings:
        pass
    elif mode_bwd and any(int(s[4]) >= 0 for s in subs) and P.walsh_diag:
        _emit_drun_walsh(w, P, subs, tp)
    elif mode_bwd and any(int(s[4]) >= 0 for s in subs):
        names = {si: [P.coup.new(w) for _ in range(1 << int(s[5]))] for si, s in enumerate(subs) if int(s[4]) >= 0}
        w("{")
        w.ind += 1
        for i in range(P.NR):
            w(f"const float c{i} = v[1][{i}].x * v[0][{i}].y - v[1][{i}].y * v[0][{i}].x;  // Im conj(l) p")
        for si, s in enumerate(subs):
            slot = int(s[4])
            if slot < 0:
                continue
            nm = names[si]
            ka, ea = _src_expr(s[0], P, tp)
            kb, eb = _src_expr(s[1], P, tp)
            ar = int(s[5])
            terms = {}
            for i in range(P.NR):
                if ar == 1:
                    e = ((i >> ea) & 1) if ka == "reg" else None
                else:
                    a = ((i >> ea) & 1) if ka == "reg" else None
                    b = ((i >> eb) & 1) if kb == "reg" else None
                    e = (a, b)
                terms.setdefault(e, []).append(i)
            w(" ".join(f"{nm[k]} = -0.f;" for k in range(1 << ar)))
            for e, idxs in terms.items():
                sy = _tree_sum([f"c{i}" for i in idxs])
                if ar == 1:
                    ix = str(e) if e is not None else ea
                else:
                    if e[0] is not None and e[1] is not None:
                        ix = str(2 * e[0] + e[1])
                    else:
                        a_e = str(e[0]) if e[0] is not None else ea
                        b_e = str(e[1]) if e[1] is not None else eb
                        ix = f"(2 * ({a_e}) + ({b_e}))"
                if ix.isdigit():
                    w(f"{nm[int(ix)]} += {sy};")
                else:
                    w(f"{{ const int e_ = {ix}; const float sy_ = {sy};")
                    for ee in range(1 << ar):
                        w(f"  {nm[ee]} += e_ == {ee} ? sy_ : 0.f;")
                    w("}")
        w.ind -= 1
        w("}")
        for si, s in enumerate(subs):
            slot = int(s[4])
            if slot >= 0:
                ne = 1 << int(s[5])
                free = [slot + 2 * e for e in range(ne)]
                for e in range(ne):
                    P.coup.add(w, names[si][e], slot + 2 * e + 1, free)
    # phases
    if not rotate:
        return
    w("{")
    w.ind += 1
    per_i = _drun_prelude(w, P, subs, tp)
    inv = "true" if mode_bwd else "false"
    for i in range(P.NR):
        expr = " + ".join(["cph"] + per_i[i])
        w(f"{{ const int32_t p_ = {expr};")
        for q in range(nv):
            if P.rho_live:  # the run's phase also carries the tangent-rotation scale back
                w(f"  v[{q}][{i}] = phase_rot_s(v[{q}][{i}], p_, {inv}, rho_);")
            else:
                w(f"  v[{q}][{i}] = phase_rot(v[{q}][{i}], p_, {inv});")
        w("}")
    if P.rho_live:
        w("rho_ = 1.f;")
        P.rho_live = False
        P.tan_count = 0
    w.ind -= 1
    w("}")


def _drun_prelude(w, P, subs, tp):
    """Emit the run's thread-constant phase cph and table pointers in the current scope;
    return the per-register-index phase terms."""
    w("int32_t cph = 0;")
    per_i = [[] for _ in range(P.NR)]
    for si, s in enumerate(subs):
        moff = int(s[3])
        ar = int(s[5])
        ka, ea = _src_expr(s[0], P, tp)
        kb, eb = _src_expr(s[1], P, tp)
        w(f"const int32_t* a{si} = reinterpret_cast<const int32_t*>(s_mat + {moff});")
        if ar == 1:
            if ka == "reg":
                for i in range(P.NR):
                    per_i[i].append(f"a{si}[{(i >> ea) & 1}]")
            else:
                w(f"cph += a{si}[{ea}];")
        else:
            if ka != "reg" and kb != "reg":
                w(f"cph += a{si}[2 * {ea} + {eb}];")
            elif ka == "reg" and kb == "reg":
                for i in range(P.NR):
                    per_i[i].append(f"a{si}[{2 * ((i >> ea) & 1) + ((i >> eb) & 1)}]")
            elif ka == "reg":
                w(f"const int32_t lo{si} = a{si}[{eb}], hi{si} = a{si}[2 + {eb}];")
                for i in range(P.NR):
                    per_i[i].append(f"{'hi' if (i >> ea) & 1 else 'lo'}{si}")
            else:
                w(f"const int32_t lo{si} = a{si}[2 * {ea}], hi{si} = a{si}[2 * {ea} + 1];")
                for i in range(P.NR):
                    per_i[i].append(f"{'hi' if (i >> eb) & 1 else 'lo'}{si}")
    return per_i


FOLD_DRUN = os.environ.get("LSQ_FOLD_DRUN", "1") != "0"
FOLD_MAXC = int(os.environ.get("LSQ_FOLD_MAXC", "2"))
FOLD_FWD = os.environ.get("LSQ_FOLD_FWD", "1") != "0"


def _fold_classes(P, op, ph_idx, k):
    """Pairs (i, i | 2^k) of a diagonal run followed by a one-qubit group on register bit k,
    grouped by their (phase_i, phase_j) term lists; None when the run has more than FOLD_MAXC
    classes (then rotating every amplitude is cheaper)."""
    subs = P.enc["subs"][op[6] : op[6] + op[7]]
    tp = f"tp{ph_idx}"
    w0 = _W()
    per_i = _drun_prelude(w0, P, subs, tp)
    cls = {}
    for i in range(P.NR):
        if (i >> k) & 1:
            continue
        j = i | (1 << k)
        cls.setdefault((tuple(per_i[i]), tuple(per_i[j])), []).append((i, j))
    return cls if len(cls) <= FOLD_MAXC else None


def _emit_fold(w, P, dop, uop, ph_idx, mode_bwd, nv):
    """Diagonal run D followed by a one-qubit group U on register bit k, applied as one op:
    forward U D (columns of U scaled by the run's phase of each pair member), adjoint
    (U D)^+ = D^+ U^+ (rows of U^+ scaled by the conjugate phases). One coefficient set per
    class of pairs (FOLD_MAXC at most) instead of a phase rotation of every amplitude of every
    vector; the run's couplings (conj(lam) psi is phase invariant) are taken after."""
    k = int(uop[1])
    moff = int(uop[5])
    subs = P.enc["subs"][dop[6] : dop[6] + dop[7]]
    tp = f"tp{ph_idx}"
    w("{")
    w.ind += 1
    per_i = _drun_prelude(w, P, subs, tp)
    w(f"const float* g_ = s_mat + {moff};")
    # U entries as complex pairs (row-major)
    w("const float2 u00_ = make_float2(g_[0], g_[1]), u01_ = make_float2(g_[2], g_[3]), "
      "u10_ = make_float2(g_[4], g_[5]), u11_ = make_float2(g_[6], g_[7]);")
    cls = {}
    for i in range(P.NR):
        if (i >> k) & 1:
            continue
        j = i | (1 << k)
        cls.setdefault((tuple(per_i[i]), tuple(per_i[j])), []).append((i, j))
    for c, ((ti, tj), pairs) in enumerate(cls.items()):
        ei = " + ".join(["cph"] + list(ti))
        ej = " + ".join(["cph"] + list(tj))
        w(f"const float2 pi{c}_ = phase_cs({ei}), pj{c}_ = phase_cs({ej});")
        if not mode_bwd:  # W = U diag(p_i, p_j)
            ent = [("u00_", f"pi{c}_"), ("u01_", f"pj{c}_"), ("u10_", f"pi{c}_"), ("u11_", f"pj{c}_")]
        else:  # W = diag(p_i, p_j)^* U^+: W_ab = conj(U_ba p_a)
            ent = [("u00_", f"pi{c}_"), ("u10_", f"pi{c}_"), ("u01_", f"pj{c}_"), ("u11_", f"pj{c}_")]
        for e, (u, ph) in enumerate(ent):
            if P.rho_live:
                w(f"const float2 t{c}_{e} = cm({ph}.x * rho_, {ph}.y * rho_, {u});")
            else:
                w(f"const float2 t{c}_{e} = cm({ph}.x, {ph}.y, {u});")
        conj = "-" if mode_bwd else ""
        w(f"const float f{c}_[8] = {{" + ", ".join(f"t{c}_{e}.x, {conj}t{c}_{e}.y" for e in range(4)) + "};")
        for q in range(nv if mode_bwd else 1):
            for i, j in pairs:
                w(f"{{ const float2 x0 = v[{q}][{i}], x1 = v[{q}][{j}];")
                for a, dst in ((0, i), (1, j)):
                    e0, e1 = 2 * a, 2 * a + 1
                    w(f"  v[{q}][{dst}] = fix(x1, f{c}_[{2 * e1 + 1}], fx(x1, f{c}_[{2 * e1}], "
                      f"fix(x0, f{c}_[{2 * e0 + 1}], mx(x0, f{c}_[{2 * e0}]))));")
                w("}")
    if P.rho_live:
        w("rho_ = 1.f;")
        P.rho_live = False
        P.tan_count = 0
    w.ind -= 1
    w("}")


def _emit_ops(w, P, ph_idx, mode_bwd, nv):
    ops = P.enc["ops"][ph_idx]
    seq = list(reversed(ops)) if mode_bwd else ops
    regs = P.pp.phases[ph_idx].regs

    def foldable(dop, uop):
        if not FOLD_DRUN or dop is None or uop is None:
            return False
        if int(dop[0]) != S.OP_DRUN or int(uop[0]) != S.OP_U1:
            return False
        grp = P.prog.groups[int(uop[3])]
        if _group_const_matrix(grp, P.drop_phase) is not None:
            return False
        if any(c != "c" for row in u1_structure(grp)[0] for c in row):
            return False  # structured (real / sparse) groups would lose their cheap apply
        return _fold_classes(P, dop, ph_idx, int(uop[1])) is not None

    def euler_plain(op):
        """one-qubit group that takes the branch-free Euler tangent form (constant |U00|)"""
        if int(op[0]) != S.OP_U1:
            return False
        grp = P.prog.groups[int(op[3])]
        if _group_const_matrix(grp, P.drop_phase) is not None:
            return False
        if any(g.layer in getattr(P.prog, "direct_layers", ()) for g, _ in grp.gates):
            return False
        if any(c != "c" for row in u1_structure(grp)[0] for c in row):
            return False
        if TAN_ROT and P.tan_ok and is_rotation(grp):
            return False
        return bool(EULER_TAN and P.drop_phase and P.walsh_diag and u00_const_mag(grp) is not None)

    def euler_coup_ok(grp):
        classes, comps = u1_structure(grp)
        cm_ = u00_const_mag(grp)
        return bool(EULER_COUP and "I" not in comps and cm_ is not None and 1e-3 < cm_ ** 2 < 1 - 1e-3)

    def merged_run(idx):
        """ops seq[idx : idx + k] forming a run of Euler-form groups to apply merged (k >=
        EULER_MERGE), else None; a group a diagonal run folds into stays on the fold path"""
        if not EULER_MERGE:
            return None
        j, bits = idx, set()
        while j < len(seq) and euler_plain(seq[j]):
            nx = seq[j + 1] if j + 1 < len(seq) else None
            if mode_bwd and foldable(nx, seq[j]):
                break
            # distinct register bits only: two groups of one wire can be neighbours when what
            # separates them emits no op (an identity permutation, e.g. ECR applied twice)
            if int(seq[j][1]) in bits:
                break
            bits.add(int(seq[j][1]))
            j += 1
        return seq[idx:j] if j - idx >= max(2, EULER_MERGE) else None

    skip = 0
    for idx, op in enumerate(seq):
        if skip:
            skip -= 1
            continue
        kind = int(op[0])
        nxt = seq[idx + 1] if idx + 1 < len(seq) else None
        run = merged_run(idx) if kind == S.OP_U1 else None
        if run is not None:
            pend = []
            if mode_bwd:  # couplings at the post-run point (invariant under the other wires' groups)
                for rop in run:
                    slot, grp = int(rop[4]), P.prog.groups[int(rop[3])]
                    if slot < 0:
                        continue
                    if euler_coup_ok(grp):
                        pend.append((rop, _emit_euler_coupling_post(w, P, int(rop[1]))))
                    else:
                        _emit_u1_coupling(w, P, int(rop[1]), slot, u1_structure(grp)[1])
            _emit_euler_merged(w, P, run, nv if mode_bwd else 1, mode_bwd)
            for rop, names in pend:
                _emit_euler_coupling_pre(w, P, int(rop[1]), int(rop[4]), names, f"(s_mat + {int(rop[5])})",
                                         u00_const_mag(P.prog.groups[int(rop[3])]))
            skip = len(run) - 1
            continue
        if not mode_bwd and FOLD_FWD and kind == S.OP_DRUN and foldable(op, nxt):
            _emit_fold(w, P, op, nxt, ph_idx, False, nv)
            skip = 1
            continue
        if mode_bwd and kind == S.OP_U1 and foldable(nxt, op):
            slot = int(op[4])
            if slot >= 0:
                _emit_u1_coupling(w, P, int(op[1]), slot, u1_structure(P.prog.groups[int(op[3])])[1])
            _emit_fold(w, P, nxt, op, ph_idx, True, nv)
            _emit_drun(w, P, nxt, ph_idx, True, nv, couplings=True, rotate=False)
            skip = 1
            continue
        if kind == S.OP_PX:
            for q in range(nv):
                w(f"perm_x<{P.R}, {int(op[1])}>(v[{q}]);")
        elif kind == S.OP_PCX:
            for q in range(nv):
                w(f"perm_cx<{P.R}, {int(op[1])}, {int(op[2])}>(v[{q}]);")
        elif kind in (S.OP_U1, S.OP_U2):
            gid = int(op[3])
            grp = P.prog.groups[gid]
            bits = [int(op[1])] + ([int(op[2])] if kind == S.OP_U2 else [])
            slot, moff = int(op[4]), int(op[5])
            U = _group_const_matrix(grp, P.drop_phase)
            direct = any(g.layer in getattr(P.prog, "direct_layers", ()) for g, _ in grp.gates)
            ecoup = None  # Euler-point couplings (constant |U00| groups in the Euler tangent form)
            if mode_bwd and slot >= 0:
                if kind == S.OP_U1:
                    classes, comps = u1_structure(grp)
                    if (EULER_COUP and U is None and EULER_TAN and not direct and P.drop_phase
                            and P.walsh_diag and "I" not in comps
                            and all(c == "c" for row in classes for c in row)
                            and not (TAN_ROT and P.tan_ok and is_rotation(grp))
                            and u00_const_mag(grp) is not None
                            and 1e-3 < u00_const_mag(grp) ** 2 < 1 - 1e-3):
                        ecoup = _emit_euler_coupling_post(w, P, bits[0])
                    else:
                        _emit_u1_coupling(w, P, bits[0], slot, comps)
                else:
                    csc = _scaled(P, "1.f")
                    fix_ = "" if csc == "1.f" else f"for (int e_ = 0; e_ < 8; ++e_) acc[e_] *= {csc}; "
                    for rr in range(4):
                        w(f"{{ float acc[8] = {{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}}; "
                          f"u2_coupling_row<{P.R}, {bits[0]}, {bits[1]}, {rr}>(v[0], v[1], acc); {fix_}"
                          f"warp_accumulate8<{P.NT}>(acc, wacc + {slot + 8 * rr}); }}")
            uf = unit_form(U) if (U is not None and UNIT_CONST and P.walsh_diag) else None
            if uf is not None:
                # U / kappa with entries in {0, +-1, +-i}; the vectors carry the deferred scale
                kappa, V = uf
                for q in range(nv if mode_bwd else 1):
                    _emit_unit_const(w, P, f"v[{q}]", V, bits, mode_bwd)
                    P.sc[q] /= kappa
                _guard_scale(w, P, nv if mode_bwd else 1)  # deep single-pass circuits: fp32 range
            elif U is not None:
                for q in range(nv):
                    _emit_const_u(w, P, f"v[{q}]", U, bits, mode_bwd)
            elif kind == S.OP_U1:
                classes = u1_structure(grp)[0]
                w(f"{{ const float* g_ = s_mat + {moff};")
                general = all(c == "c" for row in classes for c in row)
                cmag = u00_const_mag(grp) if general else None
                if TAN_ROT and P.tan_ok and not direct and is_rotation(grp):
                    _emit_tan_rot(w, P, bits[0], "g_", nv if mode_bwd else 1, mode_bwd, classes)
                    if P.tan_count >= TAN_RENORM:
                        _renorm_rho(w, P, nv if mode_bwd else 1)
                elif (EULER_TAN and general and not direct and P.drop_phase and P.walsh_diag
                        and (cmag is not None or (P.tan_ok and EULER_BRANCH))):
                    _emit_euler_tan(w, P, bits[0], "g_", nv if mode_bwd else 1, mode_bwd, classes,
                                    branch=cmag is None)
                    if ecoup is not None:
                        _emit_euler_coupling_pre(w, P, bits[0], slot, ecoup, "g_", cmag)
                        ecoup = None
                    if P.tan_count >= TAN_RENORM:
                        _renorm_rho(w, P, nv if mode_bwd else 1)
                else:
                    for q in range(nv if mode_bwd else 1):
                        _emit_u1_struct(w, f"v[{q}]", bits[0], P.R, classes, "g_", mode_bwd)
                w("}")
                assert ecoup is None, "Euler-point coupling left unfinished"
            else:
                if mode_bwd:
                    for q in range(nv):
                        w(f"u2_apply_dag<{P.R}, {bits[0]}, {bits[1]}>(v[{q}], s_mat + {moff});")
                else:
                    w(f"u2_apply<{P.R}, {bits[0]}, {bits[1]}>(v[0], s_mat + {moff});")
        else:
            _emit_drun(w, P, op, ph_idx, mode_bwd, nv)


def _pairs(P, ph):
    """Register pairs (i, j) held at adjacent local positions (local bit 0 is register bit k0):
    one 16-byte shared access moves both; None when local bit 0 is a thread bit."""
    regs = P.pp.phases[ph].regs
    if not VEC_SMEM or 0 not in regs:
        return None
    k0 = regs.index(0)
    return [(i, i | (1 << k0)) for i in range(P.NR) if not (i >> k0) & 1]


LAZY_SX = os.environ.get("LSQ_LAZY_SX", "1") != "0"


def _has_fold(P):
    """True when some diagonal run of the pass folds into the following one-qubit group."""
    for ph_idx, ops in enumerate(P.enc["ops"]):
        for a, b in zip(ops, ops[1:]):
            if int(a[0]) != S.OP_DRUN or int(b[0]) != S.OP_U1:
                continue
            grp = P.prog.groups[int(b[3])]
            if _group_const_matrix(grp, P.drop_phase) is not None:
                continue
            if all(c == "c" for row in u1_structure(grp)[0] for c in row) and \
                    _fold_classes(P, a, ph_idx, int(b[1])) is not None:
                return True
    return False


def _sx_open(w, k, P=None):
    """Swizzled thread base of layout k as an opaque local copy made where it is used (one
    LOP3 per access instead of hoisted per-register addresses; not held across the tile).
    Measured: a gain except for adjoint kernels with folded diagonal runs (their coefficient
    sets need the registers the early copies would otherwise free), which keep early copies."""
    if P is not None and P.lazy_sx:
        w(f"{{ uint32_t sxl_ = st{k}; asm volatile(\"\" : \"+r\"(sxl_));")
        return "sxl_"
    w("{")
    return f"sx{k}"


# swizzled shared index S(tp | loc) = (S(tp) ^ lo) + hi with lo = S(loc) & 0xE (the swizzle bits)
# and hi = the rest: the thread and register parts are disjoint local bits and the swizzle only
# writes bits 1..3, so after XOR-ing the (at most 8) distinct lo values into per-transpose bases
# every access is base + immediate (LDS/STS [R + imm]) instead of one LOP3 per access
SWZ_IMM = os.environ.get("LSQ_SWZ_IMM", "1") != "0"


def _swz_index(w, P, sx, offs, buf):
    """(pointer, index) expressions of the swizzled offsets `offs` off the thread base `sx` in
    `buf`: with SWZ_IMM one shared pointer per distinct swizzle-bit value and a constant index
    (folded into the LDS/STS immediate), else the buffer and an XOR-ed index."""
    if not SWZ_IMM:
        return [(buf, f"{sx} ^ {o}u") for o in offs]
    names = {}
    out = []
    for o in offs:
        lo, hi = o & 0xE, o & ~0xE
        if lo not in names:
            names[lo] = f"{sx}p{lo}_"
            w(f"float2* const {names[lo]} = {buf} + ({sx} ^ {lo}u);")
        out.append((names[lo], f"{hi}u"))
    return out


def _emit_put(w, P, buf, a, q):
    """vector q (registers, layout a) -> buf (swizzled)"""
    pr = _pairs(P, a)
    sx = _sx_open(w, a, P)
    if pr is None:
        idx = _swz_index(w, P, sx, [P.soff(a, i) for i in range(P.NR)], buf)
        for i in range(P.NR):
            w(f"{idx[i][0]}[{idx[i][1]}] = v[{q}][{i}];")
    else:
        idx = _swz_index(w, P, sx, [P.soff(a, i) for i, _ in pr], buf)
        for (i, j), (pb, e) in zip(pr, idx):
            w(f"st_pair({pb}, {e}, v[{q}][{i}], v[{q}][{j}]);")
    w("}")


def _emit_get(w, P, buf, b, q):
    """buf (swizzled) -> vector q (registers, layout b)"""
    pr = _pairs(P, b)
    sx = _sx_open(w, b, P)
    if pr is None:
        idx = _swz_index(w, P, sx, [P.soff(b, i) for i in range(P.NR)], buf)
        for i in range(P.NR):
            w(f"v[{q}][{i}] = {idx[i][0]}[{idx[i][1]}];")
    else:
        idx = _swz_index(w, P, sx, [P.soff(b, i) for i, _ in pr], buf)
        for (i, j), (pb, e) in zip(pr, idx):
            w(f"ld_pair({pb}, {e}, v[{q}][{i}], v[{q}][{j}]);")
    w("}")


VEC_SMEM = os.environ.get("LSQ_VEC_SMEM", "1") != "0"


def _emit_exchange(w, P, a, b, nv):
    for q in range(nv):
        w("__syncthreads();")
        _emit_put(w, P, "s_x", a, q)
        w("__syncthreads();")
        _emit_get(w, P, "s_x", b, q)


class _Rot:
    """Exchange buffers of the adjoint and turnaround kernels: the exchange buffer and the two
    prefetch-stage vectors (the next tile is prefetched only after the last exchange, so the
    stage is free while a tile is transposed). A buffer read since the last barrier is
    "dirty"; an exchange writes clean buffers first and pays a barrier only when it must
    reuse a dirty one, so a two-vector exchange costs two barriers instead of four and a
    one-vector exchange one instead of two."""

    def __init__(self, P, nstage, late=True, bufs=None):
        # late: the stage is free during the tile (prefetch issued after the last transpose);
        # otherwise only the stage's unused second vector (turnaround kernels) joins s_x
        self.late = late
        if bufs is not None:
            self.bufs = list(bufs)
        elif late:
            self.bufs = ["s_x", "s_stage", f"(s_stage + {1 << P.M})"][: 1 + nstage]
        else:
            self.bufs = ["s_x", f"(s_stage + {1 << P.M})"]
        self.dirty = set()

    def exchange(self, w, P, a, b, vecs):
        order = [x for x in self.bufs if x not in self.dirty] + [x for x in self.bufs if x in self.dirty]
        use = order[: len(vecs)]
        for q, buf in zip(vecs, use):
            if buf in self.dirty:
                w("__syncthreads();")
                self.dirty = set()
            _emit_put(w, P, buf, a, q)
        w("__syncthreads();")
        for q, buf in zip(vecs, use):
            _emit_get(w, P, buf, b, q)
        self.dirty = set(use)


SMEM_LIMIT = 227 * 1024
# prefetch stage in the swizzled order of the exchange buffers (LSQ_STAGE_SWZ=0: natural order,
# round 1 -- its phase-layout reads were bank-conflicted: ncu 4.4e8 excess wavefronts in cfg4 p1)
STAGE_SWZ = os.environ.get("LSQ_STAGE_SWZ", "1") != "0"


def generic_smem_bytes(prog, pi: int) -> int:
    """Mirror of smem_bytes() in csrc/lsq_lib.cu (tables + exchange buffer)."""
    pp = prog.passes[pi]
    enc = prog.enc[pi]
    nt = 1 << (pp.M - pp.R)
    nw = (nt + 31) // 32
    nops = sum(len(o) for o in enc["ops"])
    nsubs = sum(int(op[7]) for ph in enc["ops"] for op in ph if int(op[0]) == S.OP_DRUN)
    b = 8 * (1 << pp.M)
    b += 4 * (len(pp.phases) * S.PHASE_WORDS + nops * S.OP_WORDS + nsubs * S.SUB_WORDS + 64)
    b += 4 * (((enc["matf"] + 3) & ~3) + ((nw * enc["slotf"] + 3) & ~3))
    b += 8 * 34 + 4 * nw * 32
    b += 4 * nw * 8  # coupling half-block padding of the specialised kernels
    return (b + 15) & ~15


def stage_vectors(prog, pi: int, mode: int) -> int:
    """Vectors prefetched into shared memory by the specialised kernel (0 if they don't fit)."""
    nv = 1 if mode == MODE_FWD else 2
    pp = prog.passes[pi]
    if generic_smem_bytes(prog, pi) + nv * 8 * (1 << pp.M) <= SMEM_LIMIT:
        return nv
    return 0


# forward kernels with ONE tile buffer: the prefetch stage and the exchange buffer are the same
# 2^M amplitudes (the next tile is prefetched after the last transpose, like the adjoint
# kernels' late prefetch), so a CTA needs 32 KB + tables at M = 12 instead of 64 KB and the
# 128-thread forward CTAs run 4 per SM (register-limited) instead of 3 (shared-memory-limited)
FWD_SINGLE = os.environ.get("LSQ_FWD_SINGLE", "1") != "0"


def fwd_single(prog, pi: int, mode: int) -> bool:
    return bool(FWD_SINGLE and mode == MODE_FWD and stage_vectors(prog, pi, mode) > 0)


def stage_alloc(prog, pi: int, mode: int) -> int:
    """Stage vectors the C side allocates after the fixed shared-memory layout (lsq_program_jit):
    none for single-buffer forward kernels, whose stage aliases the exchange buffer."""
    return 0 if fwd_single(prog, pi, mode) else stage_vectors(prog, pi, mode)


def emit_kernel(prog, pi: int, mode: int) -> str:
    P = _Pass(prog, pi)
    P.coup = _Coup(P)
    P.drop_phase = bool(getattr(prog, "drop_phase", False))
    P.walsh_diag = os.environ.get("LSQ_WALSH_DIAG", "1") != "0"
    P.walsh = []  # (slot, arity, components) of diagonal couplings kept as Walsh sums
    P.sc = [1.0, 1.0]  # deferred (compile-time) scale of psi and lambda: computed = true x sc
    P.rho_live = False  # run-time scale rho_ (tangent-form rotations) may differ from 1
    P.ph_live = False  # run-time global phase phc_ (branching Euler groups) may differ from 1
    P.tan_count = 0
    # tangent-form rotations in the adjoint kernels only: measured -2% there, +3% in the forward
    # and turnaround kernels (the uniform fallback branch costs them their scheduling freedom)
    P.tan_ok = P.walsh_diag and mode == MODE_BWD
    P.slotf = prog.enc[pi]["slotf"]
    nv = 1 if mode == MODE_FWD else 2
    prefetch = stage_vectors(prog, pi, mode) > 0
    nph = len(P.pp.phases)
    # rotating exchange buffers (late next-tile prefetch) for the adjoint kernels: measured +2%
    # there; the turnaround keeps its early prefetch (its forward half would lose the overlap)
    rot = None
    if prefetch and os.environ.get("LSQ_ROT", "1") != "0":
        if mode == MODE_BWD and nph > 1:
            rot = _Rot(P, 2)
        elif mode == MODE_TURN and nph > 1 and os.environ.get("LSQ_ROT_TURN", "1") != "0":
            rot = _Rot(P, 2, late=False)  # psi-only stage: its lambda half is a spare buffer
        elif mode == MODE_FWD and fwd_single(prog, pi, mode):
            if nph > 1:  # the one buffer is stage and exchange buffer: late prefetch
                rot = _Rot(P, 1, bufs=["s_stage"])
        elif mode == MODE_FWD and nph >= int(os.environ.get("LSQ_ROT_FWD_PHASES", "99")):
            # forward kernels: measured neutral (one vector: the early prefetch overlap matters
            # as much as the saved barrier), so off by default
            rot = _Rot(P, 1)
    est_regs = 2 * P.NR * nv + 40
    minb = max(1, min(4, 65536 // (P.NT * est_regs)))
    if mode == MODE_FWD and P.R >= 5:
        # forward kernels with 32 amplitudes per thread: 128 registers (64 data), 4 CTAs of 128
        # threads per SM (LSQ_MINB_FWD5 overrides, A/B runs)
        # (128-register budget whatever the tile size: M = 13 has 256 threads -> 2 CTAs/SM)
        minb = int(os.environ.get("LSQ_MINB_FWD5", str(max(1, min(4, 65536 // (P.NT * 128))))))
    elif mode == MODE_FWD:
        # forward kernels: an 80-register budget (measured: 256-thread tiles at 3 CTAs/SM beat 2,
        # 128-thread tiles at 6 beat 4 -- occupancy wins over a few spills)
        minb = max(1, min(8, 65536 // (P.NT * 80)))
    if os.environ.get("LSQ_MINB_FWD") and mode == MODE_FWD:
        minb = int(os.environ["LSQ_MINB_FWD"])
    matf = P.enc["matf"]
    slotf = P.enc["slotf"]
    w = _W()
    out = [f'extern "C" __global__ void __launch_bounds__({P.NT}, {minb}) {kernel_name(pi, mode)}(lsq::PassArgs A) {{']
    w("using namespace lsq;")
    w(f"constexpr int NT = {P.NT}, NW = {P.NW}, M = {P.M};")
    w("extern __shared__ __align__(16) unsigned char smem_raw[];")
    w("float2* s_x = reinterpret_cast<float2*>(smem_raw);")
    w(f"float* s_mat = reinterpret_cast<float*>(s_x + {1 << P.M});")
    w(f"float* s_acc = s_mat + {(matf + 3) & ~3};")
    w(f"double* s_z = reinterpret_cast<double*>(s_acc + {(P.NW * (slotf + 8) + 3) & ~3});")
    w("float* s_zw = reinterpret_cast<float*>(s_z + 34);  // [NW][32] per-warp <Z> partials")
    # next-tile prefetch stage [NV][2^M], natural local order, after the fixed tables so the
    # generic kernel's shared-memory size plus NV x 2^M x 8 B covers it (lsq_program_jit)
    use_prefix = bool(getattr(prog, "prefix", None)) and pi == 0
    # byte offset of the stage as a constant so the compiler keeps the shared window (LDS, not
    # generic LD) for the stage reads
    off = (8 << P.M) + 4 * ((matf + 3) & ~3) + 4 * ((P.NW * (slotf + 8) + 3) & ~3) + 8 * 34 + 4 * P.NW * 32
    off = (off + 15) & ~15
    if fwd_single(prog, pi, mode):
        w("float2* s_stage = s_x;  // single tile buffer: prefetch stage == exchange buffer")
    else:
        w(f"float2* s_stage = reinterpret_cast<float2*>(smem_raw + {off});")
    # the prefix vectors live in the first 8*n bytes of the exchange buffer's tail region: use a
    # dedicated register-free path -- they are read from global (L1-cached, 16 B per wire)
    w("const int tid = threadIdx.x, warp = tid >> 5;")
    w("const int row = blockIdx.x / A.ctas_per_row, cslot = blockIdx.x % A.ctas_per_row;")
    w("const int mode = A.mode, flags = A.flags;")
    w("(void)mode; (void)warp; (void)s_zw;")
    # stage group tables
    pgs = P.enc["pgroups"]  # list of (gid, moff)
    w("{")
    w.ind += 1
    for j, (gid, moff) in enumerate(pgs):
        grp = prog.groups[gid]
        if not grp.diag and (_group_const_matrix(grp) is not None or grp.perm_ops is not None):
            continue  # compile-time constants, never read from the table
        if grp.perrow:
            ri = prog.rowidx[gid]
            w(f"for (int e = tid; e < {grp.mat_floats}; e += NT) s_mat[{moff} + e] = A.rowtab[((size_t)row * A.nperrow + {ri}) * 32 + e];")
        else:
            w(f"for (int e = tid; e < {grp.mat_floats}; e += NT) s_mat[{moff} + e] = A.gmats[{gid * 32} + e];")
    w(f"for (int i = tid; i < {P.NW * (slotf + 8)}; i += NT) s_acc[i] = 0.f;")
    w("for (int i = tid; i < 34; i += NT) s_z[i] = 0.0;")
    w(f"for (int i = tid; i < {P.NW * 32}; i += NT) s_zw[i] = 0.f;")
    w.ind -= 1
    w("}")
    w("__syncthreads();")
    # per-warp coupling accumulators: slotf floats + 8 padding floats (zero half-blocks)
    w(f"float* wacc = s_acc + warp * {slotf + 8};")
    w("(void)wacc;")
    w("const int lj_ = (tid >> 2) & 3;  // reduce-scatter value index within a half-block")
    w("const int pu1_ = (0x7431 >> (4 * lj_)) & 15, pdg_ = 2 * lj_ + 1;")
    w("const bool hi16_ = (tid & 16) != 0;")
    w("(void)pu1_; (void)pdg_; (void)hi16_;")
    # per-phase thread layout constants
    for k, ph in enumerate(P.pp.phases):
        tp_terms = [f"(((uint32_t)tid >> {j}) & 1u) << {lb}" for j, lb in enumerate(ph.threads)]
        gt_terms = [f"(((uint32_t)tid >> {j}) & 1u) << {P.pbit[lb]}" for j, lb in enumerate(ph.threads)]
        w(f"const uint32_t tp{k} = {' | '.join(tp_terms) if tp_terms else '0u'};")
        w(f"const uint32_t gt{k} = {' | '.join(gt_terms) if gt_terms else '0u'};")
        w(f"const uint32_t st{k} = swz(tp{k});")
        w(f"(void)tp{k}; (void)gt{k}; (void)st{k};")
    w(f"const size_t rowbase = (size_t)row << {P.n};")
    w("const int t0 = cslot * A.tiles_per_cta, t_end = t0 + A.tiles_per_cta;")
    skew_ns = int(os.environ.get("LSQ_SKEW_NS", "0"))
    if skew_ns and mode in (MODE_BWD, MODE_TURN) + ((MODE_FWD,) if os.environ.get("LSQ_SKEW_FWD") == "1" else ()):
        # experiment: de-phase the CTAs that share an SM (first wave only, later CTAs inherit the
        # offset) so one computes while the other transposes
        sm = int(os.environ.get("LSQ_SKEW_MODE", "1"))
        cond = {1: "(blockIdx.x & 1)", 2: "((blockIdx.x / 148) & 1)",
                3: f"((warpid_() / {P.NW}) & 1)"}[sm]
        if sm == 3:
            w("auto warpid_ = [] { unsigned r; asm volatile(\"mov.u32 %0, %%warpid;\" : \"=r\"(r)); return r; };")
        w(f"if (blockIdx.x < {148 * minb} && {cond}) {{ for (int s_ = 0; s_ < {max(1, skew_ns // 1000)}; ++s_) __nanosleep(1000); }}")
    last = nph - 1
    # adjoint and turnaround kernels read their tile from the prefetch stage, where any layout
    # is free: an empty last phase (kept only so forward stores are coalesced) is skipped,
    # saving one transpose per vector
    top = last
    if (mode != MODE_FWD and prefetch and nph > 1 and len(P.enc["ops"][last]) == 0
            and os.environ.get("LSQ_SKIP_EMPTY", "1") != "0"):
        top = last - 1
    # ---- next-tile prefetch: cp.async 16-byte chunks into the stage (natural local order).
    # chunk c holds local amplitudes (2c, 2c+1); c = (tid low bits) + j * 2^tid_bits.
    nchunk = 1 << (P.M - 1)
    per_thr = max(1, nchunk // P.NT)
    tid_bits = (nchunk // per_thr).bit_length() - 1
    cth_terms = [f"(((uint32_t)tid >> {jj}) & 1u) << {P.pbit[jj + 1]}" for jj in range(tid_bits)]
    w(f"const uint32_t cth = {' | '.join(cth_terms) if cth_terms else '0u'};")
    w(f"const bool cp_on = tid < {nchunk};")
    # the stage holds the tile in the exchange buffers' swizzled order (S is XOR-linear and
    # keeps every 16-byte chunk whole), so reading it in any phase layout is as conflict-free
    # as an exchange; the writer's per-thread part of the swizzled chunk address is hoisted
    w(f"const uint32_t cst_ = {'swz(2u * (tid & ' + str((1 << tid_bits) - 1) + '))' if STAGE_SWZ else '2u * (tid & ' + str((1 << tid_bits) - 1) + ')'};")
    w("(void)cth; (void)cp_on; (void)cst_;")
    ld_vecs = [(0, "A.psi_in"), (1, "A.lam")] if mode == MODE_BWD else [(0, "A.psi_in")]
    if mode == MODE_FWD:
        w("const bool do_load = !(flags & PF_SYNTH);")
    elif mode == MODE_BWD:
        w("const bool do_load = true;")
    else:
        w("const bool nofwd = (flags & PF_NOFWD) != 0;")
        w("const bool do_load = nofwd || !(flags & PF_SYNTH);")

    def emit_issue(tile_expr):
        tb2 = [f"((uint64_t)((({tile_expr}) >> {jj}) & 1)) << {p}" for jj, p in enumerate(P.nbit)]
        w.block("if (cp_on)")
        w(f"const size_t nb = rowbase + ({' | '.join(tb2) if tb2 else '0ull'});")
        for vi, ptr in ld_vecs:
            for jj in range(per_thr):
                loc = 2 * (jj << tid_bits)
                phys = sum(1 << P.pbit[b] for b in range(P.M) if (loc >> b) & 1)
                sl = S_swz(loc) if STAGE_SWZ else loc
                w(f"cp_async16(s_stage + {vi * (1 << P.M)} + (cst_ ^ {sl}u), {ptr} + nb + (cth | {phys}u));")
        w.end()

    def emit_stage_read(k):
        ph = P.pp.phases[k]
        pr = _pairs(P, k)
        for vi, _ in ld_vecs:
            if pr is not None:  # natural order: the pair on local bit 0 is adjacent
                for i, j in pr:
                    loc = sum(1 << ph.regs[b] for b in range(P.R) if (i >> b) & 1)
                    if STAGE_SWZ:
                        w(f"ld_pair(s_stage, {vi * (1 << P.M)} + (st{k} ^ {S_swz(loc)}u), v[{vi}][{i}], v[{vi}][{j}]);")
                    else:
                        w(f"ld_pair(s_stage, {vi * (1 << P.M)} + (tp{k} | {loc}u), v[{vi}][{i}], v[{vi}][{j}]);")
                continue
            for i in range(P.NR):
                loc = sum(1 << ph.regs[b] for b in range(P.R) if (i >> b) & 1)
                if STAGE_SWZ:
                    w(f"v[{vi}][{i}] = s_stage[{vi * (1 << P.M)} + (st{k} ^ {S_swz(loc)}u)];")
                else:
                    w(f"v[{vi}][{i}] = s_stage[{vi * (1 << P.M)} + (tp{k} | {loc}u)];")

    if prefetch:
        w.block("if (do_load && t0 < t_end)")
        emit_issue("t0")
        w.end()
        w("cp_async_commit();")
    w.block("for (int t = t0; t < t_end; ++t)")
    if rot is not None and not rot.late:
        # previous tile's last transpose may still be read: the first write here syncs first
        rot.dirty = set(rot.bufs)
    tb = [f"((uint64_t)((t >> {j}) & 1)) << {p}" for j, p in enumerate(P.nbit)]
    w(f"const uint64_t tbase = {' | '.join(tb) if tb else '0ull'};")
    # opaque per-tile copies of the shared-memory thread offsets: keeps the 2^R swizzled
    # exchange addresses as one LOP3 each instead of hoisted (and spilled) registers
    P.lazy_sx = LAZY_SX and not (mode == MODE_BWD and FOLD_DRUN and _has_fold(P))
    if not P.lazy_sx:
        for k in range(nph):
            w(f"uint32_t sx{k} = st{k}; asm volatile(\"\" : \"+r\"(sx{k}));")
    w("const size_t base = rowbase + tbase;")
    w(f"float2 v[{nv}][{P.NR}];")
    w("float rho_ = 1.f;  // run-time deferred scale of the tile's vectors (true = computed x rho_)")
    w("float2 phc_ = make_float2(1.f, 0.f);  // run-time global phase (true = computed x rho_ x phc_)")
    w("(void)rho_; (void)phc_;")

    def emit_load(k):
        """wait for this tile's prefetch, move it to registers (layout k), prefetch the next;
        without a stage (shared memory too small): direct streaming loads in layout k"""
        w.block("if (do_load)")
        if prefetch and rot is not None and rot.late:
            # the next tile is prefetched after the last exchange (emit_late_issue)
            w("cp_async_wait_all();")
            w("__syncthreads();")
            emit_stage_read(k)
            rot.dirty = {b for b in rot.bufs if b != "s_x"}  # stage vectors read without a barrier
        elif prefetch:
            w("cp_async_wait_all();")
            w("__syncthreads();")
            emit_stage_read(k)
            w("__syncthreads();")
            w.block("if (t + 1 < t_end)")
            emit_issue("t + 1")
            w.end()
            w("cp_async_commit();")
        else:
            for vi, ptr in ld_vecs:
                for i in range(P.NR):
                    w(f"v[{vi}][{i}] = __ldcs({ptr} + base + (gt{k} | {P.goff(k, i)}u));")
        w.end()

    def wire_of_local(lb):
        return P.n - 1 - P.pbit[lb]

    def pv(wire, idx_expr):
        """prefix vector entry v_wire[idx] (float2) of this CTA's row"""
        return f"reinterpret_cast<const float2*>(A.ptab)[((size_t)row * {P.n} + {wire}) * 2 + ({idx_expr})]"

    def emit_synth(k):
        if not use_prefix:
            for i in range(P.NR):
                w(f"v[0][{i}] = make_float2(((tbase | (uint64_t)(gt{k} | {P.goff(k, i)}u)) == 0) ? 1.f : 0.f, 0.f);")
            return
        # product state (x)_w v_w: constant factor over thread and tile bits, then a Kronecker
        # expansion over the register bits (one complex multiply per amplitude)
        ph = P.pp.phases[k]
        w("{")
        w.ind += 1
        w("float2 cst = make_float2(1.f, 0.f);")
        for lb in ph.threads:
            w(f"{{ const float2 f_ = {pv(wire_of_local(lb), f'(tp{k} >> {lb}) & 1u')}; cst = cm(f_.x, f_.y, cst); }}")
        for p in P.nbit:
            w(f"{{ const float2 f_ = {pv(P.n - 1 - p, f'(int)((tbase >> {p}) & 1ull)')}; cst = cm(f_.x, f_.y, cst); }}")
        w("v[0][0] = cst;")
        for kk in range(P.R):
            wr = wire_of_local(ph.regs[kk])
            w(f"{{ const float2 a0 = {pv(wr, '0')}, a1 = {pv(wr, '1')};")
            for i in range(1 << kk):
                w(f"  v[0][{i | (1 << kk)}] = cm(a1.x, a1.y, v[0][{i}]); v[0][{i}] = cm(a0.x, a0.y, v[0][{i}]);")
            w("}")
        w.ind -= 1
        w("}")

    def emit_prefix_lambda(k):
        """Lambda_w(a) = sum_{j: bit_w(j)=a} conj(lam_j) prod_{w' != w} v_w'(bit_w'(j)) for every
        prefix wire with a coupling slot, at the prefix boundary (end of the last adjoint pass).

        With S = sum_i conj(lam_i) Kr_i over the thread's registers (Kr: Kronecker product of
        the register wires' factors), C_thr / C_nl the products of the thread-bit / tile-bit
        wires' factors:
        * tile-bit wire t: Lambda_t(b_t) += NLO_t * sum_warp (C_thr S), NLO_t = prod over the
          other tile-bit wires (one complex per warp and tile, lane 0);
        * thread-bit wire t: C_nl * C_thr/t * S per thread (leave-one-out with a running
          suffix: O(#thread bits) registers);
        * register wire k: C_nl * C_thr * sum_{b_k(i)=a} conj(lam_i) prod_{k' != k} v_k'."""
        slots = {}
        pre = prog.prefix
        for wire, gid in pre.items():
            sl = prog.enc[0]["prefix_slots"].get(gid)
            if sl is not None:
                slots[wire] = sl
        if not slots:
            return
        ph = P.pp.phases[k]
        reg_w = [wire_of_local(ph.regs[kk]) for kk in range(P.R)]
        thr = [(wire_of_local(lb), f"(tp{k} >> {lb}) & 1u") for lb in ph.threads]
        nl = [(P.n - 1 - p, f"(int)((tbase >> {p}) & 1ull)") for p in P.nbit]
        nt = len(thr)
        w("{")
        w.ind += 1
        # thread-bit factors, prefix products
        for ci, (wr, ix) in enumerate(thr):
            w(f"const float2 f{ci} = {pv(wr, ix)};")
        w("float2 pre0 = make_float2(1.f, 0.f);")
        for ci in range(nt):
            w(f"const float2 pre{ci + 1} = cm(f{ci}.x, f{ci}.y, pre{ci});")
        # register Kronecker product Kr and S = sum conj(lam) Kr
        w(f"float2 S_ = make_float2(0.f, 0.f);")
        w("{")
        w(f"float2 kr[{P.NR}]; kr[0] = make_float2(1.f, 0.f);")
        for kk in range(P.R):
            w(f"{{ const float2 a0 = {pv(reg_w[kk], '0')}, a1 = {pv(reg_w[kk], '1')};")
            for i in range(1 << kk):
                w(f"  kr[{i | (1 << kk)}] = cm(a1.x, a1.y, kr[{i}]); kr[{i}] = cm(a0.x, a0.y, kr[{i}]);")
            w("}")
        for i in range(P.NR):
            w(f"S_ = cjfma(v[1][{i}], kr[{i}], S_);")
        w("}")
        w(f"const float2 Q_ = cm(pre{nt}.x, pre{nt}.y, S_);  // C_thr S")
        # tile-bit wires: warp sum of Q, lane 0 scales by the leave-one-out tile products
        w("float2 cnl_ = make_float2(1.f, 0.f);")
        if nl:
            w("{ float q_[2] = {Q_.x, Q_.y}; warp_sum<NT, 2>(q_);")
            w.block("if ((tid & 31) == 0)")
            for ci, (wr, ix) in enumerate(nl):
                w(f"const float2 g{ci} = {pv(wr, ix)};")
            w("float2 run_ = make_float2(1.f, 0.f);")
            w(f"float2 gp_[{len(nl) + 1}]; gp_[0] = run_;")
            for ci in range(len(nl)):
                w(f"gp_[{ci + 1}] = cm(g{ci}.x, g{ci}.y, gp_[{ci}]);")
            for ci in range(len(nl) - 1, -1, -1):
                wr, ix = nl[ci]
                if wr in slots:
                    w(f"{{ const float2 lo = cm(run_.x, run_.y, gp_[{ci}]); const float2 val = cm(lo.x, lo.y, make_float2(q_[0], q_[1]));")
                    w(f"  const int b_ = {ix}; wacc[{slots[wr]} + 2 * b_] += val.x; wacc[{slots[wr]} + 2 * b_ + 1] += val.y; }}")
                w(f"run_ = cm(g{ci}.x, g{ci}.y, run_);")
            w(f"cnl_ = gp_[{len(nl)}];")
            w.end()
            w("const unsigned FULL_ = 0xffffffffu;" if P.NT >= 32 else f"const unsigned FULL_ = {(1 << P.NT) - 1}u;")
            w("cnl_.x = __shfl_sync(FULL_, cnl_.x, 0); cnl_.y = __shfl_sync(FULL_, cnl_.y, 0); }")
        # thread-bit wires: running suffix over the thread factors
        names = {}
        for ci, (wr, _) in enumerate(thr):
            if wr in slots:
                names[ci] = [P.coup.new(w) for _ in range(4)]
        regn = {}
        for kk in range(P.R):
            if reg_w[kk] in slots:
                regn[kk] = [P.coup.new(w) for _ in range(4)]
        w("{")
        w.ind += 1
        w("const float2 cs_ = cm(cnl_.x, cnl_.y, S_);  // C_nl S")
        w("float2 suf_ = make_float2(1.f, 0.f);")
        for ci in range(nt - 1, -1, -1):
            wr, ix = thr[ci]
            if ci in names:
                nm = names[ci]
                w(f"{{ const float2 lo = cm(suf_.x, suf_.y, pre{ci}); const float2 val = cm(lo.x, lo.y, cs_); const bool b_ = {ix};")
                w(f"  {nm[0]} = b_ ? 0.f : val.x; {nm[1]} = b_ ? 0.f : val.y; {nm[2]} = b_ ? val.x : 0.f; {nm[3]} = b_ ? val.y : 0.f; }}")
            if ci > 0:
                w(f"suf_ = cm(f{ci}.x, f{ci}.y, suf_);")
        # register wires
        w(f"const float2 call_ = cm(cnl_.x, cnl_.y, pre{nt});")
        for kk in range(P.R):
            if kk not in regn:
                continue
            others = [k2 for k2 in range(P.R) if k2 != kk]
            w("{")
            w.ind += 1
            w(f"float2 ko[{1 << (P.R - 1)}]; ko[0] = call_;")
            for t2, k2 in enumerate(others):
                w(f"{{ const float2 a0 = {pv(reg_w[k2], '0')}, a1 = {pv(reg_w[k2], '1')};")
                for i in range(1 << t2):
                    w(f"  ko[{i | (1 << t2)}] = cm(a1.x, a1.y, ko[{i}]); ko[{i}] = cm(a0.x, a0.y, ko[{i}]);")
                w("}")
            w("float2 L0 = make_float2(0.f, 0.f), L1 = make_float2(0.f, 0.f);")
            for i in range(P.NR):
                oi = sum(((i >> k2) & 1) << t2 for t2, k2 in enumerate(others))
                tgt = "L1" if (i >> kk) & 1 else "L0"
                w(f"{tgt} = cjfma(v[1][{i}], ko[{oi}], {tgt});")
            nm = regn[kk]
            w(f"{nm[0]} = L0.x; {nm[1]} = L0.y; {nm[2]} = L1.x; {nm[3]} = L1.y;")
            w.ind -= 1
            w("}")
        w.ind -= 1
        w("}")
        for ci, nm in names.items():
            sl = slots[thr[ci][0]]
            for q in range(4):
                P.coup.add(w, nm[q], sl + q, [])
        for kk, nm in regn.items():
            sl = slots[reg_w[kk]]
            for q in range(4):
                P.coup.add(w, nm[q], sl + q, [])
        P.coup.flush(w)
        w.ind -= 1
        w("}")

    def emit_fwd_phases(end):
        # forward phases carry psi only (the turnaround's lambda is formed after them)
        for k in range(end + 1):
            _emit_ops(w, P, k, False, 1)
            if k < end:
                if rot is not None:
                    rot.exchange(w, P, k, k + 1, [0])
                    if k == end - 1 and mode == MODE_FWD and rot.late:
                        emit_late_issue()
                else:
                    _emit_exchange(w, P, k, k + 1, 1)

    obs = getattr(prog, "obs", None) if mode == MODE_TURN else None

    def obs_parts(k, q):
        """(register-bit mask over register index, thread local-bit mask, tile physical mask, c)
        of the folded observable parity of wire q in layout k."""
        m, c = obs[q]
        ph = P.pp.phases[k]
        rmask = sum(1 << kk for kk in range(P.R) if (m >> P.pbit[ph.regs[kk]]) & 1)
        tmask = sum(1 << lb for lb in ph.threads if (m >> P.pbit[lb]) & 1)
        nmask = sum(1 << p for p in P.nbit if (m >> p) & 1)
        return rmask, tmask, nmask, c

    def emit_obs_signs(k):
        """per-thread sign of every wire's parity: thread bits, tile bits and the constant"""
        for q in range(P.n):
            rmask, tmask, nmask, c = obs_parts(k, q)
            terms = [f"(__popc(tp{k} & {tmask}u) & 1)" if tmask else "0",
                     f"(__popcll(tbase & {nmask}ull) & 1)" if nmask else "0", str(c)]
            w(f"const float sg{q} = ((({' ^ '.join(terms)}) & 1) ? -1.f : 1.f);")

    def emit_wht(init, dst):
        """dst[m] = sum_i (-1)^popc(i & m) x[i] over the 2^R register indices, x[i] = init(i)."""
        w(f"float {dst}[{P.NR}];")
        for i in range(P.NR):
            w(f"{dst}[{i}] = {init(i)};")
        for b in range(P.R):
            for i in range(P.NR):
                if (i >> b) & 1:
                    continue
                jj = i | (1 << b)
                w(f"{{ const float a_ = {dst}[{i}], b_ = {dst}[{jj}]; {dst}[{i}] = a_ + b_; {dst}[{jj}] = a_ - b_; }}")

    def emit_zpart_obs(k):
        w("{")
        w.ind += 1
        emit_obs_signs(k)
        emit_wht(lambda i: f"v[0][{i}].x * v[0][{i}].x + v[0][{i}].y * v[0][{i}].y", "hz_")
        vals = [f"sg{q} * hz_[{obs_parts(k, q)[0]}]" for q in range(P.n)] + ["hz_[0]"]
        vals = [_scaled(P, v_, (0, 0)) for v_ in vals]
        offs = [P.n - 1 - q for q in range(P.n)] + [P.n]
        w("float* zw = s_zw + warp * 32;")
        npad = (-len(vals)) % 8
        if P.NT >= 32 and len(vals) + npad <= 32:
            # reduce-scatter 8 values per call; zero padding goes to the unused tail slots
            pad_offs = list(range(P.n + 1, P.n + 1 + npad))
            vals += ["0.f"] * npad
            offs += pad_offs
            for c0 in range(0, len(vals), 8):
                ov = offs[c0:c0 + 8]
                exprs = []
                for h in (0, 4):
                    o = ov[h:h + 4]
                    d = o[1] - o[0]
                    if all(o[t] == o[0] + d * t for t in range(4)):
                        exprs.append(f"{o[0]} + {d} * lj_")
                    else:
                        exprs.append(f"(lj_ & 2 ? (lj_ & 1 ? {o[3]} : {o[2]}) : (lj_ & 1 ? {o[1]} : {o[0]}))")
                w(f"{{ float a8_[8] = {{{', '.join(vals[c0:c0 + 8])}}}; "
                  f"warp_accumulate8p<NT>(a8_, zw + (hi16_ ? {exprs[1]} : {exprs[0]})); }}")
        else:
            w(f"float pz[{len(vals)}] = {{{', '.join(vals)}}};")
            w(f"warp_sum<NT, {len(vals)}>(pz);")
            w.block("if ((tid & 31) == 0)")
            for e, o in enumerate(offs):
                w(f"zw[{o}] += pz[{e}];")
            w.end()
        w.ind -= 1
        w("}")

    def emit_lambda_obs(k):
        P.sc[1] = P.sc[0]  # lambda = O psi carries psi's deferred scale
        w("{")
        w.ind += 1
        emit_obs_signs(k)
        # o_i = sum_q ws_q (-1)^popc(i & rmask_q): collect ws by register mask, then one WHT
        byr = {}
        for q in range(P.n):
            byr.setdefault(obs_parts(k, q)[0], []).append(q)
        wsum = {m: " + ".join(f"sg{q} * (A.wts ? (float)A.wts[{q}] : 1.f)" for q in qs) for m, qs in byr.items()}
        emit_wht(lambda i: wsum.get(i, "0.f"), "ow_")
        for i in range(P.NR):
            w(f"v[1][{i}] = make_float2(ow_[{i}] * v[0][{i}].x, ow_[{i}] * v[0][{i}].y);")
        w.ind -= 1
        w("}")

    def emit_zpart(k):
        # <Z> partials without block barriers: warp shuffle tree, then lane 0 of each warp adds
        # into its own per-warp slot (indexed by physical bit; [n] = norm). Reduced over warps in
        # fp64 once per CTA, after the tile loop.
        if obs:
            emit_zpart_obs(k)
            return
        ph = P.pp.phases[k]
        w("{")
        w.ind += 1
        w(f"float pz[{P.M + 1}];")
        w(f"for (int e = 0; e <= {P.M}; ++e) pz[e] = 0.f;")
        w("float S_ = 0.f;")
        for kk in range(P.R):
            w(f"float D{kk} = 0.f;")
        for i in range(P.NR):
            w(f"{{ const float pr = v[0][{i}].x * v[0][{i}].x + v[0][{i}].y * v[0][{i}].y; S_ += pr;")
            w("  " + " ".join(f"D{kk} {'-' if (i >> kk) & 1 else '+'}= pr;" for kk in range(P.R)) + " }")
        w(f"pz[{P.M}] = S_;")
        for kk in range(P.R):
            w(f"pz[{ph.regs[kk]}] += D{kk};")
        for j, lb in enumerate(ph.threads):
            w(f"pz[{lb}] += ((tp{k} >> {lb}) & 1u) ? -S_ : S_;")
        if _scaled(P, "1.f", (0, 0)) != "1.f":
            w(f"for (int e_ = 0; e_ <= {P.M}; ++e_) pz[e_] *= {_scaled(P, '1.f', (0, 0))};")
        w(f"warp_sum<NT, {P.M + 1}>(pz);")
        w.block("if ((tid & 31) == 0)")
        w(f"float* zw = s_zw + warp * 32;")
        for e, p in enumerate(P.pbit):
            w(f"zw[{p}] += pz[{e}];")
        for p in P.nbit:
            w(f"zw[{p}] += ((tbase >> {p}) & 1ull) ? -pz[{P.M}] : pz[{P.M}];")
        w(f"zw[{P.n}] += pz[{P.M}];")
        w.end()
        w.ind -= 1
        w("}")

    def emit_lambda_init(k):
        P.sc[1] = P.sc[0]  # lambda = O psi carries psi's deferred scale
        if obs:
            emit_lambda_obs(k)
            return
        ph = P.pp.phases[k]
        w("{")
        w.ind += 1
        wt = lambda p: f"(A.wts ? (float)A.wts[{P.n - 1 - p}] : 1.f)"  # noqa: E731
        terms = []
        for lb in ph.threads:
            p = P.pbit[lb]
            terms.append(f"(((tp{k} >> {lb}) & 1u) ? -{wt(p)} : {wt(p)})")
        for p in P.nbit:
            terms.append(f"(((tbase >> {p}) & 1ull) ? -{wt(p)} : {wt(p)})")
        w(f"const float ob = {' + '.join(terms) if terms else '0.f'};")
        for kk in range(P.R):
            w(f"const float w{kk} = {wt(P.pbit[ph.regs[kk]])};")
        for i in range(P.NR):
            o = " ".join(f"{'-' if (i >> kk) & 1 else '+'} w{kk}" for kk in range(P.R))
            w(f"{{ const float o = ob {o}; v[1][{i}] = make_float2(o * v[0][{i}].x, o * v[0][{i}].y); }}")
        w.ind -= 1
        w("}")

    def emit_late_issue():
        """rot mode: every thread is past its last read of the stage -> prefetch tile t + 1"""
        w("__syncthreads();")
        rot.dirty = set()
        w.block("if (do_load && t + 1 < t_end)")
        emit_issue("t + 1")
        w.end()
        w("cp_async_commit();")

    def emit_bwd_phases():
        if rot is not None and rot.late and top == 0:
            emit_late_issue()
        for k in range(top, -1, -1):
            _emit_ops(w, P, k, True, nv)
            if k > 0:
                if rot is not None:
                    rot.exchange(w, P, k, k - 1, list(range(nv)))
                    if k == 1 and rot.late:
                        emit_late_issue()
                else:
                    _emit_exchange(w, P, k, k - 1, nv)
        P.coup.flush(w)

    def emit_store(k, what):
        q = 0 if what == "psi" else 1
        c = 1.0 / P.sc[q]

        def val(i):
            f = _f(c) if abs(c - 1.0) >= 1e-15 else None
            if P.rho_live:
                f = "rho_" if f is None else f"({f} * rho_)"
            x = f"v[{q}][{i}]" if f is None else f"mx(v[{q}][{i}], {f})"
            return f"cm(phc_.x, phc_.y, {x})" if P.ph_live else x
        if what == "psi":
            w.block("if (flags & PF_STORE_PSI)")
            for i in range(P.NR):
                w(f"__stcs(A.psi_out + base + (gt{k} | {P.goff(k, i)}u), {val(i)});")
            w.end()
        else:
            w.block("if (flags & PF_STORE_LAM)")
            for i in range(P.NR):
                w(f"__stcs(A.lam + base + (gt{k} | {P.goff(k, i)}u), {val(i)});")
            w.end()

    def renormalize(q):
        """bring vector q back to the true scale (a deferred scale would not survive a merge);
        the run-time scale is shared by both vectors, so only the last user may reset it"""
        c = 1.0 / P.sc[q]
        f = _f(c) if abs(c - 1.0) > 1e-15 else None
        if P.rho_live:
            f = "rho_" if f is None else f"({f} * rho_)"
        if f is not None:
            for i in range(P.NR):
                w(f"v[{q}][{i}] = mx(v[{q}][{i}], {f});")
        if P.ph_live:  # only lambda is renormalized (prefix couplings): psi is dead by then
            for i in range(P.NR):
                w(f"v[{q}][{i}] = cm(phc_.x, phc_.y, v[{q}][{i}]);")
            w("phc_ = make_float2(1.f, 0.f);")
            P.ph_live = False
        P.sc[q] = 1.0
        if P.rho_live:
            w("rho_ = 1.f;")
            P.rho_live = False
            P.tan_count = 0

    if mode == MODE_FWD:
        emit_load(0)
        w.block("if (!do_load)")
        emit_synth(0)
        w.end()
        emit_fwd_phases(last)
        w.block("if (flags & PF_ZPART)")
        emit_zpart(last)
        w.end()
        emit_store(last, "psi")
    elif mode == MODE_BWD:
        emit_load(top)
        emit_bwd_phases()
        # stores first: psi is dead before the prefix-boundary couplings (which read lambda only)
        emit_store(0, "psi")
        emit_store(0, "lam")
        if use_prefix:
            renormalize(1)
            emit_prefix_lambda(0)
    else:
        # turnaround: forward phases (unless NOFWD), <Z>, lambda = O psi, adjoint phases
        d0 = set(rot.dirty) if rot is not None else None
        w.block("if (nofwd)")
        emit_load(top)
        w.end()
        d1 = set(rot.dirty) if rot is not None else None
        if rot is not None:
            rot.dirty = set(d0)
        w.block("else")
        w.block("if (do_load)")
        emit_load(0)
        w.end()
        w.block("else")
        emit_synth(0)
        w.end()
        emit_fwd_phases(top)
        renormalize(0)  # the nofwd branch joins with psi at scale 1
        w.end()
        if rot is not None:
            rot.dirty |= d1  # either branch may have run
        emit_zpart(top)
        emit_lambda_init(top)
        emit_bwd_phases()
        emit_store(0, "psi")
        emit_store(0, "lam")
        if use_prefix and len(prog.passes) == 1:
            renormalize(1)
            emit_prefix_lambda(0)
    w.end()  # tile loop
    # flush partials
    w("__syncthreads();")
    if slotf:
        w.block("if (A.part)")
        w(f"double* dst = A.part + (size_t)blockIdx.x * {slotf};")
        w(f"for (int f = tid; f < {slotf}; f += NT) {{ double s = 0.0; for (int ww = 0; ww < NW; ++ww) s += (double)s_acc[ww * {slotf + 8} + f]; dst[f] = s; }}")
        if P.walsh:
            # Walsh component sums -> per-class values S'_e = 2^-ar sum_c V_c (-1)^popc(c & e)
            # (the constant component is dropped: it multiplies Im<lam|psi> = 0)
            w("__syncthreads();")
            for idx, (slot, ar, comps) in enumerate(P.walsh):
                d = 1 << ar
                w.block(f"if (tid == {idx % P.NT})")
                for c in comps:
                    w(f"double V{c} = 0.0; for (int ww = 0; ww < NW; ++ww) V{c} += (double)s_acc[ww * {slotf + 8} + {slot + 2 * c - 1}];")
                for e in range(d):
                    terms = " ".join(f"{'-' if bin(c & e).count('1') & 1 else '+'} V{c}" for c in comps)
                    w(f"dst[{slot + 2 * e}] = 0.0; dst[{slot + 2 * e + 1}] = ({terms}) * {1.0 / d!r};")
                w.end()
        w.end()
    w.block(f"if ((mode == PMODE_TURN || (flags & PF_ZPART)) && A.zpart)")
    w(f"double* dst = A.zpart + (size_t)blockIdx.x * {P.n + 1};")
    w(f"for (int f = tid; f <= {P.n}; f += NT) {{ double s = 0.0; for (int ww = 0; ww < NW; ++ww) s += (double)s_zw[ww * 32 + f]; dst[f] = s; }}")
    w.end()
    out.extend(w.lines)
    out.append("}")
    return "\n".join(out)


def program_modes(prog):
    """(pass, mode) kernels a program needs for forward-only and forward+adjoint calls."""
    L = len(prog.passes)
    need = []
    for pi in range(L):
        need.append((pi, MODE_FWD))
        if pi < L - 1:
            need.append((pi, MODE_BWD))
    need.append((L - 1, MODE_TURN))
    return need


def generate_kernels(prog) -> list:
    """[(pass, mode, name, full NVRTC source)] -- one translation unit per kernel so the
    C side can compile them in parallel."""
    with open(PRIMS) as f:
        prims = f.read()
    if os.environ.get("LSQ_FAST_PHASE") == "1":  # A/B runs: MUFU phases
        prims = "#define LSQ_FAST_PHASE 1\n" + prims
    elif os.environ.get("LSQ_SINCOSPI") == "1":  # A/B runs: CUDA's sincospif
        prims = "#define LSQ_SINCOSPI 1\n" + prims
    elif os.environ.get("LSQ_MUFU_REDUCED") == "1":  # A/B runs: MUFU after exact reduction
        prims = "#define LSQ_MUFU_REDUCED 1\n" + prims
    out = []
    for pi, mode in program_modes(prog):
        out.append((pi, mode, kernel_name(pi, mode), prims + "\n" + emit_kernel(prog, pi, mode) + "\n",
                    stage_alloc(prog, pi, mode)))
    return out


def kernel_set(prog, prog_fwd=None) -> list:
    """[(pass, mode, name, source, stage_vecs, reg_bits)] of a program; with `prog_fwd` (the same
    pass partition compiled with more register bits, see engine.forward_program) the forward
    kernels come from it: 2^R_fwd amplitudes per thread and fewer phase transposes."""
    out = [k + (prog.passes[k[0]].R,) for k in generate_kernels(prog) if prog_fwd is None or k[1] != MODE_FWD]
    if prog_fwd is not None:
        out += [k + (prog_fwd.passes[k[0]].R,) for k in generate_kernels(prog_fwd) if k[1] == MODE_FWD]
    return out


def generate(prog) -> tuple[str, list]:
    """Full NVRTC source (primitives + kernels) and the (pass, mode, name) list."""
    with open(PRIMS) as f:
        prims = f.read()
    parts = [prims, ""]
    names = []
    for pi, mode in program_modes(prog):
        parts.append(emit_kernel(prog, pi, mode))
        parts.append("")
        names.append((pi, mode, kernel_name(pi, mode)))
    return "\n".join(parts), names
