"""CPU interpreter of the compiled pass program -- TEST INFRASTRUCTURE.

Executes the int32 program words produced by `paper_2506_04891_b200.schedule` with the
exact semantics the CUDA pass kernel implements (tile gather by tile-bit mask, register-bit
to local-bit decoding per phase, diagonal-run sources REG/THREAD/NONLOCAL, fixed-point
diagonal angles, per-group coupling matrices at the post-group point, W-contraction), in
complex128. Comparing it with the oracle validates the scheduler and the encoding on the
CPU; the GPU tests then compare the kernel with the oracle.
"""

from __future__ import annotations

import numpy as np

from paper_2506_04891_b200 import schedule as S
from paper_2506_04891_b200.gates import GATE_CODE, GateKind, gate_matrix, gate_matrix_derivative

CODE_GATE = {v: k for k, v in GATE_CODE.items()}
SWAP4 = [0, 2, 1, 3]


def _params(gw, fvals, theta, x):
    """Per-gate parameter array: (k,) shared or (B, k) per row."""
    kind = CODE_GATE[int(gw[0])]
    k = int(gw[7])
    if k == 0:
        return kind, None
    cols = []
    perrow = False
    for j in range(k):
        s = int(gw[2 + j])
        if s == S.FIXED_SRC:
            cols.append(fvals[int(gw[5]) + j])
        elif s & S.ENC_FLAG:
            cols.append(x[:, s & ~S.ENC_FLAG])
            perrow = True
        else:
            cols.append(theta[s])
    if perrow:
        B = x.shape[0]
        return kind, np.stack([np.broadcast_to(c, (B,)) for c in cols], axis=-1)
    return kind, np.array(cols, dtype=float)


def group_gate_mats(words, fvals, theta, x, gid):
    grp = S.section(words, S.SEC_GROUPS, S.GROUP_WORDS)[gid]
    gates = S.section(words, S.SEC_GATES, S.GATE_WORDS)
    arity, ng, g0 = int(grp[0]), int(grp[3]), int(grp[4])
    out = []
    for j in range(g0, g0 + ng):
        gw = gates[j]
        kind, p = _params(gw, fvals, theta, x)
        m = gate_matrix(kind, p)
        ders = [gate_matrix_derivative(kind, p, k) for k in range(int(gw[7]))]
        if arity == 2 and int(gw[1]):
            m = m[..., SWAP4, :][..., :, SWAP4]
            ders = [d[..., SWAP4, :][..., :, SWAP4] for d in ders]
        out.append((gw, m, ders))
    return grp, out


def _mm(a, b):
    return np.matmul(a, b)


def group_unitary(words, fvals, theta, x, gid):
    grp, mats = group_gate_mats(words, fvals, theta, x, gid)
    d = 1 << int(grp[0])
    U = np.eye(d, dtype=complex)
    for _, m, _ in mats:
        U = _mm(m, U)
    return U


def _bit(arr, b):
    return (arr >> b) & 1


class Emulator:
    def __init__(self, prog):
        self.prog = prog
        self.w = prog.words
        self.fv = prog.fvals
        self.n = prog.n
        self.passes = S.section(self.w, S.SEC_PASSES, S.PASS_WORDS)
        self.phases = S.section(self.w, S.SEC_PHASES, S.PHASE_WORDS)
        self.ops = S.section(self.w, S.SEC_OPS, S.OP_WORDS)
        self.subs = S.section(self.w, S.SEC_SUBS, S.SUB_WORDS)
        self.groups = S.section(self.w, S.SEC_GROUPS, S.GROUP_WORDS)

    # -- tile geometry -------------------------------------------------------------------
    def tile_index(self, pw):
        n, M = self.n, int(pw[0])
        mask = int(pw[4])
        loc = [p for p in range(n) if mask >> p & 1]
        non = [p for p in range(n) if not mask >> p & 1]
        L = np.arange(1 << M)
        lphys = np.zeros(1 << M, dtype=np.int64)
        for i, p in enumerate(loc):
            lphys |= _bit(L, i) << p
        t = np.arange(1 << (n - M))
        tbase = np.zeros(1 << (n - M), dtype=np.int64)
        for i, p in enumerate(non):
            tbase |= _bit(t, i) << p
        return tbase[:, None] | lphys[None, :], tbase, M

    # -- ops on a tile array (B, ntiles, 2^M) ----------------------------------------------
    @staticmethod
    def _apply_local(v, U, bits):
        """U (d,d) or (B,d,d) on local bits (first = more significant) of v (B,T,2^M)."""
        B, Tn, D = v.shape
        L = np.arange(D)
        if len(bits) == 1:
            (a,) = bits
            i0 = L[_bit(L, a) == 0]
            i1 = i0 | (1 << a)
            x0, x1 = v[:, :, i0].copy(), v[:, :, i1].copy()
            if U.ndim == 2:
                v[:, :, i0] = U[0, 0] * x0 + U[0, 1] * x1
                v[:, :, i1] = U[1, 0] * x0 + U[1, 1] * x1
            else:
                u = U[:, None, None]
                v[:, :, i0] = u[..., 0, 0] * x0 + u[..., 0, 1] * x1
                v[:, :, i1] = u[..., 1, 0] * x0 + u[..., 1, 1] * x1
            return
        a, b = bits
        base = L[(_bit(L, a) == 0) & (_bit(L, b) == 0)]
        idx = [base, base | (1 << b), base | (1 << a), base | (1 << a) | (1 << b)]
        xs = [v[:, :, i].copy() for i in idx]
        for r in range(4):
            acc = 0
            for c in range(4):
                coef = U[r, c] if U.ndim == 2 else U[:, r, c][:, None, None]
                acc = acc + coef * xs[c]
            v[:, :, idx[r]] = acc

    @staticmethod
    def _perm_local(v, kind, a, b=None):
        """X on local bit a, or CX local a -> local b (register-permutation ops)."""
        D = v.shape[2]
        L = np.arange(D)
        if kind == S.OP_PX:
            sel = L[_bit(L, a) == 0]
            dst = sel | (1 << a)
        else:
            sel = L[(_bit(L, a) == 1) & (_bit(L, b) == 0)]
            dst = sel | (1 << b)
        t = v[:, :, sel].copy()
        v[:, :, sel] = v[:, :, dst]
        v[:, :, dst] = t

    @staticmethod
    def _coupling(lam, psi, bits):
        B, Tn, D = psi.shape
        L = np.arange(D)
        if len(bits) == 1:
            (a,) = bits
            i0 = L[_bit(L, a) == 0]
            idx = [i0, i0 | (1 << a)]
        else:
            a, b = bits
            base = L[(_bit(L, a) == 0) & (_bit(L, b) == 0)]
            idx = [base, base | (1 << b), base | (1 << a), base | (1 << a) | (1 << b)]
        d = len(idx)
        Mm = np.empty((B, d, d), dtype=complex)
        for r in range(d):
            for c in range(d):
                Mm[:, r, c] = np.sum(np.conj(lam[:, :, idx[r]]) * psi[:, :, idx[c]], axis=(1, 2))
        return Mm

    def _drun_index(self, sub, pw, phase, tbase, D):
        """Per (tile, local) diag index 0..3 for a DRUN sub-op."""
        regs = phase[:5]
        L = np.arange(D)
        vals = []
        for sw in sub[:2]:
            kind, val = int(sw) >> 8, int(sw) & 0xFF
            if kind == S.SRC_NONE:
                vals.append(None)
            elif kind == S.SRC_REG:
                vals.append(np.broadcast_to(_bit(L, int(regs[val]))[None, :], (len(tbase), D)))
            elif kind == S.SRC_THREAD:
                vals.append(np.broadcast_to(_bit(L, val)[None, :], (len(tbase), D)))
            else:
                vals.append(np.broadcast_to(_bit(tbase, val)[:, None], (len(tbase), D)))
        if vals[1] is None:
            return vals[0]
        return 2 * vals[0] + vals[1]

    def _diag_phases(self, gid, theta, x):
        U = group_unitary(self.w, self.fv, theta, x, gid)
        d = np.diagonal(U, axis1=-2, axis2=-1)
        # device stores angles in 32-bit fixed point turns; emulate that quantisation
        turns = np.angle(d) / (2 * np.pi)
        fx = np.round(turns * 2.0**32).astype(np.int64)
        fx = ((fx + 2**31) % 2**32) - 2**31
        return np.exp(2j * np.pi * fx / 2.0**32)

    # -- one pass --------------------------------------------------------------------------
    def run_pass(self, pi, mode, psi, lam, theta, x, wts, acc, zq):
        pw = self.passes[pi]
        idx, tbase, M = self.tile_index(pw)
        D = 1 << M
        P = psi[:, idx]  # (B, T, D) copy
        Lm = lam[:, idx] if mode == "bwd" else None
        nph, ph0 = int(pw[2]), int(pw[3])
        B = psi.shape[0]

        def ops_of(phase):
            o0, no = int(phase[21]), int(phase[22])
            return self.ops[o0 : o0 + no]

        def fwd_phase(phase):
            regs = phase[:5]
            for op in ops_of(phase):
                kind = int(op[0])
                if kind in (S.OP_PX, S.OP_PCX):
                    self._perm_local(P, kind, int(regs[op[1]]), int(regs[op[2]]) if kind == S.OP_PCX else None)
                elif kind == S.OP_U1:
                    U = group_unitary(self.w, self.fv, theta, x, int(op[3]))
                    self._apply_local(P, U, [int(regs[op[1]])])
                elif kind == S.OP_U2:
                    U = group_unitary(self.w, self.fv, theta, x, int(op[3]))
                    self._apply_local(P, U, [int(regs[op[1]]), int(regs[op[2]])])
                else:
                    for sub in self.subs[int(op[6]) : int(op[6]) + int(op[7])]:
                        ph = self._diag_phases(int(sub[2]), theta, x)  # (d,) or (B,d)
                        ix = self._drun_index(sub, pw, phase, tbase, D)
                        if ph.ndim == 1:
                            P[:] *= ph[ix][None]
                        else:
                            P[:] *= ph[np.arange(B)[:, None, None], ix[None]]

        def bwd_phase(phase, vecs):
            regs = phase[:5]
            Pv, Lv = vecs
            for op in ops_of(phase)[::-1]:
                kind = int(op[0])
                gid = int(op[3]) if int(op[0]) != S.OP_DRUN else -1
                if kind in (S.OP_PX, S.OP_PCX):
                    for v in (Pv, Lv):
                        self._perm_local(v, kind, int(regs[op[1]]), int(regs[op[2]]) if kind == S.OP_PCX else None)
                elif kind in (S.OP_U1, S.OP_U2):
                    bits = [int(regs[op[1]])] + ([int(regs[op[2]])] if kind == S.OP_U2 else [])
                    grp = self.groups[gid]
                    if int(grp[10]):
                        acc[gid] = acc.get(gid, 0) + self._coupling(Lv, Pv, bits)
                    U = group_unitary(self.w, self.fv, theta, x, gid)
                    Ud = np.conj(np.swapaxes(U, -1, -2))
                    self._apply_local(Pv, Ud, bits)
                    self._apply_local(Lv, Ud, bits)
                else:
                    subs = self.subs[int(op[6]) : int(op[6]) + int(op[7])]
                    prod = np.conj(Lv) * Pv
                    for sub in subs:
                        g = int(sub[2])
                        if int(self.groups[g][10]):
                            ix = self._drun_index(sub, pw, phase, tbase, D)
                            nd = 1 << int(sub[5])
                            m = np.zeros((B, nd), dtype=complex)
                            for e in range(nd):
                                m[:, e] = np.sum(np.where(ix[None] == e, prod, 0), axis=(1, 2))
                            acc[g] = acc.get(g, 0) + m
                    for sub in subs[::-1]:
                        ph = np.conj(self._diag_phases(int(sub[2]), theta, x))
                        ix = self._drun_index(sub, pw, phase, tbase, D)
                        f = ph[ix][None] if ph.ndim == 1 else ph[np.arange(B)[:, None, None], ix[None]]
                        Pv *= f
                        Lv *= f

        phases = [self.phases[ph0 + j] for j in range(nph)]
        if mode in ("fwd", "turn"):
            for ph in phases:
                fwd_phase(ph)
        if mode == "turn":
            prob = np.abs(P) ** 2
            # <Z_q> partials and lam = O psi; with a folded observable Z_q reads the parity of
            # (mask_q & j) ^ c_q (trailing permutations)
            full = idx  # (T, D) physical index
            O = np.zeros(full.shape)
            obs = S.section(self.w, S.SEC_OBS, 4) if int(self.w[30]) else None
            for q in range(self.n):
                if obs is None:
                    b = _bit(full, self.n - 1 - q)
                else:
                    m, c = int(obs[q][0]), int(obs[q][1])
                    b = np.zeros_like(full)
                    for pbit in range(self.n):
                        if (m >> pbit) & 1:
                            b ^= _bit(full, pbit)
                    b ^= c
                s = 1.0 - 2.0 * b
                zq[:, q] += np.sum(prob * s[None], axis=(1, 2))
                O += wts[q] * s
            Lm = P * O[None]
        if mode in ("turn", "bwd"):
            for ph in phases[::-1]:
                bwd_phase(ph, (P, Lm))
        psi[:, idx] = P
        if Lm is not None:
            lam[:, idx] = Lm

    # -- product-state prefix ----------------------------------------------------------------
    def prefix_vectors(self, theta, x, batch):
        """v[b, w] = U_w |0> for wires with a prefix group, |0> otherwise (B, n, 2)."""
        v = np.zeros((batch, self.n, 2), dtype=complex)
        v[:, :, 0] = 1
        pre = S.section(self.w, S.SEC_PREFIX, 4) if int(self.w[29]) else []
        for w, row in enumerate(pre):
            gid = int(row[0])
            if gid >= 0:
                U = group_unitary(self.w, self.fv, theta, x, gid)
                v[:, w, :] = U[..., :, 0] if U.ndim == 3 else U[None, :, 0]
        return v

    def product_state(self, v, skip=None):
        B = v.shape[0]
        out = np.ones((B, 1 << self.n), dtype=complex)
        idx = np.arange(1 << self.n)
        for w in range(self.n):
            if w == skip:
                continue
            bit = (idx >> (self.n - 1 - w)) & 1
            out *= v[:, w, :][:, bit]
        return out

    def prefix_lambda(self, v, lam, acc):
        """Couplings of the prefix groups at the prefix boundary:
        Lambda_w(a) = sum_{j: bit_w(j) = a} conj(lam_j) prod_{w' != w} v_w'(bit_w'(j))."""
        pre = S.section(self.w, S.SEC_PREFIX, 4)
        idx = np.arange(1 << self.n)
        for w, row in enumerate(pre):
            gid, slot = int(row[0]), int(row[1])
            if gid < 0 or slot < 0:
                continue
            Q = self.product_state(v, skip=w)
            bit = (idx >> (self.n - 1 - w)) & 1
            L = np.stack([np.sum(np.conj(lam[:, bit == a]) * Q[:, bit == a], axis=1) for a in (0, 1)], axis=1)
            acc[gid] = acc.get(gid, 0) + L

    # -- whole program -----------------------------------------------------------------------
    def gradient(self, theta, x, batch, weights=None):
        n = self.n
        theta = np.zeros(0) if theta is None else np.asarray(theta, float)
        x = np.zeros((batch, 0)) if x is None else np.asarray(x, float)
        wts = np.ones(n) if weights is None else np.asarray(weights, float)
        prefix = bool(int(self.w[29]))
        v = self.prefix_vectors(theta, x, batch) if prefix else None
        if prefix:
            psi = self.product_state(v)
        else:
            psi = np.zeros((batch, 1 << n), dtype=complex)
            psi[:, 0] = 1
        lam = np.zeros_like(psi)
        acc, zq = {}, np.zeros((batch, n))
        Pn = len(self.passes)
        for pi in range(Pn - 1):
            self.run_pass(pi, "fwd", psi, lam, theta, x, wts, acc, zq)
        self.run_pass(Pn - 1, "turn", psi, lam, theta, x, wts, acc, zq)
        for pi in range(Pn - 2, -1, -1):
            self.run_pass(pi, "bwd", psi, lam, theta, x, wts, acc, zq)
        if prefix:
            self.prefix_lambda(v, lam, acc)
        grads = np.zeros((batch, self.prog.trainable_count))
        egrads = np.zeros((batch, self.prog.encoding_count))
        for gid, m in acc.items():
            self._contract(gid, m, theta, x, grads, egrads)
        value = zq @ wts
        return {"value": value, "zq": zq, "grads": grads, "encoding_grads": egrads}

    def forward(self, theta, x, batch, state=None):
        n = self.n
        theta = np.zeros(0) if theta is None else np.asarray(theta, float)
        x = np.zeros((batch, 0)) if x is None else np.asarray(x, float)
        if state is None:
            psi = np.zeros((batch, 1 << n), dtype=complex)
            psi[:, 0] = 1
        else:
            psi = np.array(state, dtype=complex)
        for pi in range(len(self.passes)):
            self.run_pass(pi, "fwd", psi, None, theta, x, None, {}, None)
        return psi

    def _contract(self, gid, m, theta, x, grads, egrads):
        grp, mats = group_gate_mats(self.w, self.fv, theta, x, gid)
        d = 1 << int(grp[0])
        diag = bool(int(grp[1]))
        if int(grp[12]):  # prefix group: M_ab = Lambda(a) v(b), v = U|0>
            U0 = group_unitary(self.w, self.fv, theta, x, gid)
            v = U0[..., :, 0]
            m = m[:, :, None] * (v[:, None, :] if v.ndim == 2 else v[None, None, :])
            diag = False
        if diag:
            mm = np.zeros(m.shape[:1] + (d, d), dtype=complex)
            for e in range(d):
                mm[:, e, e] = m[:, e]
            m = mm
        U = np.eye(d, dtype=complex)
        for _, g, _ in mats:
            U = g @ U
        Ud = np.conj(np.swapaxes(U, -1, -2))
        A = np.eye(d, dtype=complex)
        for j, (gw, g, ders) in enumerate(mats):
            Bm = np.eye(d, dtype=complex)
            for _, g2, _ in mats[j + 1 :]:
                Bm = g2 @ Bm
            for k, dG in enumerate(ders):
                W = Bm @ dG @ A @ Ud
                val = 2.0 * np.real(np.einsum("...ij,bij->b", W, m) if W.ndim == 2 else np.einsum("bij,bij->b", W, m))
                s = int(gw[2 + k])
                if s == S.FIXED_SRC:
                    continue
                if s & S.ENC_FLAG:
                    egrads[:, s & ~S.ENC_FLAG] += val
                else:
                    grads[:, s] += val
            A = g @ A
