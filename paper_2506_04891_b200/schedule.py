"""Host-side circuit compiler: layers -> fused gate groups -> tile passes -> register phases.

This replaces the reference's per-layer applier loop (`core.py:46-72`, `grad.py:169-204`,
one full state pass per gate position, `kernels.py:579-637`) by a schedule that streams the
state through HBM a few times per circuit. The output is a flat int32/float64 "program"
consumed by the sm_100a pass kernel (`csrc/lsq_kernels.cu`) through the C ABI
(`include/layersim_cuda.h`). Everything here is pure Python/numpy, so schedule bugs are
caught on the CPU by `tests/emulator.py`, which interprets the same program words.

Vocabulary
----------
* wire w (reference convention: wire 0 = most significant) sits at physical bit p = n-1-w.
* group   -- a maximal run of gates acting on exactly the same wire set (1q on w, or 2q on
             {a,b}) with nothing else touching those wires in between. One group = one
             local unitary U = G_s...G_1. The backward pass needs ONE coupling matrix per
             group, M_ab = sum conj(lam_a) psi_b at the post-group point; every parameter of
             every gate in the group is then 2 Re sum W_ab M_ab with
             W = (G_s..G_{j+1}) dG_j (G_{j-1}..G_1) U^dag (contracted on device in fp64).
             This generalises the reference's commuting/descending rules (grad.py:102-140).
* pass    -- one HBM round trip over all tiles. A tile is 2^M amplitudes of one row whose
             index bits vary over a set of M physical bits (always including the COAL lowest
             bits, so every 2^COAL x 8 B = 128 B line is read whole). Any non-diagonal group
             of a pass acts only on tile bits; diagonal groups may touch any bits (a bit
             outside the tile is constant over the tile).
* phase   -- inside a pass, each thread holds 2^R amplitudes in registers; the R register
             bits are the only bits a non-diagonal op may touch. Phases are separated by
             a transpose through shared memory. The first and last phase keep the COAL low
             bits on the lanes so global loads/stores are coalesced.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .circuits import positions, slot_table, Role
from .gates import GATE_CODE, GATE_TRAITS, GateKind

import os as _os

# low physical bits always inside a tile (4 -> 16 amplitudes = one 128 B line); LSQ_COAL
# overrides it for tiling experiments (profiles/sweep_tiling.sh)
COAL = int(_os.environ.get("LSQ_COAL", "4"))
MAX_R = 5  # register bits per thread (2^5 = 32 amplitudes per vector per thread)
MAX_M_FWD = 14
MAX_M_BWD = 13
# measured on B200 (profiles/r01/sweep_c2_*.log): 12 tile bits with 16 amplitudes per thread
# per vector balances passes (HBM) against occupancy/exchanges best for the adjoint kernels
DEFAULT_M = 12
DEFAULT_R_SPECIALISED = 4
ENC_FLAG = 1 << 30  # param source tag: encoding column
FIXED_SRC = -1

# op kinds (must match csrc/lsq_program.h)
OP_U1, OP_U2, OP_DRUN, OP_PX, OP_PCX = 1, 2, 3, 4, 5  # PX: X on reg a; PCX: CX reg a -> reg b
# diag source kinds
SRC_NONE, SRC_REG, SRC_THREAD, SRC_NONLOCAL = 0, 1, 2, 3
MAGIC = 0x4C535131  # "LSQ1"

# program word layout sizes
HDR_WORDS = 32
GATE_WORDS = 8
GROUP_WORDS = 16
PASS_WORDS = 24
PHASE_WORDS = 24  # 5 regbits, 16 thrbits, op0, nops, pad
OP_WORDS = 8
SUB_WORDS = 8


def default_r(m: int) -> int:
    """Register bits for a tile of M bits: 32 threads per tile when possible, <=MAX_R."""
    if m <= 1:
        return m
    return max(2, min(MAX_R, m - 5))


# ----------------------------------------------------------------------------- gates


@dataclass
class GateRef:
    kind: GateKind
    wires: tuple
    src: list  # per parameter: FIXED_SRC | t | ENC_FLAG|e
    fixed: list  # fixed values (same length as src)
    layer: int

    @property
    def diag(self) -> bool:
        return GATE_TRAITS[self.kind].diagonal

    @property
    def needs_grad(self) -> bool:
        return any(s != FIXED_SRC for s in self.src)

    @property
    def perrow(self) -> bool:
        return any(s != FIXED_SRC and (s & ENC_FLAG) for s in self.src)


def flatten_gates(circuit) -> list[GateRef]:
    """Gate list in application order with parameter sources bound to slots
    (reference slot layout circuits.py:143-214: start + pos*k + j)."""
    n = circuit.n
    slots = slot_table(circuit)
    out = []
    for li, layer in enumerate(circuit.layers):
        kind = GateKind(layer.gate.value)
        k = GATE_TRAITS[kind].param_count
        pos = positions(layer, n)
        slot = slots[li]
        vals = None
        if layer.values is not None:
            vals = np.asarray(layer.values, dtype=np.float64).reshape(len(pos), k)
        for pi, ws in enumerate(pos):
            src, fixed = [], []
            for j in range(k):
                if slot is None or slot.role is Role.FIXED:
                    src.append(FIXED_SRC)
                    fixed.append(float(vals[pi, j]) if vals is not None else 0.0)
                elif slot.role is Role.TRAINABLE:
                    src.append(slot.start + pi * k + j)
                    fixed.append(0.0)
                else:
                    src.append(ENC_FLAG | (slot.start + pi * k + j))
                    fixed.append(0.0)
            out.append(GateRef(kind, tuple(ws), src, fixed, li))
    return out


# ----------------------------------------------------------------------------- groups


@dataclass
class Group:
    gid: int
    wires: tuple  # group basis order (first wire = more significant local bit)
    gates: list = field(default_factory=list)  # list of (GateRef, reversed: bool)
    prefix: bool = False  # synthesized product-state prefix (not executed by any pass)
    trailing: bool = False  # folded into the observable (not executed, zero gradient)

    @property
    def arity(self) -> int:
        return len(self.wires)

    @property
    def diag(self) -> bool:
        return all(g.diag for g, _ in self.gates)

    @property
    def needs_grad(self) -> bool:
        return any(g.needs_grad for g, _ in self.gates)

    @property
    def perrow(self) -> bool:
        return any(g.perrow for g, _ in self.gates)

    @property
    def mat_floats(self) -> int:
        if self.diag:
            return 1 << self.arity  # fixed-point phase angles, one word each
        # one-qubit: U (8 floats) + its Euler / tangent form (c, t, e^{ia}, e^{ig}, pad)
        return 16 if self.arity == 1 else 32

    @property
    def perm_ops(self):
        """For a parameter-free group whose unitary is a 0/1 permutation matrix: the shortest
        sequence of register primitives ('x', bit) / ('cx', ctrl, tgt) realising it (bit 0 =
        first group wire, the more significant local bit); None otherwise."""
        if any(GATE_TRAITS[g.kind].param_count for g, _ in self.gates):
            return None
        U = group_matrix_host(self)
        d = U.shape[0]
        if not (np.all((np.abs(U) < 1e-12) | (np.abs(U - 1) < 1e-12)) and np.allclose(np.abs(U).sum(0), 1)):
            return None
        target = tuple(int(np.argmax(np.abs(U[:, c]))) for c in range(d))  # |c> -> |target[c]>
        return _perm_sequence(target, self.arity)

    @property
    def slot_floats(self) -> int:
        if not self.needs_grad or self.trailing:
            return 0
        if self.prefix:
            return 4  # Lambda(0), Lambda(1): M_ab = Lambda(a) v(b), v = U|0>
        if self.diag:
            return 2 << self.arity  # complex diagonal of M
        return 8 if self.arity == 1 else 32


def group_matrix_host(grp: Group) -> np.ndarray:
    """Unitary of a parameter-free group in its basis (host fp64)."""
    from .gates import gate_matrix

    d = 1 << grp.arity
    U = np.eye(d, dtype=complex)
    P = np.eye(4)[[0, 2, 1, 3]]
    for g, rev in grp.gates:
        G = gate_matrix(g.kind, g.fixed if g.fixed else None) if GATE_TRAITS[g.kind].param_count else gate_matrix(g.kind)
        if rev:
            G = P @ G @ P
        U = G @ U
    return U


def _perm_sequence(target, arity):
    """BFS over the primitives X_A, X_B, CX(A->B), CX(B->A) on local basis indices."""
    from collections import deque

    d = 1 << arity
    if arity == 1:
        prims = [("x", 0)]
    else:
        prims = [("x", 0), ("x", 1), ("cx", 0, 1), ("cx", 1, 0)]

    def act(p, idx):
        bits = [(idx >> (arity - 1 - k)) & 1 for k in range(arity)]  # bit 0 = first wire (MSB)
        if p[0] == "x":
            bits[p[1]] ^= 1
        else:
            bits[p[2]] ^= bits[p[1]]
        return sum(b << (arity - 1 - k) for k, b in enumerate(bits))

    start = tuple(range(d))
    goal = tuple(target)
    prev = {start: None}
    q = deque([start])
    while q:
        cur = q.popleft()
        if cur == goal:
            break
        for p in prims:
            nxt = tuple(act(p, v) for v in cur)
            if nxt not in prev:
                prev[nxt] = (cur, p)
                q.append(nxt)
    seq = []
    cur = goal
    while prev[cur] is not None:
        cur, p = prev[cur]
        seq.append(p)
    return seq[::-1]


def fuse_groups(gates: list[GateRef]) -> list[Group]:
    groups: list[Group] = []
    last: dict[int, int] = {}
    for g in gates:
        ws = g.wires
        cand = last.get(ws[0])
        ok = cand is not None and set(groups[cand].wires) == set(ws)
        ok = ok and all(last.get(w) == cand for w in ws)
        if ok:
            grp = groups[cand]
            rev = len(ws) == 2 and ws != grp.wires
            grp.gates.append((g, rev))
        else:
            grp = Group(len(groups), tuple(ws), [(g, False)])
            groups.append(grp)
            for w in ws:
                last[w] = grp.gid
    return groups


def _apply_cost(grp: Group, drop_phase: bool = False) -> int:
    """Packed-FMA count per amplitude pair of a one-qubit group in the specialised kernels."""
    from .codegen import phase_normalized, u1_structure

    if drop_phase and not grp.needs_grad and not any(GATE_TRAITS[g.kind].param_count and
                                                     any(s != FIXED_SRC for s in g.src)
                                                     for g, _ in grp.gates):
        U = phase_normalized(group_matrix_host(grp))
        cls = [["0" if abs(z) < 1e-12 else "c" if abs(z.real) > 1e-12 and abs(z.imag) > 1e-12
                else "r" if abs(z.real) > 1e-12 else "i" for z in row] for row in U]
    else:
        cls = u1_structure(grp)[0]
    return sum({"0": 0, "r": 1, "i": 1, "c": 2}[c] for row in cls for c in row)


def split_diagonal(groups: list[Group], keep=(), drop_phase: bool = False, force=()) -> list[Group]:
    """Split one-qubit groups into runs of diagonal and non-diagonal gates when the
    non-diagonal remainder is cheaper to apply (RZ.RY -> real RY + a phase in a diagonal
    run). The diagonal parts then join diagonal runs, where a wire that is not a register bit
    costs no per-amplitude work. Groups in `keep` (product-state prefix) stay whole; groups
    with a gate of a layer in `force` (planner variant SPLIT) are split whatever the cost."""
    force = set(force)
    out: list[Group] = []
    for g in groups:
        runs = []
        for gr in g.gates:
            if runs and runs[-1][0].diag == gr[0].diag:
                runs[-1].append(gr)
            else:
                runs.append([gr[0], gr])
        parts = [r[1:] for r in runs]
        # a diagonal part followed by a non-diagonal one runs where its wire is a register bit
        # (one complex phase per amplitude, charged 4); trailing diagonal parts are deferred
        split = g.gid not in keep and g.arity == 1 and len(parts) > 1
        forced = any(gr.layer in force for gr, _ in g.gates)
        if split and not forced and _os.environ.get("LSQ_SPLIT_FORCE") != "1":
            cost = sum(_apply_cost(Group(0, g.wires, p), drop_phase) if not p[0][0].diag else
                       (4 if k < len(parts) - 1 else 0) for k, p in enumerate(parts))
            split = cost < _apply_cost(g, drop_phase)
        for p in (parts if split else [g.gates]):
            out.append(Group(len(out), g.wires, list(p), g.prefix, g.trailing))
    return out


def group_preds(groups: list[Group]) -> list[set]:
    """Dependency sets: two groups sharing a wire are ordered unless both are diagonal."""
    preds = [set() for _ in groups]
    last_nd: dict[int, int] = {}  # wire -> last non-diagonal group
    diag_since: dict[int, list] = {}  # wire -> diagonal groups after it
    for g in groups:
        for w in g.wires:
            if w in last_nd:
                preds[g.gid].add(last_nd[w])
            if not g.diag:
                preds[g.gid].update(diag_since.get(w, []))
        for w in g.wires:
            if g.diag:
                diag_since.setdefault(w, []).append(g.gid)
            else:
                last_nd[w] = g.gid
                diag_since[w] = []
    return preds


# ----------------------------------------------------------------------------- passes


@dataclass
class PassPlan:
    tile_wires: set
    groups: list  # ordered gids
    M: int = 0
    R: int = 0
    phases: list = field(default_factory=list)  # list of PhasePlan
    local_of_phys: dict = field(default_factory=dict)
    phys_of_local: list = field(default_factory=list)


@dataclass
class PhasePlan:
    regs: list  # local bits held in registers (len R)
    threads: list  # local bits on thread-index bits (len M-R), lane bits first
    ops: list  # list of gids (application order)


def _greedy_pass(order, groups, preds, done, base, M, first_forced=None):
    S = set(base)
    chosen, chosen_set = [], set()
    work = 0
    seq = list(order)
    if first_forced is not None:
        seq.remove(first_forced)
        seq.insert(0, first_forced)
    for gid in seq:
        g = groups[gid]
        if not preds[gid] <= (done | chosen_set):
            continue
        if g.diag:
            chosen.append(gid)
            chosen_set.add(gid)
            continue
        need = set(g.wires) - S
        if len(S) + len(need) <= M:
            S |= need
            chosen.append(gid)
            chosen_set.add(gid)
            work += 1 + len(g.gates)
    if first_forced is not None:
        # restore program order (the forced group had no unscheduled preds)
        pos = {gid: i for i, gid in enumerate(order)}
        chosen.sort(key=lambda x: pos[x])
    return S, chosen, work


PASS_BEAM = int(_os.environ.get("LSQ_PASS_BEAM", "8"))  # 1: greedy pass partition (round 1)


def _search_passes(groups, preds, remaining, done, base, M, seeds):
    """Pass partition with the fewest HBM round trips: beam search over sequences of greedy
    passes (one candidate per seed group, as the greedy partition tries them), ranked by the
    non-diagonal work done so far. The greedy partition takes the heaviest pass at every step,
    which on ladder circuits strands a few groups in extra, nearly empty passes at the end
    (cfg4 at M = 12: 10 passes greedy, 8 searched). Returns [(tile wires, groups)] or None."""
    if not remaining:
        return None
    work = {gid: (0 if groups[gid].diag else 1 + len(groups[gid].gates)) for gid in remaining}
    total = set(remaining)
    states = [(frozenset(done), ())]
    for _depth in range(4 * len(remaining) + 2):
        fin = [st for st in states if total <= st[0]]
        if fin:
            # fewest passes reached: prefer the most even split of the work
            fin.sort(key=lambda st: max((sum(work[g] for g in ch) for _, ch in st[1]), default=0))
            return [(set(S_), list(ch)) for S_, ch in fin[0][1]]
        nxt = {}
        for dn, plan in states:
            rem = [g for g in remaining if g not in dn]
            dset = set(dn)
            cands = [_greedy_pass(rem, groups, preds, dset, base, M)]
            ready = [g for g in rem if preds[g] <= dset and not groups[g].diag][:seeds]
            for gid in ready[1:]:
                cands.append(_greedy_pass(rem, groups, preds, dset, base, M, first_forced=gid))
            for S_, chosen, _w in cands:
                if not chosen:
                    continue
                d2 = dn | frozenset(chosen)
                if d2 not in nxt:
                    nxt[d2] = plan + ((frozenset(S_), tuple(chosen)),)
        if not nxt:
            return None
        ranked = sorted(nxt.items(), key=lambda kv: -sum(work.get(g, 0) for g in kv[0]))
        states = ranked[:PASS_BEAM]
    return None


def schedule_passes(groups, n, M, seeds: int = 12, skip=()) -> list[PassPlan]:
    """Greedy tile-pass partition; tries a few seeds per pass and keeps the one that
    schedules the most non-diagonal work. Groups in `skip` (the synthesized product-state
    prefix) count as already executed."""
    preds = group_preds(groups)
    skip = set(skip)
    remaining = [g.gid for g in groups if g.gid not in skip]
    done: set = set(skip)
    passes = []
    if n <= M:
        return [PassPlan(set(range(n)), remaining, M=n)]
    # wires at the lowest physical bits (coalescing); leave room for one 2-qubit gate
    base = {n - 1 - p for p in range(min(COAL, max(0, M - 2)))}
    plan = _search_passes(groups, preds, remaining, done, base, M, seeds) if PASS_BEAM > 1 else None
    step = 0
    while remaining:
        if plan is not None:
            S, chosen = set(plan[step][0]), list(plan[step][1])
            step += 1
        else:
            best = _greedy_pass(remaining, groups, preds, done, base, M)
            ready_nd = [
                gid for gid in remaining if preds[gid] <= done and not groups[gid].diag
            ][:seeds]
            for gid in ready_nd[1:]:
                cand = _greedy_pass(remaining, groups, preds, done, base, M, first_forced=gid)
                if cand[2] > best[2]:
                    best = cand
            S, chosen, _ = best
        if not chosen:
            raise RuntimeError("scheduler made no progress")
        # fill the tile to exactly M wires with the wires needed soonest
        if len(S) < M:
            for gid in remaining:
                for w in groups[gid].wires:
                    if len(S) < M and w not in S:
                        S.add(w)
            for w in range(n):
                if len(S) < M and w not in S:
                    S.add(w)
        passes.append(PassPlan(S, chosen, M=M))
        done |= set(chosen)
        cs = set(chosen)
        remaining = [g for g in remaining if g not in cs]
    if not passes:  # empty circuit: one pass over the lowest M bits (observables only)
        passes.append(PassPlan({n - 1 - p for p in range(M)}, [], M=M))
    return passes


def _fp_cost(g: Group) -> float:
    """Estimated packed-FP32 ops per amplitude of one group in an adjoint kernel (U^+ on psi and
    lambda plus couplings); forward kernels are about half. Diagonal groups ride on runs."""
    if g.diag:
        return 1.0
    if g.arity == 1:
        return 11.0 if g.needs_grad else 6.0
    return 8.0 if any(GATE_TRAITS[x.kind].param_count for x, _ in g.gates) else 3.0


# adjoint-pass budget in packed ops per amplitude that still hides under its HBM time (3
# vector transfers, 24 B per amplitude, at ~70% of the FP32 and HBM peaks)
REBALANCE_BUDGET = float(_os.environ.get("LSQ_REBALANCE_BUDGET", "40"))
REBALANCE = _os.environ.get("LSQ_REBALANCE", "1") != "0"


def rebalance_passes(passes: list[PassPlan], groups, n: int, budget: float | None = None) -> None:
    """Move work from heavy passes into the light ones after them (in place). The greedy
    partition packs each pass as full as its tile allows, so the last passes of a circuit carry
    little FP32 work and run at the HBM roofline with the FMA pipe mostly idle (cfg4's last two
    adjoint passes: 15% FMA-pipe activity). Walking from the last pass back, a pass whose
    estimated FP32 load is under REBALANCE_BUDGET takes groups from the end of the pass before
    it: a group may move when every group that depends on it is already in a later pass and,
    if it is not diagonal, its wires are tile wires of the receiving pass. Program semantics are
    unchanged (dependencies stay ordered; gids are a topological order)."""
    if len(passes) < 2:
        return
    budget = REBALANCE_BUDGET if budget is None else float(budget)
    succ = [set() for _ in groups]
    for g in groups:
        for p_ in group_preds(groups)[g.gid]:
            succ[p_].add(g.gid)
    where = {gid: i for i, pp in enumerate(passes) for gid in pp.groups}
    for i in range(len(passes) - 1, 0, -1):
        dst, src = passes[i], passes[i - 1]
        load = sum(_fp_cost(groups[x]) for x in dst.groups)
        moved = True
        while moved and load < budget:
            moved = False
            for gid in sorted(src.groups, reverse=True):
                g = groups[gid]
                if any(where.get(sx, -1) <= i - 1 for sx in succ[gid]):
                    continue  # a dependent group stays in this pass or earlier
                if not g.diag and not set(g.wires) <= dst.tile_wires:
                    continue
                c = _fp_cost(g)
                if load + c > budget:
                    continue
                src.groups.remove(gid)
                dst.groups = sorted(dst.groups + [gid])
                where[gid] = i
                load += c
                moved = True
                break
    passes[:] = [pp for pp in passes if pp.groups] or passes[:1]


# ----------------------------------------------------------------------------- phases

# Shared-memory XOR swizzle of the amplitude index: S(L) = L ^ h(L >> 4), h linear into local
# bits 1..3 only. Bit 0 is never swizzled, so the two amplitudes of a register pair on local
# bit 0 stay adjacent and 16-byte aligned: one 16 B shared access moves both.
SWZ_H = [2, 4, 8, 6, 12, 10, 14, 2, 4, 8, 6, 12, 10, 14]


def swz_vec(local_bit: int) -> int:
    """Contribution of local bit to the low-4 bank index of S(L)."""
    if local_bit < 4:
        return 1 << local_bit
    return SWZ_H[local_bit - 4]


def _lane_order(thread_bits, coalesced):
    """Order thread bits so the lowest lanes hit distinct banks: with 8-byte accesses (local bit
    0 on a lane) bit 0 leads and three lanes independent over swizzle bits 1..3 follow; with
    16-byte pair accesses (local bit 0 in registers) the first three lanes are independent."""
    tb = sorted(thread_bits)
    if coalesced:
        return tb  # local bits 0..3 first: contiguous 128 B per half-warp
    chosen, basis = [], []
    rest = list(tb)
    if 0 in rest:
        chosen.append(0)
        rest.remove(0)
    for b in list(rest):
        if len(chosen) == 4:
            break
        v = swz_vec(b) & 14
        for e in basis:
            v = min(v, v ^ e)
        if v:
            basis.append(v)
            basis.sort(reverse=True)
            chosen.append(b)
            rest.remove(b)
    return chosen + rest


PHASE_SEARCH = _os.environ.get("LSQ_PHASE_SEARCH", "1") != "0"
PHASE_BEAM = int(_os.environ.get("LSQ_PHASE_BEAM", "6"))
FIRST_FREE = _os.environ.get("LSQ_FIRST_FREE", "1") != "0"


def _phase_closure(remaining, groups, ipreds, done, regs, loc):
    """Non-diagonal groups of `remaining` (program order) a phase with register bits `regs` can
    run after `done`: in-pass predecessors satisfied and wires on register bits; diagonal groups
    run wherever their predecessors are done (they never need a register bit)."""
    nd, opset = [], set()
    for gid in remaining:
        ip = ipreds[gid]
        if not (ip <= done or ip <= (done | opset)):
            continue
        g = groups[gid]
        if g.diag:
            opset.add(gid)
        elif loc[gid] <= regs:
            opset.add(gid)
            nd.append(gid)
    return nd, opset


def search_phase_registers(pp: PassPlan, groups, preds, n: int, R: int, low: set, last_free: bool,
                           first_free: bool = False):
    """Register-bit sets of the pass's phases, fewest phases first: beam search over all
    R-subsets of the tile's local bits per phase (the greedy scan packs a phase with the first
    groups that fit, which on ladder circuits -- ECR / MS / CNOT chains -- leaves phases with two
    or three groups and pays a transpose of every vector for each). The first phase keeps the
    coalescing bits on lanes; with `last_free` a plan whose last phase does too is preferred
    (forward programs store from it: otherwise an empty phase, i.e. one more transpose, follows).
    Returns a list of register sets, or None (no non-diagonal group / search failed)."""
    from itertools import combinations

    in_pass = set(pp.groups)
    ipreds = {gid: {p for p in preds[gid] if p in in_pass} for gid in pp.groups}
    lop = {p: i for i, p in enumerate(sorted(n - 1 - w for w in pp.tile_wires))}
    nd_all = [gid for gid in pp.groups if not groups[gid].diag]
    if not nd_all:
        return None
    loc = {gid: frozenset(lop[n - 1 - w] for w in groups[gid].wires) for gid in nd_all}
    useful = sorted(set().union(*(loc[g] for g in nd_all)))
    r = min(R, len(useful))
    allsets = [frozenset(c) for c in combinations(useful, r)]
    firstsets = allsets if first_free else [s for s in allsets if not (s & low)]
    if not firstsets:  # fewer than R non-coalescing bits in use: any subset of them
        hi = [b for b in useful if b not in low]
        firstsets = [frozenset(c) for c in combinations(hi, min(r, len(hi)))] if hi else []
    cost = {gid: _fp_cost(groups[gid]) for gid in pp.groups}
    states = [(frozenset(), ())]  # (done groups incl. diagonal ones, plan)
    for depth in range(4 * len(nd_all) + 2):
        fin = [st for st in states if all(g in st[0] for g in nd_all)]
        if fin:
            if last_free:
                fin.sort(key=lambda st: bool(st[1][-1] & low))
            return [set(x) for x in fin[0][1]]
        nxt = {}
        for done, plan in states:
            remaining = [g for g in pp.groups if g not in done]
            for regs in (firstsets if depth == 0 else allsets):
                nd, opset = _phase_closure(remaining, groups, ipreds, done, regs, loc)
                if not nd:
                    continue
                d2 = done | opset
                if d2 not in nxt:
                    nxt[d2] = plan + (regs,)
        if not nxt:
            return None
        ranked = sorted(nxt.items(), key=lambda kv: -sum(cost[g] for g in kv[0]))
        states = ranked[:PHASE_BEAM]
    return None


def schedule_phases(pp: PassPlan, groups, preds, n: int, R: int, last_free: bool = False) -> None:
    M = pp.M
    phys = sorted(n - 1 - w for w in pp.tile_wires)
    pp.phys_of_local = phys
    pp.local_of_phys = {p: i for i, p in enumerate(phys)}
    loc = lambda w: pp.local_of_phys[n - 1 - w]  # noqa: E731
    coal = COAL if (M - R) >= COAL else 0
    low = set(range(coal))
    in_pass = set(pp.groups)
    # forward-only programs read their tile from the prefetch stage, where any layout is as
    # good as another: only the LAST phase (global stores) must keep the coalescing bits on lanes
    first_free = bool(last_free and FIRST_FREE and M <= 13)

    def build(plan):
        """phases [[register bits, ops]] with the greedy scan (plan None) or with the register
        bits of every phase given by the searched plan"""
        remaining = list(pp.groups)
        done: set = set()
        phases = []
        first = True
        while remaining:
            fixed = plan[len(phases)] if plan is not None and len(phases) < len(plan) else None
            regs: set = set()
            ops = []
            opset = set()
            for gid in remaining:
                g = groups[gid]
                if not {p for p in preds[gid] if p in in_pass} <= (done | opset):
                    continue
                if g.diag:
                    ops.append(gid)
                    opset.add(gid)
                    continue
                need = {loc(w) for w in g.wires} - regs
                if fixed is not None:  # searched plan: the phase's register bits are given
                    if {loc(w) for w in g.wires} <= fixed:
                        regs |= need
                        ops.append(gid)
                        opset.add(gid)
                    continue
                if first and need & low and not first_free:
                    continue
                if len(regs) + len(need) <= R:
                    regs |= need
                    ops.append(gid)
                    opset.add(gid)
            if not ops and not first:
                raise RuntimeError("phase scheduler made no progress")
            ops = _defer_diagonal(ops, regs, remaining, groups,
                                  lambda w: pp.local_of_phys.get(n - 1 - w, -1))
            opset = set(ops)
            phases.append([regs, ops])
            done |= opset
            remaining = [g for g in remaining if g not in opset]
            first = False
        if not phases:
            phases.append([set(), []])
        if coal and (phases[-1][0] & low):
            phases.append([set(), []])
        if coal and (phases[0][0] & low) and not first_free:  # cannot happen (first-phase rule)
            phases.insert(0, [set(), []])
        return phases

    ff, first_free = first_free, False
    phases = build(None)
    if PHASE_SEARCH and len(phases) > 2:
        # transposes a kernel pays: forward-only programs store from the last phase (an empty
        # coalescing phase counts); adjoint kernels read their tile from the stage in any
        # layout, so an empty last phase costs them nothing
        cost = (lambda ph: len(ph)) if last_free else (lambda ph: len(ph) - (not ph[-1][1]))
        for free in ((False, True) if ff else (False,)):
            first_free = free
            plan = search_phase_registers(pp, groups, preds, n, R, low, last_free, free)
            if plan is not None:
                cand = build(plan)
                if cost(cand) < cost(phases):
                    phases = cand
    out = []
    for i, (regs, ops) in enumerate(phases):
        ops = _sink_diagonal(ops, groups)
        coalesced = coal and (i == 0 or i == len(phases) - 1) and not (set(regs) & low)
        regs = sorted(regs)
        pool = [b for b in range(M) if b not in regs and not (coalesced and b in low)]
        # pad register bits, preferring high local bits (keeps low bits on lanes)
        for b in sorted(pool, reverse=True):
            if len(regs) >= R:
                break
            regs.append(b)
        assert len(regs) == R, (regs, R, M)
        threads = [b for b in range(M) if b not in regs]
        threads = _lane_order(threads, coalesced)
        out.append(PhasePlan(regs, threads, ops))
    pp.phases = out
    pp.R = R


def _defer_diagonal(ops, regs, remaining, groups, loc):
    """Drop from this phase the diagonal groups that touch one of its register bits when
    nothing later in the phase needs them and a later phase exists: applied in a phase where
    their wires are thread or tile bits, their phase is one value per thread."""
    nd_left = any(not groups[g].diag for g in remaining if g not in ops)
    if not nd_left:
        return ops
    keep = []
    for idx, gid in enumerate(ops):
        g = groups[gid]
        if g.diag and {loc(w) for w in g.wires} & regs:
            later = ops[idx + 1:]
            if not any(not groups[x].diag and set(groups[x].wires) & set(g.wires) for x in later):
                continue
        keep.append(gid)
    return keep


def _sink_diagonal(ops, groups):
    """Move every diagonal group as late as its wires allow (before the next non-diagonal
    group sharing a wire, else to the end) so diagonal groups form long runs (one DRUN)."""
    nd = [g for g in ops if not groups[g].diag]
    slots: dict = {}  # index into nd (or len(nd)) -> diagonal groups placed before it
    for idx, gid in enumerate(ops):
        g = groups[gid]
        if not g.diag:
            continue
        pos = len(nd)
        seen_nd = sum(1 for x in ops[:idx] if not groups[x].diag)
        for k in range(seen_nd, len(nd)):
            if set(groups[nd[k]].wires) & set(g.wires):
                pos = k
                break
        slots.setdefault(pos, []).append(gid)
    out = []
    for k in range(len(nd) + 1):
        out += slots.get(k, [])
        if k < len(nd):
            out.append(nd[k])
    return out


# ----------------------------------------------------------------------------- program


@dataclass
class Program:
    n: int
    groups: list
    passes: list
    trainable_count: int
    encoding_count: int
    slot_base: dict  # gid -> global float offset of its coupling slot
    slot_total: int
    words: np.ndarray = None
    fvals: np.ndarray = None
    M: int = 0
    gates: list = None
    enc: list = None  # per pass: ops per phase, subs, table sizes (consumed by codegen)
    rowidx: dict = None  # gid -> per-row table index

    @property
    def n_passes(self) -> int:
        return len(self.passes)


def prefix_groups(groups) -> dict:
    """wire -> gid of its product-state prefix group: the FIRST group touching the wire when it
    is a single-qubit group. Applied to |0..0> these groups give the product state
    (x)_w U_w|0>, which the first pass synthesizes instead of executing them."""
    first: dict = {}
    for g in groups:
        for w in g.wires:
            first.setdefault(w, g)
    return {w: g.gid for w, g in first.items() if g.arity == 1}


def trailing_groups(groups) -> tuple[list, list]:
    """Groups after which only diagonal or parameter-free permutation groups touch their wires.
    Returns (trailing gids, the trailing permutation groups in application order).

    Trailing diagonal groups commute with the observable sum_q w_q Z_q: they change neither
    <Z_q> nor any gradient (theirs are structurally zero). Trailing permutations relabel the
    basis: Z_q measured after them is the parity (-1)^(a_q . j + c_q) of the state before them.
    """
    nt_wires: set = set()
    trailing = []
    for g in reversed(groups):
        foldable = g.diag or g.perm_ops is not None
        if foldable and not (set(g.wires) & nt_wires):
            trailing.append(g.gid)
        else:
            nt_wires |= set(g.wires)
    tset = set(trailing)
    perms = [g for g in groups if g.gid in tset and not g.diag]
    return sorted(tset), perms


def observable_masks(perms, n: int):
    """Affine GF(2) map of the trailing permutations: for every wire q, (mask_q, c_q) over
    PHYSICAL index bits such that bit_q(pi(j)) = parity(mask_q & j) ^ c_q."""
    rows = [1 << w for w in range(n)]  # rows[w]: set of source wires (bit w') feeding wire w
    const = [0] * n
    for g in perms:
        for prim in g.perm_ops:
            if prim[0] == "x":
                const[g.wires[prim[1]]] ^= 1
            else:
                c, t = g.wires[prim[1]], g.wires[prim[2]]
                rows[t] ^= rows[c]
                const[t] ^= const[c]
    masks = []
    for q in range(n):
        m = 0
        for w in range(n):
            if (rows[q] >> w) & 1:
                m |= 1 << (n - 1 - w)
        masks.append((m, const[q]))
    return masks


def compile_circuit(circuit, M: int | None = None, R: int | None = None, isolate=(),
                    prefix: bool = False, fold: bool = False, split: bool = False, direct=(),
                    split_layers=(), fwd_only: bool = False, rebalance_budget: float | None = None) -> Program:
    """Compile a (reference-compatible) circuit into a pass program.

    Planner variants (layer indices): `isolate` -- executed with pass boundaries of their own
    (ISOLATED): their gates fuse only among themselves and share no pass with other layers;
    `direct` -- one-qubit groups containing a gate of these layers are applied in the direct
    8-op form, not the Euler tangent form (DIRECT); `split_layers` -- one-qubit groups with a
    gate of these (diagonal) layers are split into diagonal runs and the rest (SPLIT).
    `fwd_only`: the program only provides forward kernels (engine.forward_program), so the phase
    search prefers plans whose LAST phase keeps the coalescing bits on lanes (forward stores).
    `rebalance_budget`: estimated FP32 load (packed ops per amplitude) up to which a pass takes
    groups from the pass before it (rebalance_passes); None = REBALANCE_BUDGET. A plan carries the
    value the planner measured best for its circuit.
    """
    n = int(circuit.n)
    gates = flatten_gates(circuit)
    if M is None:
        M = min(n, DEFAULT_M)
    M = min(M, n)
    iso = set(int(i) for i in isolate)
    # segments of consecutive layers: each isolated layer alone, maximal runs of the others
    segs, cur, cur_key = [], [], None
    for g in gates:
        key = ("iso", g.layer) if g.layer in iso else ("run",)
        if cur and key != cur_key:
            segs.append(cur)
            cur = []
        cur.append(g)
        cur_key = key
    if cur or not segs:
        segs.append(cur)
    groups, passes = [], []
    pre: dict = {}
    obs = None
    for si, seg in enumerate(segs):
        grp = fuse_groups(seg)
        if split:
            grp = split_diagonal(grp, set(prefix_groups(grp).values()) if (prefix and si == 0) else (),
                                 drop_phase=fold, force=split_layers)
        preds = group_preds(grp)
        skip = set()
        if prefix and si == 0:
            pre = prefix_groups(grp)
            skip |= set(pre.values())
        if fold and si == len(segs) - 1:
            tr, perms = trailing_groups(grp)
            # a permutation group that is also its wire's product-state prefix (e.g. SX.SX = X on
            # a wire only permutations touch afterwards) is synthesized, not folded: it must not
            # flip the observable a second time
            perms = [g for g in perms if g.gid not in skip]
            tr = [g for g in tr if g not in skip]
            skip |= set(tr)
            obs = observable_masks(perms, n)
            for gid in tr:
                grp[gid].trailing = True
        seg_passes = schedule_passes(grp, n, M, skip=skip) if (grp or not passes) else []
        if REBALANCE and not (prefix and si == 0 and len(segs) > 1):
            rebalance_passes(seg_passes, grp, n, rebalance_budget)
        need2 = any(g.arity == 2 and not g.diag for g in grp)
        for pp in seg_passes:
            r = default_r(pp.M) if R is None else min(R, pp.M)
            if need2 and r < 2:
                r = min(2, pp.M)
            schedule_phases(pp, grp, preds, n, r, last_free=fwd_only)
        off = len(groups)
        for g in grp:
            g.gid += off
        for pp in seg_passes:
            pp.groups = [x + off for x in pp.groups]
            for ph in pp.phases:
                ph.ops = [x + off for x in ph.ops]
        groups += grp
        passes += seg_passes
    for w, gid in pre.items():
        groups[gid].prefix = True
    if passes:
        # the prefix groups' couplings are produced by the last adjoint pass (pass 0)
        passes[0].prefix_groups = [gid for w, gid in sorted(pre.items())]
    slot_base, total = {}, 0
    for pp in passes:
        for gid in pp.groups + getattr(pp, "prefix_groups", []):
            g = groups[gid]
            if g.slot_floats:
                slot_base[gid] = total
                total += g.slot_floats
    T = getattr(circuit, "trainable_count", None)
    E = getattr(circuit, "encoding_count", None)
    if T is None:
        from .circuits import Circuit

        c2 = Circuit(circuit.n, circuit.layers)
        T, E = c2.trainable_count, c2.encoding_count
    prog = Program(n, groups, passes, T, E, slot_base, total, M=M, gates=gates)
    prog.isolate = tuple(sorted(iso))
    prog.direct_layers = frozenset(int(i) for i in direct)
    prog.split_layers = tuple(sorted(int(i) for i in split_layers))
    prog.rebalance_budget = rebalance_budget
    prog.prefix = {w: gid for w, gid in pre.items()}
    prog.obs = obs
    prog.drop_phase = bool(fold)  # gradient program: global phases of constant groups dropped
    encode(prog)
    return prog


def _src_word(gw, src):
    return src


def encode(prog: Program) -> None:
    """Serialise the program (layout documented in include/layersim_cuda.h)."""
    n = prog.n
    gates_w, fvals = [], []
    group_w = []
    gate_index = 0
    rowidx = 0
    for g in prog.groups:
        g0 = gate_index
        for gate, rev in g.gates:
            src = list(gate.src) + [FIXED_SRC] * (3 - len(gate.src))
            fixed = list(gate.fixed) + [0.0] * (3 - len(gate.fixed))
            foff = len(fvals)
            fvals.extend(fixed)
            gates_w.append([GATE_CODE[gate.kind], int(rev), src[0], src[1], src[2], foff, g.gid, len(gate.src)])
            gate_index += 1
        wa = g.wires[0]
        wb = g.wires[1] if g.arity == 2 else -1
        group_w.append(
            [g.arity, int(g.diag), int(g.perrow), len(g.gates), g0, wa, wb,
             prog.slot_base.get(g.gid, -1), g.slot_floats, g.mat_floats, int(g.needs_grad),
             rowidx if g.perrow else -1, int(g.prefix), 0, 0, 0]
        )
        rowidx += int(g.perrow)
    pass_w, phase_w, op_w, sub_w, pgrp_w = [], [], [], [], []
    prog.enc = []
    prog.rowidx = {}
    ri = 0
    for g in prog.groups:
        if g.perrow:
            prog.rowidx[g.gid] = ri
            ri += 1
    for pi, pp in enumerate(prog.passes):
        # per-pass shared-memory tables: group matrices, coupling slots (float offsets)
        mat_off, slot_off = {}, {}
        mo = so = 0
        for gid in pp.groups:
            g = prog.groups[gid]
            mat_off[gid] = mo
            mo += g.mat_floats
            if g.slot_floats:
                slot_off[gid] = so
                so += g.slot_floats
        for gid in getattr(pp, "prefix_groups", []):
            g = prog.groups[gid]
            if g.slot_floats:
                slot_off[gid] = so
                so += g.slot_floats
        pg0 = len(pgrp_w)
        for gid in pp.groups:
            pgrp_w.append([gid, mat_off[gid], slot_off.get(gid, -1), 0])
        tile_mask = 0
        for p in pp.phys_of_local:
            tile_mask |= 1 << p
        ph0 = len(phase_w)
        first_slot = min((prog.slot_base[g] for g in pp.groups + getattr(pp, "prefix_groups", [])
                          if g in prog.slot_base), default=0)
        enc = {"ops": [], "subs": sub_w, "matf": mo, "slotf": so,
               "pgroups": [(gid, mat_off[gid]) for gid in pp.groups],
               "prefix_slots": {gid: slot_off[gid] for gid in getattr(pp, "prefix_groups", [])
                                if gid in slot_off}}
        prog.enc.append(enc)
        for ph in pp.phases:
            op0 = len(op_w)
            reg_of_local = {b: k for k, b in enumerate(ph.regs)}
            ops = list(ph.ops)
            i = 0
            while i < len(ops):
                g = prog.groups[ops[i]]
                perm = g.perm_ops if not g.diag else None
                if perm is not None:
                    regs_of = [reg_of_local[pp.local_of_phys[n - 1 - w]] for w in g.wires]
                    for p in perm:
                        if p[0] == "x":
                            op_w.append([OP_PX, regs_of[p[1]], -1, g.gid, -1, -1, 0, 0])
                        else:
                            op_w.append([OP_PCX, regs_of[p[1]], regs_of[p[2]], g.gid, -1, -1, 0, 0])
                    i += 1
                    continue
                if not g.diag:
                    if g.arity == 1:
                        a = reg_of_local[pp.local_of_phys[n - 1 - g.wires[0]]]
                        b = -1
                        kind = OP_U1
                    else:
                        a = reg_of_local[pp.local_of_phys[n - 1 - g.wires[0]]]
                        b = reg_of_local[pp.local_of_phys[n - 1 - g.wires[1]]]
                        kind = OP_U2
                    op_w.append([kind, a, b, g.gid, slot_off.get(g.gid, -1), mat_off[g.gid], 0, 0])
                    i += 1
                    continue
                # maximal run of consecutive diagonal groups -> one DRUN op
                s0 = len(sub_w)
                while i < len(ops) and prog.groups[ops[i]].diag:
                    gd = prog.groups[ops[i]]
                    srcs = []
                    for w in gd.wires:
                        p = n - 1 - w
                        if p in pp.local_of_phys:
                            lb = pp.local_of_phys[p]
                            if lb in reg_of_local:
                                srcs.append((SRC_REG << 8) | reg_of_local[lb])
                            else:
                                srcs.append((SRC_THREAD << 8) | lb)
                        else:
                            srcs.append((SRC_NONLOCAL << 8) | p)
                    if len(srcs) == 1:
                        srcs.append(SRC_NONE << 8)
                    sub_w.append([srcs[0], srcs[1], gd.gid, mat_off[gd.gid], slot_off.get(gd.gid, -1), gd.arity, 0, 0])
                    i += 1
                op_w.append([OP_DRUN, -1, -1, -1, -1, -1, s0, len(sub_w) - s0])
            enc["ops"].append([list(r) for r in op_w[op0:]])
            regs = list(ph.regs) + [0] * (MAX_R - len(ph.regs))
            thr = list(ph.threads) + [0] * (16 - len(ph.threads))
            phase_w.append(regs + thr + [op0, len(op_w) - op0, 0])
        ops_lo = int(phase_w[ph0][21]) if pp.phases else len(op_w)
        subs_lo = min((r[6] for r in op_w[ops_lo:] if r[0] == OP_DRUN), default=len(sub_w))
        pass_w.append(
            [pp.M, pp.R, len(pp.phases), ph0, tile_mask, len(pp.groups), pg0, mo, so,
             first_slot, ops_lo, len(op_w) - ops_lo, subs_lo, len(sub_w) - subs_lo]
            + [0] * (PASS_WORDS - 14)
        )
    # prefix section: per wire, the pass-0 slot offset of its prefix group's Lambda (-1: none or
    # no gradient needed) and its gid (-1: no prefix group, the factor is |0>)
    pre = getattr(prog, "prefix", {}) or {}
    pslots = prog.enc[0]["prefix_slots"] if prog.enc else {}
    prefix_w = [[pre.get(w, -1), pslots.get(pre.get(w, -1), -1), 0, 0] for w in range(n)] if pre else []
    obs = getattr(prog, "obs", None)
    obs_w = [[m, c, 0, 0] for (m, c) in obs] if obs else []
    hdr = [0] * HDR_WORDS
    sections = [gates_w, group_w, pass_w, phase_w, op_w, sub_w, pgrp_w, prefix_w, obs_w]
    widths = [GATE_WORDS, GROUP_WORDS, PASS_WORDS, PHASE_WORDS, OP_WORDS, SUB_WORDS, 4, 4, 4]
    hdr[0] = MAGIC
    hdr[1] = 1
    hdr[2] = n
    hdr[3] = prog.trainable_count
    hdr[4] = prog.encoding_count
    hdr[5] = prog.slot_total
    hdr[6] = len(prog.passes)
    hdr[7] = len(prog.groups)
    hdr[28] = rowidx  # number of per-row (encoding) groups
    hdr[29] = int(bool(pre))  # product-state prefix synthesized by the first pass
    hdr[30] = int(bool(obs))  # observable folded through trailing permutations (section 8)
    off = HDR_WORDS
    flat = []
    for si, (sec, wd) in enumerate(zip(sections, widths)):
        hdr[8 + 2 * si] = off
        hdr[9 + 2 * si] = len(sec)
        for row in sec:
            assert len(row) == wd, (si, row)
            flat.extend(row)
        off += wd * len(sec)
    words = np.array(hdr + flat, dtype=np.int64)
    assert words.min() >= -(2**31) and words.max() < 2**31
    prog.words = words.astype(np.int32)
    prog.fvals = np.asarray(fvals if fvals else [0.0], dtype=np.float64)


def section(words: np.ndarray, idx: int, width: int) -> np.ndarray:
    off, cnt = int(words[8 + 2 * idx]), int(words[9 + 2 * idx])
    return words[off : off + cnt * width].reshape(cnt, width)


SEC_GATES, SEC_GROUPS, SEC_PASSES, SEC_PHASES, SEC_OPS, SEC_SUBS, SEC_PGROUPS, SEC_PREFIX, SEC_OBS = range(9)
SEC_WIDTH = [GATE_WORDS, GROUP_WORDS, PASS_WORDS, PHASE_WORDS, OP_WORDS, SUB_WORDS, 4, 4, 4]


def describe(prog: Program) -> str:
    lines = [f"n={prog.n} groups={len(prog.groups)} passes={len(prog.passes)} slot_floats={prog.slot_total}"]
    for i, pp in enumerate(prog.passes):
        nd = sum(1 for g in pp.groups if not prog.groups[g].diag)
        lines.append(
            f"  pass {i}: M={pp.M} R={pp.R} phases={len(pp.phases)} groups={len(pp.groups)} (non-diag {nd}) "
            f"wires={sorted(pp.tile_wires)}"
        )
    return "\n".join(lines)
