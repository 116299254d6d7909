"""Scheduler + program encoding, validated on the CPU by interpreting the program words
(tests/emulator.py) and comparing with the oracle."""

import numpy as np
import pytest

from conftest import load_golden
from emulator import Emulator
from oracle import layersim_oracle as orc
from paper_2506_04891_b200 import schedule as S
from paper_2506_04891_b200.configs import build_config_circuit, make_workload
from test_oracle import rebuild_random


def _cmp(res, ref, atol=1e-9):
    for k in ("value", "zq", "grads", "encoding_grads"):
        np.testing.assert_allclose(res[k], ref[k], atol=atol, err_msg=k)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("M,R", [(6, 1), (5, 2), (4, 2), (3, 1)])
def test_small_configs_all_tilings(cfg, M, R):
    wl = make_workload(cfg, n=6, batch=3)
    prog = S.compile_circuit(wl.circuit, M=M, R=R)
    res = Emulator(prog).gradient(wl.theta, wl.x, 3, wl.weights)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=3, weights=wl.weights)
    _cmp(res, ref)


@pytest.mark.parametrize("c", range(6))
@pytest.mark.parametrize("M,R", [(5, 2), (4, 2), (3, 2)])
def test_random_circuits(c, M, R):
    gold = load_golden("random_circuits")
    circ = rebuild_random(gold[f"c{c}_spec"])
    prog = S.compile_circuit(circ, M=M, R=R)
    res = Emulator(prog).gradient(gold[f"c{c}_theta"], gold[f"c{c}_x"], 3, gold[f"c{c}_w"])
    _cmp(res, {k[len(f"c{c}_"):]: v for k, v in gold.items() if k.startswith(f"c{c}_")})


def test_forward_state_matches_oracle():
    wl = make_workload(5, n=7, batch=2)
    prog = S.compile_circuit(wl.circuit, M=5, R=2)
    psi = Emulator(prog).forward(wl.theta, wl.x, 2)
    ref = orc.apply_circuit(wl.circuit, wl.theta, wl.x, batch=2)
    np.testing.assert_allclose(psi, ref, atol=1e-9)


@pytest.mark.parametrize("cfg", [2, 4, 5])
def test_forward_register_tiling_same_partition(cfg):
    """The forward kernels' coarser register tiling (engine.forward_program, R=5) keeps the pass
    partition -- groups and tile wires -- and its own phase plan computes the same states."""
    from paper_2506_04891_b200.engine import forward_program

    wl = make_workload(cfg, n=13, batch=2)
    kw = dict(prefix=False, fold=False, split=True)
    p4 = S.compile_circuit(wl.circuit, M=10, R=4, **kw)
    p5 = forward_program(wl.circuit, p4, M=10, **kw)
    assert p5 is not None and all(pp.R == 5 for pp in p5.passes)
    psi = Emulator(p5).forward(wl.theta, wl.x, 2)
    np.testing.assert_allclose(psi, orc.apply_circuit(wl.circuit, wl.theta, wl.x, batch=2), atol=1e-9)


def test_cfg1_full_golden():
    gold = load_golden("cfg1_full")
    wl = make_workload(1)
    prog = S.compile_circuit(wl.circuit)
    res = Emulator(prog).gradient(wl.theta, wl.x, 64, wl.weights)
    _cmp(res, gold)


def test_program_invariants():
    for cfg in range(1, 6):
        prog = S.compile_circuit(build_config_circuit(cfg))
        seen = []
        for pp in prog.passes:
            assert len(pp.tile_wires) == pp.M
            seen += pp.groups
            for i, ph in enumerate(pp.phases):
                assert sorted(ph.regs + ph.threads) == list(range(pp.M))
                if pp.M - pp.R >= S.COAL and i in (0, len(pp.phases) - 1):
                    assert ph.threads[: S.COAL] == list(range(S.COAL))
        assert sorted(seen) == list(range(len(prog.groups)))


@pytest.mark.parametrize("cfg", [2, 5])
def test_isolated_layers_keep_semantics(cfg):
    """Planner variant ISOLATED (own pass boundaries) must not change results."""
    wl = make_workload(cfg, n=6, batch=2)
    iso = [i for i in range(len(wl.circuit.layers)) if i % 3 == 1]
    prog = S.compile_circuit(wl.circuit, M=4, R=2, isolate=iso)
    # no pass mixes an isolated layer's groups with other layers
    for pp in prog.passes:
        layers = {g.layer for gid in pp.groups for g, _ in prog.groups[gid].gates}
        if layers & set(iso):
            assert len(layers) == 1
    res = Emulator(prog).gradient(wl.theta, wl.x, 2, wl.weights)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=2, weights=wl.weights)
    _cmp(res, ref, atol=1e-8)  # isolated RZ layers become diagonal runs: 2^-32-turn angle grid


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("M,R", [(6, 2), (4, 2)])
def test_product_state_prefix(cfg, M, R):
    """The first group of every wire (single-qubit) is synthesized as a product state; its
    gradient comes from Lambda couplings at the prefix boundary."""
    wl = make_workload(cfg, n=6, batch=3)
    prog = S.compile_circuit(wl.circuit, M=M, R=R, prefix=True)
    executed = {gid for pp in prog.passes for gid in pp.groups}
    assert prog.prefix and not (set(prog.prefix.values()) & executed)
    res = Emulator(prog).gradient(wl.theta, wl.x, 3, wl.weights)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=3, weights=wl.weights)
    _cmp(res, ref, atol=1e-8)


@pytest.mark.parametrize("c", range(6))
def test_random_circuits_prefix(c):
    gold = load_golden("random_circuits")
    circ = rebuild_random(gold[f"c{c}_spec"])
    prog = S.compile_circuit(circ, M=4, R=2, prefix=True)
    res = Emulator(prog).gradient(gold[f"c{c}_theta"], gold[f"c{c}_x"], 3, gold[f"c{c}_w"])
    _cmp(res, {k[len(f"c{c}_"):]: v for k, v in gold.items() if k.startswith(f"c{c}_")}, atol=1e-8)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_observable_folding(cfg):
    """Trailing diagonal / permutation groups are folded into the observable."""
    wl = make_workload(cfg, n=6, batch=3)
    prog = S.compile_circuit(wl.circuit, M=4, R=2, prefix=True, fold=True)
    folded = [g.gid for g in prog.groups if g.trailing]
    executed = {gid for pp in prog.passes for gid in pp.groups}
    assert not (set(folded) & executed)
    if cfg in (1, 2, 5):  # circuits ending with a CNOT ring (+ ZZ)
        assert folded
    res = Emulator(prog).gradient(wl.theta, wl.x, 3, wl.weights)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=3, weights=wl.weights)
    _cmp(res, ref, atol=1e-8)


@pytest.mark.parametrize("c", range(6))
def test_random_circuits_folding(c):
    gold = load_golden("random_circuits")
    circ = rebuild_random(gold[f"c{c}_spec"])
    prog = S.compile_circuit(circ, M=4, R=2, prefix=True, fold=True)
    res = Emulator(prog).gradient(gold[f"c{c}_theta"], gold[f"c{c}_x"], 3, gold[f"c{c}_w"])
    _cmp(res, {k[len(f"c{c}_"):]: v for k, v in gold.items() if k.startswith(f"c{c}_")}, atol=1e-8)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("M,R", [(6, 2), (5, 3), (4, 2)])
def test_split_diagonal(cfg, M, R):
    """Diagonal gates split out of one-qubit groups (RZ.RY -> RY + diagonal run), deferred off
    register bits and sunk into runs: same results."""
    wl = make_workload(cfg, n=6, batch=3)
    prog = S.compile_circuit(wl.circuit, M=M, R=R, prefix=True, fold=True, split=True)
    if cfg == 2:  # RY.RZ groups outside the prefix are split
        assert any(g.diag and g.arity == 1 and not g.prefix for g in prog.groups)
    res = Emulator(prog).gradient(wl.theta, wl.x, 3, wl.weights)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=3, weights=wl.weights)
    _cmp(res, ref, atol=1e-8)


@pytest.mark.parametrize("c", range(6))
def test_random_circuits_split(c):
    gold = load_golden("random_circuits")
    circ = rebuild_random(gold[f"c{c}_spec"])
    prog = S.compile_circuit(circ, M=4, R=2, prefix=True, fold=True, split=True)
    res = Emulator(prog).gradient(gold[f"c{c}_theta"], gold[f"c{c}_x"], 3, gold[f"c{c}_w"])
    _cmp(res, {k[len(f"c{c}_"):]: v for k, v in gold.items() if k.startswith(f"c{c}_")}, atol=1e-8)


def test_diagonal_runs_are_sunk():
    """After sinking, no phase has two diagonal runs separated only by groups on other wires."""
    wl = make_workload(2, n=16, batch=1)
    prog = S.compile_circuit(wl.circuit, M=12, R=4, prefix=True, fold=True, split=True)
    for pp in prog.passes:
        for ph in pp.phases:
            kinds = [prog.groups[g].diag for g in ph.ops]
            runs = sum(1 for i, d in enumerate(kinds) if d and (i == 0 or not kinds[i - 1]))
            nd_after = [i for i, d in enumerate(kinds) if not d]
            assert runs <= max(1, len(nd_after)), (kinds,)


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(REF_SRC), reason="reference sources absent (GPU box)")
@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_reference_circuit_objects_compile_by_duck_typing(cfg):
    """The drop-in accepts the REFERENCE's own layersim.Circuit objects: compiled by
    schedule.compile_circuit and interpreted on the CPU, they give the oracle's results for our
    equivalent circuit (the reference package is imported read-only, in this container only)."""
    import importlib
    import sys

    sys.path.insert(0, REF_SRC)
    try:
        ls = importlib.import_module("layersim")
    finally:
        sys.path.remove(REF_SRC)
    wl = make_workload(cfg, n=6, batch=3)
    layers = []
    for layer in wl.circuit.layers:
        pat = ls.WirePattern(ls.PatternKind(layer.pattern.kind.value), layer.pattern.wires)
        role = None if layer.role is None else ls.Role(layer.role.value)
        layers.append(ls.Layer(ls.GateKind(layer.gate.value), pat, role, layer.values))
    rc = ls.Circuit(wl.n, layers)
    assert type(rc).__module__.startswith("layersim")
    prog = S.compile_circuit(rc, M=5, R=2)
    res = Emulator(prog).gradient(wl.theta, wl.x, 3, wl.weights)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=3, weights=wl.weights)
    _cmp(res, ref)


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_all_variants_compile_and_emulate(cfg):
    """The compile of tests/test_gpu_parity.py::test_all_variants_forced_vs_oracle (every
    non-default variant at once: isolated segments whose groups are all synthesized or folded
    leave a segment with nothing to schedule) on the CPU, at n=12 for the pass / phase searches
    and at n=6 on the emulator against the oracle."""
    from paper_2506_04891_b200 import planner as P

    def variants(circ, n):
        K = P.KernelKind
        sel = {K.DIRECT: [], K.SPLIT: [], K.ISOLATED: []}
        for i, layer in enumerate(circ.layers):
            av = P.applicable_variants(layer, n)
            k = K.DIRECT if K.DIRECT in av else K.SPLIT if K.SPLIT in av else K.ISOLATED if i < 6 else None
            if k is not None:
                sel[k].append(i)
        return dict(isolate=sel[K.ISOLATED], direct=sel[K.DIRECT], split_layers=sel[K.SPLIT])

    wl = make_workload(cfg, n=12, batch=1)
    for R in (4, 5):
        prog = S.compile_circuit(wl.circuit, M=9, R=R, prefix=True, fold=True, split=True,
                                 fwd_only=R == 5, **variants(wl.circuit, 12))
        seen = sorted(g for pp in prog.passes for g in pp.groups)
        assert len(seen) == len(set(seen))
    wl = make_workload(cfg, n=6, batch=2)
    prog = S.compile_circuit(wl.circuit, M=4, R=2, prefix=True, fold=True, split=True, **variants(wl.circuit, 6))
    res = Emulator(prog).gradient(wl.theta, wl.x, 2, wl.weights)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=2, weights=wl.weights)
    _cmp(res, ref, atol=1e-8)


def test_rebalance_budget_moves_groups_and_keeps_semantics():
    """A larger pass-rebalancing budget moves groups into later passes (cfg4-shaped circuit) and
    the program still matches the oracle on the emulator."""
    wl = make_workload(4, n=12, batch=1)
    a = S.compile_circuit(wl.circuit, M=8, R=4, prefix=True, fold=True, split=True, rebalance_budget=0.0)
    b = S.compile_circuit(wl.circuit, M=8, R=4, prefix=True, fold=True, split=True, rebalance_budget=400.0)
    assert [sorted(p.groups) for p in a.passes] != [sorted(p.groups) for p in b.passes]
    assert sorted(g for p in b.passes for g in p.groups) == sorted(g for p in a.passes for g in p.groups)
    wl = make_workload(4, n=7, batch=2)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=2, weights=wl.weights)
    for budget in (0.0, 60.0, 400.0):
        prog = S.compile_circuit(wl.circuit, M=4, R=2, prefix=True, fold=True, split=True, rebalance_budget=budget)
        _cmp(Emulator(prog).gradient(wl.theta, wl.x, 2, wl.weights), ref, atol=1e-8)


def test_prefix_group_that_is_also_a_trailing_permutation():
    """SX.SX = X on wires that only permutations / diagonals touch afterwards is both the wire's
    product-state prefix and a trailing permutation: it is synthesized, and must not flip the
    folded observable as well (found by profiles/stress_random.py on the GPU: <Z> off by 2)."""
    from paper_2506_04891_b200.circuits import Circuit, Layer, Role, all_qubits, explicit, ring_pairs
    from paper_2506_04891_b200.gates import GateKind

    n = 6
    circ = Circuit(n, [Layer(GateKind("sx"), all_qubits()), Layer(GateKind("sx"), all_qubits()),
                       Layer(GateKind("ms"), explicit((4, 1), (0, 1), (2, 3)), Role.TRAINABLE),
                       Layer(GateKind("cnot"), ring_pairs()), Layer(GateKind("swap"), explicit((0, 4), (5, 1))),
                       Layer(GateKind("cz"), ring_pairs())])
    rng = np.random.default_rng(3)
    theta = rng.uniform(-3, 3, circ.trainable_count)
    w = rng.normal(size=n)
    ref = orc.gradient(circ, theta, None, batch=2, weights=w)
    for M in (4, 6):
        prog = S.compile_circuit(circ, M=M, R=2, prefix=True, fold=True, split=True)
        assert any(g.prefix and g.perm_ops is not None for g in prog.groups)
        _cmp(Emulator(prog).gradient(theta, None, 2, w), ref, atol=1e-8)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_all_gate_circuits_on_the_emulator(seed):
    """The draw sequence of the GPU stress run (profiles/stress_random.py) on the CPU: random
    circuits of all gate kinds, widths and tilings compiled like the engine does and interpreted
    by the emulator against the oracle (the narrow ones; seed 0 holds the case whose folded
    observable was flipped twice)."""
    from circuit_helpers import random_circuit

    rng = np.random.default_rng(seed)
    checked = 0
    for _ in range(70):
        n = int(rng.integers(6, 13))
        M = int(rng.integers(5, n + 1))
        circ = random_circuit(rng, n, int(rng.integers(6, 18)))
        B = int(rng.integers(1, 4))
        theta = rng.uniform(-3, 3, circ.trainable_count)
        x = rng.uniform(0, 3, (B, circ.encoding_count))
        w = rng.normal(size=n)
        if n > 8:
            continue
        m = min(n, M)
        prog = S.compile_circuit(circ, M=M, R=S.DEFAULT_R_SPECIALISED if m >= 9 else S.default_r(m),
                                 prefix=True, fold=True, split=True)
        _cmp(Emulator(prog).gradient(theta, x, B, w), orc.gradient(circ, theta, x, batch=B, weights=w), atol=1e-7)
        checked += 1
    assert checked >= 20
