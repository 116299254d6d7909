"""Planner: CUDA-variant selection logic with injected measurements, Plan JSON format
(reference planner.py:165-309 and tests/test_planner.py strategy: fake clocks/tables)."""

import json
import warnings

import numpy as np
import pytest

from paper_2506_04891_b200 import planner as P
from paper_2506_04891_b200.circuits import Circuit, Layer, Role, all_qubits, explicit, ring_pairs
from paper_2506_04891_b200.configs import build_config_circuit
from paper_2506_04891_b200.core import plan_kernels
from paper_2506_04891_b200.errors import PlanMismatchError
from paper_2506_04891_b200.gates import GateKind


def _table(iso_faster=(), tile=None):
    tile = tile or {10: 3.0, 11: 2.0, 12: 1.0, 13: 1.5}

    def measure(layer, k):
        if layer is None:
            return P.TimingStats(tile.get(k, 5.0), 0.0, 10, 3)
        g = layer.gate.value
        if k is P.KernelKind.ISOLATED:
            return P.TimingStats(0.5 if g in iso_faster else 2.0, 0.0, 10, 3)
        return P.TimingStats(1.0, 0.0, 10, 3)

    return measure


def test_build_plan_argmin_and_tile_bits():
    c = build_config_circuit(2, n=14)
    plan = P.build_plan(c, 8, measure=_table(iso_faster=("rzz",)))
    assert plan.tile_bits == 12
    for layer, k in zip(c.layers, plan.assignments):
        assert k is (P.KernelKind.ISOLATED if layer.gate is GateKind.RZZ else P.KernelKind.FUSED)
    # every layer has a measurement for every applicable variant
    assert len(plan.measurements) == sum(len(P.applicable_variants(l, c.n)) for l in c.layers)


def test_variant_space_per_gate_kind():
    """FUSED/ISOLATED everywhere, DIRECT for one-qubit non-diagonal gates (Euler/tangent form
    off), SPLIT for one-qubit diagonal gates (forced diagonal runs)."""
    K = P.KernelKind
    n = 4
    av = lambda g, pat=None: P.applicable_variants(Layer(g, pat or all_qubits(), Role.TRAINABLE  # noqa: E731
                                                         if P.gate_traits(g).param_count else None), n)
    assert av(GateKind.RY) == (K.FUSED, K.ISOLATED, K.DIRECT)
    assert av(GateKind.RZ) == (K.FUSED, K.ISOLATED, K.SPLIT)
    assert av(GateKind.CNOT, ring_pairs()) == (K.FUSED, K.ISOLATED)
    assert av(GateKind.X) == (K.FUSED, K.ISOLATED)


def test_variants_change_the_program():
    """SPLIT forces the diagonal split of the groups it touches; DIRECT is recorded for the
    codegen (both compile to valid programs the emulator runs like the default)."""
    from emulator import Emulator
    from oracle import layersim_oracle as orc
    from paper_2506_04891_b200.configs import make_workload
    from paper_2506_04891_b200.schedule import compile_circuit

    wl = make_workload(4, n=6, batch=2)
    rz = [i for i, l in enumerate(wl.circuit.layers) if l.gate is GateKind.RZ and l.role is Role.TRAINABLE]
    sx = [i for i, l in enumerate(wl.circuit.layers) if l.gate is GateKind.SX]
    base = compile_circuit(wl.circuit, M=4, R=2, split=True)
    forced = compile_circuit(wl.circuit, M=4, R=2, split=True, split_layers=rz, direct=sx)
    assert len(forced.groups) > len(base.groups)
    assert forced.direct_layers == frozenset(sx)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=2, weights=wl.weights)
    res = Emulator(forced).gradient(wl.theta, wl.x, 2, wl.weights)
    np.testing.assert_allclose(res["grads"], ref["grads"], atol=1e-9)


def test_tie_break_prefers_declaration_order():
    c = build_config_circuit(1)

    def measure(layer, k):
        return P.TimingStats(1.0, 0.0, 3, 1)

    plan = P.build_plan(c, 4, measure=measure)
    assert all(k is P.KernelKind.FUSED for k in plan.assignments)
    assert plan.tile_bits == 8  # n=8: all candidates clamp to 8


def test_signature_includes_explicit_wires():
    c = Circuit(4, [Layer(GateKind.CNOT, explicit((0, 1))), Layer(GateKind.CNOT, explicit((2, 3)))])
    assert P.layer_signature(c.layers[0], 4) != P.layer_signature(c.layers[1], 4)
    seen = []

    def measure(layer, k):
        if layer is not None:
            seen.append(layer.pattern.wires)
        return P.TimingStats(1.0, 0.0, 1, 0)

    P.build_plan(c, 2, measure=measure)
    assert ((0, 1),) in seen and ((2, 3),) in seen


def test_plan_json_roundtrip_and_errors(tmp_path):
    c = build_config_circuit(5, n=8)
    plan = P.build_plan(c, 2, P.Objective.FORWARD_BACKWARD, measure=_table(iso_faster=("cnot",)))
    again = P.plan_roundtrip(plan)
    assert again == plan
    assert plan.rebalance_budget is None  # an injected measure leaves the default budget
    doc = json.loads(P.serialize_plan(plan))
    assert set(doc) >= {"machine_id", "n", "batch", "objective", "assignments", "measurements", "tile_bits"}
    # the measured pass-rebalancing budget travels with the plan; plans without one still parse
    import dataclasses

    with_b = dataclasses.replace(plan, rebalance_budget=160.0)
    assert P.plan_roundtrip(with_b) == with_b and P.plan_roundtrip(with_b).rebalance_budget == 160.0
    assert P.parse_plan(json.dumps({k: v for k, v in doc.items() if k != "rebalance_budget"})).rebalance_budget is None
    with pytest.raises(ValueError):
        P.parse_plan(json.dumps({k: v for k, v in doc.items() if k != "n"}))
    bad = dict(doc)
    bad["assignments"] = doc["assignments"][1:]
    with pytest.raises(ValueError):
        P.parse_plan(json.dumps(bad))
    path = tmp_path / "plan.json"
    P.save_plan(plan, path)
    foreign = dict(doc)
    foreign["machine_id"] = "somewhere-else"
    path.write_text(json.dumps(foreign))
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        loaded = P.load_plan(path)
    assert loaded.assignments == plan.assignments
    assert any("timings may not transfer" in str(x.message) for x in w)


def test_plan_validation_against_circuit():
    c = build_config_circuit(1)
    plan = P.build_plan(c, 4, measure=_table())
    assert plan_kernels(c, plan) == list(plan.assignments)
    other = build_config_circuit(1, n=6)
    with pytest.raises(PlanMismatchError):
        plan_kernels(other, plan)
    short = P.Plan(plan.machine_id, plan.n, plan.batch, plan.objective, plan.assignments[:-1], ())
    with pytest.raises(PlanMismatchError):
        plan_kernels(c, short)


def test_timing_stats_validation():
    with pytest.raises(ValueError):
        P.TimingStats(1.0, 0.0, 0, 0)
    with pytest.raises(ValueError):
        P.TimingStats(-1.0, 0.0, 1, 0)


def test_plan_for_tile_bits_roundtrip_and_validation():
    circ = build_config_circuit(2)
    plan = P.plan_for_tile_bits(circ, 16, 11)
    assert plan.tile_bits == 11 and all(k is P.KernelKind.FUSED for k in plan.assignments)
    assert plan_kernels(circ, plan) == list(plan.assignments)
    assert P.plan_roundtrip(plan) == plan
    assert P.tiling_of(plan, circ) == (11, None)
