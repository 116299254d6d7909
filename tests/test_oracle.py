"""Pin the CPU oracle (oracle/layersim_oracle.py) against the reference's own outputs.

Golden fixtures come from running the reference itself (tests/golden/make_golden.py).
Known-answer values repeat the reference test-suite's pins (test_acceptance.py:104-141,
test_kernels.py:196-220, test_core.py:68-78, test_grad.py:24-39, test_gates.py:32-132).
"""

import ast

import numpy as np
import pytest

from conftest import load_golden
from oracle import layersim_oracle as orc
from paper_2506_04891_b200 import gates as G
from paper_2506_04891_b200.circuits import Circuit, Layer, PatternKind, Role, WirePattern, all_qubits
from paper_2506_04891_b200.configs import make_workload


def test_gate_matrices_match_reference():
    kv = load_golden("known_answers")
    for g in G.GateKind:
        cnt = G.GATE_TRAITS[g].param_count
        p = kv.get(f"gate_{g.value}_params")
        ref = kv[f"gate_{g.value}"]
        np.testing.assert_allclose(orc.gate_matrix(g.value, p), ref, atol=1e-14)
        np.testing.assert_allclose(G.gate_matrix(g, p), ref, atol=1e-14)
        for k in range(cnt):
            dref = kv[f"dgate_{g.value}_{k}"]
            np.testing.assert_allclose(orc.gate_derivative(g.value, p, k), dref, atol=1e-13)
            np.testing.assert_allclose(G.gate_matrix_derivative(g, p, k), dref, atol=1e-13)


def _perm_from_oracle(layer, n):
    """sigma with psi'[j] = psi[sigma[j]], read off basis-state images (bit-exact)."""
    c = Circuit(n, [layer])
    eye = np.eye(1 << n, dtype=complex)
    out = orc.apply_circuit(c, state=eye)  # row i = image of |i>
    sigma = np.empty(1 << n, dtype=np.int64)
    for i in range(1 << n):
        (j,) = np.nonzero(out[i])
        assert out[i, j[0]] == 1.0
        sigma[j[0]] = i
    return sigma


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8])
def test_cnot_ring_permutation_bit_exact(n):
    kv = load_golden("known_answers")
    from paper_2506_04891_b200.circuits import ring_pairs

    sig = _perm_from_oracle(Layer(G.GateKind.CNOT, ring_pairs()), n)
    np.testing.assert_array_equal(sig, kv[f"sigma_cnot_ring_{n}"])


def test_x_and_swap_permutations():
    from paper_2506_04891_b200.circuits import explicit

    kv = load_golden("known_answers")
    np.testing.assert_array_equal(_perm_from_oracle(Layer(G.GateKind.X, all_qubits()), 2), kv["sigma_x_all_2"])
    np.testing.assert_array_equal(
        _perm_from_oracle(Layer(G.GateKind.SWAP, explicit((0, 2))), 3), kv["sigma_swap_02_3"]
    )
    np.testing.assert_array_equal(kv["sigma_x_all_2"], [3, 2, 1, 0])


def test_z_weights_and_k_matrix():
    kv = load_golden("known_answers")
    np.testing.assert_array_equal(orc.z_diag(3), kv["z_weights_3"])
    np.testing.assert_array_equal(orc.z_diag(3), [3, 1, 1, -1, 1, -1, -1, -3])
    for w in range(3):  # K_RZ[i, w] = 1 - 2 bit of wire w (wire 0 = MSB)
        e = np.zeros(3)
        e[w] = 1
        np.testing.assert_array_equal(orc.z_diag(3, e), kv["k_rz_3"][:, w])


@pytest.mark.parametrize("name", ["rzz_ring", "ms_chain", "ecr_explicit", "cnot_ring", "rot_all"])
def test_layer_unitaries(name):
    kv = load_golden("known_answers")
    spec = {
        "rzz_ring": (G.GateKind.RZZ, WirePattern(PatternKind.RING_PAIRS), Role.TRAINABLE),
        "ms_chain": (G.GateKind.MS, WirePattern(PatternKind.CHAIN_PAIRS), Role.TRAINABLE),
        "ecr_explicit": (G.GateKind.ECR, WirePattern(PatternKind.EXPLICIT, ((2, 0), (1, 3))), None),
        "cnot_ring": (G.GateKind.CNOT, WirePattern(PatternKind.RING_PAIRS), None),
        "rot_all": (G.GateKind.ROT, all_qubits(), Role.TRAINABLE),
    }[name]
    layer = Layer(*spec)
    c = Circuit(4, [layer])
    p = kv[f"layer_{name}_params"]
    theta = p.reshape(-1) if p.size else None
    out = orc.apply_circuit(c, theta, state=np.eye(16, dtype=complex))
    np.testing.assert_allclose(out.T, kv[f"layer_{name}"], atol=1e-13)


def _check(res, gold, atol=1e-10):
    np.testing.assert_allclose(res["value"], gold["value"], atol=atol)
    np.testing.assert_allclose(res["zq"], gold["zq"], atol=atol)
    np.testing.assert_allclose(res["grads"], gold["grads"], atol=atol)
    np.testing.assert_allclose(res["encoding_grads"], gold["encoding_grads"], atol=atol)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_small_configs_match_reference(cfg):
    gold = load_golden(f"small_cfg{cfg}")
    wl = make_workload(cfg, n=6, batch=3)
    np.testing.assert_array_equal(wl.x, gold["x"])
    np.testing.assert_array_equal(wl.theta, gold["theta"])
    np.testing.assert_array_equal(wl.weights, gold["weights"])
    res = orc.gradient(wl.circuit, wl.theta, wl.x, batch=3, weights=wl.weights)
    _check(res, gold)


def test_cfg1_full_matches_reference():
    gold = load_golden("cfg1_full")
    wl = make_workload(1)
    res = orc.gradient(wl.circuit, wl.theta, wl.x, batch=64, weights=wl.weights)
    _check(res, gold)


def rebuild_random(spec_str, n=5):
    spec = ast.literal_eval(str(spec_str))
    layers = []
    for gate, pk, wires, role, values in spec:
        layers.append(
            Layer(
                G.GateKind(gate),
                WirePattern(PatternKind(pk), wires),
                None if role is None else Role(role),
                values,
            )
        )
    return Circuit(n, layers)


@pytest.mark.parametrize("c", range(6))
def test_random_circuits_match_reference(c):
    gold = load_golden("random_circuits")
    circ = rebuild_random(gold[f"c{c}_spec"])
    res = orc.gradient(circ, gold[f"c{c}_theta"], gold[f"c{c}_x"], batch=3, weights=gold[f"c{c}_w"])
    _check(res, {k[len(f"c{c}_"):]: v for k, v in gold.items() if k.startswith(f"c{c}_")})


def test_single_ry_analytic():
    c = Circuit(1, [Layer(G.GateKind.RY, all_qubits(), Role.TRAINABLE)])
    for th in (0.3, np.pi / 2, 2.1):
        r = orc.gradient(c, np.array([th]))
        assert r["value"][0] == pytest.approx(np.cos(th), abs=1e-12)
        assert r["grads"][0, 0] == pytest.approx(-np.sin(th), abs=1e-12)


def test_rz_on_basis_state_zero_gradient():
    c = Circuit(2, [Layer(G.GateKind.RZ, all_qubits(), Role.TRAINABLE)])
    r = orc.gradient(c, np.array([0.4, -1.1]))
    np.testing.assert_allclose(r["grads"], 0.0, atol=1e-14)
    assert r["value"][0] == pytest.approx(2.0)
