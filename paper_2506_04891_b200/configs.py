"""The five BASELINE.json workloads as reference-IR circuits plus their seeded inputs.

Layer lists follow SURVEY §0.2 (verified there against the reference IR). Decisions on the
BASELINE ambiguities (recorded in DESIGN.md):

* A1 -- "ZZ on all adjacent pairs" is the CHAIN pattern (n-1 pairs); `zz_pattern="ring"`
  switches it.
* A4 -- cfg4's encoding x is drawn from U[0, pi) like the others.
* A5 -- `np.random.default_rng(1000 + cfg)`, draw order: x (B x E), then the trainable
  vector (T, slot order, U[-pi, pi) radians), then the loss weights w ~ N(0, 1) (n).
* GPi / GPi2 angles are drawn in radians (BASELINE wording) and handed to the API in the
  reference's unit, turns (phi / 2 pi); MS(0,0) is the reference MS with fixed (0, 0, 0.25).
* Every input is rounded to float32 once; the engine and the oracle both receive
  float64(float32(.)) so input rounding is never counted as an error.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .circuits import Circuit, Layer, Role, all_qubits, chain_pairs, explicit, ring_pairs
from .gates import GateKind

TR, ENC, FIX = Role.TRAINABLE, Role.ENCODING, Role.FIXED


@dataclass(frozen=True)
class Workload:
    index: int
    name: str
    n: int
    batch: int
    circuit: Circuit
    x: np.ndarray  # (batch, E) float64 of float32 values
    theta: np.ndarray  # (T,) float64 of float32 values, API units
    weights: np.ndarray  # (n,) float64 of float32 values


def _pairs(n: int, start: int):
    return explicit(*[(q, q + 1) for q in range(start, n - 1, 2)])


def build_config_circuit(cfg: int, n: int | None = None, zz_pattern: str = "chain") -> Circuit:
    """Circuit of BASELINE config `cfg` (1-based), optionally at a reduced width `n`."""
    zz = chain_pairs() if zz_pattern == "chain" else ring_pairs()
    if cfg == 1:
        n = 8 if n is None else n
        layers = [Layer(GateKind.RY, all_qubits(), ENC)]
        for _ in range(2):
            layers += [
                Layer(GateKind.RX, all_qubits(), TR),
                Layer(GateKind.RZ, all_qubits(), TR),
                Layer(GateKind.CNOT, ring_pairs()),
            ]
    elif cfg == 2:
        n = 16 if n is None else n
        layers = [Layer(GateKind.RY, all_qubits(), ENC)]
        for _ in range(4):
            layers += [
                Layer(GateKind.RY, all_qubits(), TR),
                Layer(GateKind.RZ, all_qubits(), TR),
                Layer(GateKind.CNOT, ring_pairs()),
            ]
        layers.append(Layer(GateKind.RZZ, zz, TR))
    elif cfg == 3:
        n = 20 if n is None else n
        even, odd = _pairs(n, 0), _pairs(n, 1)
        ms = ((0.0, 0.0, 0.25),)
        layers = [Layer(GateKind.RY, all_qubits(), ENC)]
        for _ in range(3):
            layers += [
                Layer(GateKind.GPI2, all_qubits(), TR),
                Layer(GateKind.GPI, all_qubits(), TR),
                Layer(GateKind.MS, even, FIX, ms * len(even.wires)),
                Layer(GateKind.MS, odd, FIX, ms * len(odd.wires)),
            ]
    elif cfg == 4:
        n = 22 if n is None else n
        even, odd = _pairs(n, 0), _pairs(n, 1)
        layers = [Layer(GateKind.SX, all_qubits()), Layer(GateKind.RZ, all_qubits(), ENC)]
        for _ in range(4):
            layers += [
                Layer(GateKind.RZ, all_qubits(), TR),
                Layer(GateKind.SX, all_qubits()),
                Layer(GateKind.RZ, all_qubits(), TR),
                Layer(GateKind.ECR, even),
                Layer(GateKind.ECR, odd),
            ]
    elif cfg == 5:
        n = 24 if n is None else n
        layers = [Layer(GateKind.RY, all_qubits(), ENC)]
        for _ in range(6):
            layers += [
                Layer(GateKind.RX, all_qubits(), TR),
                Layer(GateKind.RY, all_qubits(), TR),
                Layer(GateKind.RZ, all_qubits(), TR),
                Layer(GateKind.CNOT, ring_pairs()),
                Layer(GateKind.RZZ, zz, TR),
            ]
    else:
        raise ValueError(f"unknown config {cfg}")
    return Circuit(n, layers)


# (encoding/head layers, layers per repeated block, blocks) of each config circuit
BLOCK_LAYOUT = {1: (1, 3, 2), 2: (1, 3, 4), 3: (1, 4, 3), 4: (2, 5, 4), 5: (1, 5, 6)}

CONFIG_SHAPES = {1: (8, 64), 2: (16, 512), 3: (20, 128), 4: (22, 256), 5: (24, 1024)}
CONFIG_NAMES = {
    1: "cfg1_n8_b64_rx_rz_cnotring",
    2: "cfg2_n16_b512_ry_rz_cnotring_zz",
    3: "cfg3_n20_b128_ionq_gpi2_gpi_ms",
    4: "cfg4_n22_b256_ibm_rz_sx_ecr",
    5: "cfg5_n24_b1024_rx_ry_rz_cnotring_zz",
}


def _turn_slots(circuit: Circuit) -> np.ndarray:
    """Boolean mask over the trainable vector: slots whose gate takes turns."""
    mask = np.zeros(circuit.trainable_count, dtype=bool)
    for i, layer in enumerate(circuit.layers):
        s = circuit.layer_slot(i)
        if s is not None and s.role is Role.TRAINABLE and layer.gate in (
            GateKind.GPI,
            GateKind.GPI2,
            GateKind.MS,
        ):
            mask[s.start : s.start + s.count] = True
    return mask


def make_workload(
    cfg: int, n: int | None = None, batch: int | None = None, zz_pattern: str = "chain"
) -> Workload:
    """Seeded inputs for config `cfg` (A5). A reduced `n`/`batch` keeps the draw order,
    so the first rows of a reduced batch equal the first rows of the full one."""
    n0, b0 = CONFIG_SHAPES[cfg]
    n = n0 if n is None else n
    batch = b0 if batch is None else batch
    circ = build_config_circuit(cfg, n, zz_pattern)
    rng = np.random.default_rng(1000 + cfg)
    x = rng.uniform(0.0, np.pi, (b0 if batch <= b0 else batch, circ.encoding_count))[:batch]
    theta = rng.uniform(-np.pi, np.pi, circ.trainable_count)
    turns = _turn_slots(circ)
    theta = np.where(turns, theta / (2.0 * np.pi), theta)
    w = rng.standard_normal(n)
    f = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    return Workload(cfg, CONFIG_NAMES[cfg], n, batch, circ, f(x), f(theta), f(w))
