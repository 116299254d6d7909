"""Benchmark harness over the CUDA engine (the reference's `layersim bench`, bench.py:1-248,
SURVEY §8(f) rank 3): the four circuit families, a correctness gate, forward / backward /
total timings per (n, batch), and the same two CSV reports -- the timing rows with GPU columns
added, and the per-layer-signature variant choices ("crossover" file).

Differences from the reference, all forced by the engine: timings are CUDA events on the
engine's stream (device time of one call, inputs already on the device); the correctness gate
compares the planned program with the default one on the device to complex64 rounding
(1e-5 on amplitudes and gradients instead of 1e-12: both are complex64 computations that fuse
gates differently); the plan is the CUDA-variant plan of `planner.build_plan`.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .circuits import Circuit, Layer, Role, all_qubits, chain_pairs, ring_pairs
from .errors import CapacityError, CorrectnessError
from .gates import GateKind
from .planner import Objective, TimingStats, build_plan, layer_signature, load_plan

FAMILIES = ("vq", "qdi", "ibm", "ionq")

# the reference's columns (bench.py:41-52), then the GPU ones
CSV_COLUMNS = ("family", "n", "batch", "phase", "plan_source", "mean_s", "std_s", "reps", "warmup", "seed",
               "device", "tile_bits", "passes", "evals_per_s")
CROSSOVER_COLUMNS = ("family", "n", "batch", "gate", "pattern", "role", "kernel")
CORRECTNESS_TOL = 1e-5


@dataclass(frozen=True)
class BenchConfig:
    family: str
    qubits: tuple
    batches: tuple
    blocks: int = 8
    reps: int = 10
    warmup: int = 3
    objective: Objective = Objective.FORWARD
    seed: int = 0
    out: str = "results.csv"
    plan_path: str | None = None

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown family {self.family!r}")
        if self.blocks < 1:
            raise ValueError("blocks must be at least 1")
        if not self.qubits or not self.batches:
            raise ValueError("need at least one qubit count and one batch size")


def build_circuit(family: str, n: int, blocks: int = 8) -> Circuit:
    """The reference's four benchmark families (bench.py:81-124): vq / qdi (initial RY + CNOT
    ring, then blocks of RZ / RY / CNOT ring; vq encodes in the first block's RZ only, qdi in
    every block's), ibm (RZ enc, SX, RZ, X, ECR chain) and ionq (RZ enc, GPI2, RZ, GPI, RZZ ring)."""
    if family not in FAMILIES:
        raise ValueError(f"unknown family {family!r}")
    if n < 2:
        raise ValueError("benchmark families need n >= 2")
    if blocks < 1:
        raise ValueError("blocks must be at least 1")
    L = []
    if family in ("vq", "qdi"):
        L += [Layer(GateKind.RY, all_qubits(), Role.TRAINABLE), Layer(GateKind.CNOT, ring_pairs())]
        for b in range(blocks):
            enc = family == "qdi" or b == 0
            L += [Layer(GateKind.RZ, all_qubits(), Role.ENCODING if enc else Role.TRAINABLE),
                  Layer(GateKind.RY, all_qubits(), Role.TRAINABLE), Layer(GateKind.CNOT, ring_pairs())]
    elif family == "ibm":
        for _ in range(blocks):
            L += [Layer(GateKind.RZ, all_qubits(), Role.ENCODING), Layer(GateKind.SX, all_qubits()),
                  Layer(GateKind.RZ, all_qubits(), Role.TRAINABLE), Layer(GateKind.X, all_qubits()),
                  Layer(GateKind.ECR, chain_pairs())]
    else:
        for _ in range(blocks):
            L += [Layer(GateKind.RZ, all_qubits(), Role.ENCODING), Layer(GateKind.GPI2, all_qubits(), Role.TRAINABLE),
                  Layer(GateKind.RZ, all_qubits(), Role.TRAINABLE), Layer(GateKind.GPI, all_qubits(), Role.TRAINABLE),
                  Layer(GateKind.RZZ, ring_pairs(), Role.TRAINABLE)]
    return Circuit(n, L)


def draw_params(circuit: Circuit, batch: int, seed: int, n: int):
    """Parameters drawn like the reference (bench.py:127-136): default_rng([seed, n, batch])."""
    rng = np.random.default_rng([seed, n, batch])
    tr = rng.uniform(-np.pi, np.pi, circuit.trainable_count) if circuit.trainable_count else None
    enc = rng.uniform(-np.pi, np.pi, (batch, circuit.encoding_count)) if circuit.encoding_count else None
    return tr, enc


def _time_cuda(fn, reps: int, warmup: int, timer=None) -> TimingStats:
    import torch

    for _ in range(warmup):
        fn()
    samples = np.empty(reps)
    for r in range(reps):
        if timer is None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            samples[r] = e0.elapsed_time(e1) / 1e3
        else:
            torch.cuda.synchronize()
            t0 = timer()
            fn()
            torch.cuda.synchronize()
            samples[r] = timer() - t0
    return TimingStats(float(samples.mean()), float(samples.std()), reps, warmup)


def crossover_path(out) -> str:
    p = Path(out)
    return str(p.with_name(p.stem + "_crossover" + p.suffix))


def _crossover_rows(circuit, plan, family, n, batch):
    seen, rows = set(), []
    for layer, k in zip(circuit.layers, plan.assignments):
        sig = layer_signature(layer, n)
        if sig in seen:
            continue
        seen.add(sig)
        rows.append([family, n, batch, layer.gate.value, layer.pattern.kind.value,
                     "" if layer.role is None else layer.role.value, k.value])
    return rows


def _write_csv(path, header, rows) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(header)
        w.writerows(rows)


def run_benchmark(config: BenchConfig, timer=None) -> list:
    """The sweep: per (n, batch) a plan (saved file or build_plan), the correctness gate
    (planned vs default program on the device), then forward / backward / total timed; writes
    the CSV and its crossover companion, returns the data rows. Capacity overflows are reported
    and skipped; a failed gate aborts (reference run_benchmark, bench.py:172-248)."""
    import sys

    import torch

    from .core import _engine
    from .planner import machine_id

    rows, cross = [], []
    device = machine_id().split("|")[0]
    for n in config.qubits:
        for batch in config.batches:
            try:
                circuit = build_circuit(config.family, n, config.blocks)
                tr, enc = draw_params(circuit, batch, config.seed, n)
                if config.plan_path is not None:
                    plan, source = load_plan(config.plan_path), "file"
                else:
                    plan = build_plan(circuit, batch, objective=config.objective, timer=timer, reps=config.reps,
                                      warmup=config.warmup, seed=config.seed)
                    source = "autotuned"
                planned = _engine(circuit, plan, None, prefix=False)
                default = _engine(circuit, None, None, prefix=False)
                a, _, _ = planned.forward(tr, enc, batch=batch)
                b, _, _ = default.forward(tr, enc, batch=batch)
                gap = float((a - b).abs().max())
                ga = _engine(circuit, plan, None).fwd_bwd(tr, enc, batch=batch)["grads"]
                gb = _engine(circuit, None, None).fwd_bwd(tr, enc, batch=batch)["grads"]
                if ga is not None:
                    gap = max(gap, float((ga - gb).abs().max()))
                if gap > CORRECTNESS_TOL:
                    raise CorrectnessError(f"planned vs default outputs differ by {gap:.3e} "
                                           f"(family={config.family} n={n} batch={batch})")
            except CapacityError as exc:
                print(f"skipping family={config.family} n={n} batch={batch}: {exc}", file=sys.stderr)
                continue
            th = None if tr is None else torch.as_tensor(tr, device=planned.device)
            x = None if enc is None else torch.as_tensor(enc, device=planned.device)
            final, _, _ = planned.forward(th, x, batch=batch)
            gengine = _engine(circuit, plan, None)
            phases = {
                "forward": lambda: planned.forward(th, x, batch=batch),
                "backward": lambda: planned.backward_from_state(th, x, final),
                "total": lambda: gengine.fwd_bwd(th, x, batch=batch, rows=False, encoding_grads=False),
            }
            for phase, fn in phases.items():
                st = _time_cuda(fn, config.reps, config.warmup, timer)
                rows.append([config.family, n, batch, phase, source, st.mean_seconds, st.std_seconds,
                             config.reps, config.warmup, config.seed, device, planned.program.passes[0].M,
                             len(planned.program.passes), batch / st.mean_seconds if st.mean_seconds else ""])
            cross.extend(_crossover_rows(circuit, plan, config.family, n, batch))
    rows.sort(key=lambda r: (r[0], r[1], r[2], r[3]))
    cross.sort(key=lambda r: tuple(str(v) for v in r))
    _write_csv(config.out, CSV_COLUMNS, rows)
    _write_csv(crossover_path(config.out), CROSSOVER_COLUMNS, cross)
    return rows
