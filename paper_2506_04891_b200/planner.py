"""Per-layer method choice over CUDA variants (drop-in for reference planner.py:1-309).

The reference times its nine CPU techniques per layer signature and replays the argmin
(`build_plan`, planner.py:165-220). Here the candidates are CUDA implementations of the same
fused engine, chosen per layer signature by measurement:

* FUSED    -- the default: the layer's gates join the surrounding fused groups and tile passes,
              one-qubit groups in the Euler tangent form (6 packed ops per pair) where it
              applies, diagonal parts split off by the codegen cost model;
* ISOLATED -- the layer gets pass boundaries of its own (the GPU analogue of one layer at a
              time): fewer fused gates per pass, lighter kernels;
* DIRECT   -- (one-qubit non-diagonal gates) groups containing the layer's gates use the
              direct complex 2x2 form (8 packed ops per pair, no run-time scale, no tangent
              rotation);
* SPLIT    -- (one-qubit diagonal gates) groups containing the layer's gates are split into a
              diagonal run (phase table / sincos over many wires at once) and the non-diagonal
              remainder, whatever the cost model says;
* per circuit: the tile exponent M (bits per tile pass), part of the plan.

Timing follows the reference protocol (warmup untimed, `reps` timed, mean and population
std, argmin with enum-order tie-break, injectable `timer` / `measure` for tests) but uses
CUDA events on the launching stream. Plans keep the reference JSON shape plus "tile_bits".
"""

from __future__ import annotations

import json
import warnings
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .circuits import positions
from .gates import GateKind, gate_traits


class Objective(Enum):
    FORWARD = "forward"
    FORWARD_BACKWARD = "forward+backward"


class KernelKind(Enum):
    """CUDA variants; declaration order is the tie-break order."""

    FUSED = "fused"
    ISOLATED = "isolated"
    DIRECT = "direct"
    SPLIT = "split"


KERNEL_ORDER = tuple(KernelKind)
_RANK = {k: i for i, k in enumerate(KERNEL_ORDER)}


def kernel_rank(kind: KernelKind) -> int:
    return _RANK[kind]


def applicable_variants(layer, n: int) -> tuple:
    positions(layer, n)  # validates the pattern
    tr = gate_traits(layer.gate)
    out = [KernelKind.FUSED, KernelKind.ISOLATED]
    if tr.arity == 1 and not tr.diagonal and not tr.permutation:
        out.append(KernelKind.DIRECT)
    if tr.arity == 1 and tr.diagonal:
        out.append(KernelKind.SPLIT)
    return tuple(out)


def default_variant(layer, n: int) -> KernelKind:
    return KernelKind.FUSED


@dataclass(frozen=True)
class TimingStats:
    mean_seconds: float
    std_seconds: float
    reps: int
    warmup: int

    def __post_init__(self):
        if self.reps < 1:
            raise ValueError("reps must be at least 1")
        if self.mean_seconds < 0 or self.std_seconds < 0:
            raise ValueError("timing statistics cannot be negative")


@dataclass(frozen=True)
class PlanMeasurement:
    layer_index: int
    kernel: KernelKind
    mean_s: float
    std_s: float
    reps: int


@dataclass(frozen=True)
class Plan:
    machine_id: str
    n: int
    batch: int
    objective: Objective
    assignments: tuple
    measurements: tuple
    tile_bits: int | None = None
    rebalance_budget: float | None = None  # pass-rebalancing budget measured best (None: default)


def tiling_of(plan, circuit):
    """(M, R) the engine should compile with for this plan (None = defaults)."""
    if plan is None:
        return None, None
    return getattr(plan, "tile_bits", None), None


def layer_signature(layer, n: int) -> tuple:
    """Layers sharing a signature share one measurement set. Unlike the reference
    (planner.py:185) the explicit wires are part of it."""
    role = None if layer.role is None else layer.role.value
    return (layer.gate.value, layer.pattern.kind.value, tuple(map(tuple, layer.pattern.wires)), n, role)


TILE_BITS_CANDIDATES = (10, 11, 12, 13)
# pass-rebalancing budgets (estimated packed FP32 ops per amplitude a pass may reach by taking
# groups from the pass before it, schedule.rebalance_passes) tried by build_plan
REBALANCE_CANDIDATES = (40.0, 120.0, 220.0)


def _draw(circuit, batch, seed):
    rng = np.random.default_rng(seed)
    th = rng.uniform(-np.pi, np.pi, circuit.trainable_count) if circuit.trainable_count else None
    x = rng.uniform(-np.pi, np.pi, (batch, circuit.encoding_count)) if circuit.encoding_count else None
    return th, x


def time_program(circuit, batch: int, objective: "Objective" = None, M=None, isolate=(), reps: int = 10,
                 warmup: int = 3, timer=None, seed: int = 0, device=None, direct=(),
                 split_layers=(), rebalance_budget=None) -> TimingStats:
    """Time the whole compiled program (one CUDA variant) with the reference's protocol:
    `warmup` untimed runs then `reps` timed runs (reference planner.py:106-162). Default clock:
    CUDA events on the engine's stream; an injected `timer` is called around each rep after
    a device synchronisation."""
    import torch

    from .engine import Engine

    objective = objective or Objective.FORWARD
    if reps < 1:
        raise ValueError("reps must be at least 1")
    if warmup < 0:
        raise ValueError("warmup cannot be negative")
    eng = Engine(circuit, M=M, isolate=isolate, device=device, direct=direct, split_layers=split_layers,
                 fold=False if objective is Objective.FORWARD else None, rebalance_budget=rebalance_budget)
    th, x = _draw(circuit, batch, seed)
    th_d = None if th is None else torch.as_tensor(th, device=eng.device)
    x_d = None if x is None else torch.as_tensor(x, device=eng.device)

    def run():
        if objective is Objective.FORWARD:
            eng.forward(th_d, x_d, batch=batch)
        else:
            eng.fwd_bwd(th_d, x_d, batch=batch, rows=False, encoding_grads=False)

    for _ in range(warmup):
        run()
    samples = np.empty(reps)
    stream = torch.cuda.current_stream(eng.device)
    for r in range(reps):
        if timer is None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            e1.synchronize()
            samples[r] = e0.elapsed_time(e1) / 1e3
        else:
            torch.cuda.synchronize(eng.device)
            t0 = timer()
            run()
            torch.cuda.synchronize(eng.device)
            samples[r] = timer() - t0
    return TimingStats(float(samples.mean()), float(samples.std()), reps, warmup)


def build_plan(circuit, batch: int, objective: "Objective" = None, timer=None, reps: int = 10,
               warmup: int = 3, seed: int = 0, measure=None, tile_bits=None) -> "Plan":
    """Per-layer CUDA variant choice by measurement (reference build_plan, planner.py:165-220).

    1. tile exponent M: every candidate (<= n) is timed on the whole program; argmin.
    2. per layer signature, in order of first appearance: every applicable variant (ISOLATED,
       DIRECT, SPLIT) is timed on the whole program with the variants kept so far; the fastest
       is kept for all layers of the signature (ties -> declaration order, FUSED first).
    3. the pass-rebalancing budget: every candidate of REBALANCE_CANDIDATES is timed on the
       whole program with the kept variants; argmin (real timing only: an injected `measure`
       leaves the default budget).

    `measure(layer, kernel) -> TimingStats` replaces real timing (tests): it is asked for the
    per-layer variants, and `measure(None, M)` for tile exponents.
    """
    objective = objective or Objective.FORWARD
    n = int(circuit.n)
    layers = list(circuit.layers)

    def timed(M, assign, budget=None):
        sel = lambda kk: sorted(i for i, k in assign.items() if k is kk)  # noqa: E731
        return time_program(circuit, batch, objective, M=M, isolate=sel(KernelKind.ISOLATED), reps=reps,
                            warmup=warmup, timer=timer, seed=seed, direct=sel(KernelKind.DIRECT),
                            split_layers=sel(KernelKind.SPLIT), rebalance_budget=budget)

    if tile_bits is None:
        cands = sorted({min(n, m) for m in TILE_BITS_CANDIDATES})
        stats_m = {m: (measure(None, m) if measure is not None else timed(m, {})) for m in cands}
        tile_bits = min(cands, key=lambda m: (stats_m[m].mean_seconds, -m))
        base = stats_m[tile_bits]
    else:
        base = measure(None, tile_bits) if measure is not None else timed(tile_bits, {})
    chosen: dict = {}  # layer index -> non-default variant kept so far
    cache: dict = {}
    measurements = []
    assignments = [KernelKind.FUSED] * len(layers)
    for idx, layer in enumerate(layers):
        sig = layer_signature(layer, n)
        if sig not in cache:
            members = [i for i, l in enumerate(layers) if layer_signature(l, n) == sig]
            stats = {}
            for k in applicable_variants(layer, n):
                if measure is not None:
                    stats[k] = measure(layer, k)
                elif k is KernelKind.FUSED:
                    stats[k] = base
                else:
                    stats[k] = timed(tile_bits, {**chosen, **{i: k for i in members}})
            best = min(stats, key=lambda k: (stats[k].mean_seconds, kernel_rank(k)))
            if best is not KernelKind.FUSED:
                chosen.update({i: best for i in members})
                if measure is None:
                    base = stats[best]
            cache[sig] = (best, stats)
        best, stats = cache[sig]
        assignments[idx] = best
        for k, st in stats.items():
            measurements.append(PlanMeasurement(idx, k, st.mean_seconds, st.std_seconds, st.reps))
    budget = None
    if measure is None and objective is Objective.FORWARD_BACKWARD:
        from .schedule import REBALANCE_BUDGET

        stats_b = {b: (base if b == REBALANCE_BUDGET else timed(tile_bits, chosen, b)) for b in REBALANCE_CANDIDATES}
        budget = min(stats_b, key=lambda b: (stats_b[b].mean_seconds, b))
    return Plan(machine_id(), n, batch, objective, tuple(assignments), tuple(measurements), tile_bits, budget)


def choose_tile_bits(circuit, batch: int, objective: "Objective" = None, candidates=TILE_BITS_CANDIDATES,
                     reps: int = 3, warmup: int = 2, device=None, timer=None):
    """Tile exponent M by measurement only (step 1 of build_plan without the per-layer
    variants): every candidate <= n is timed on the whole program. Returns (M, {M: stats})."""
    objective = objective or Objective.FORWARD_BACKWARD
    n = int(circuit.n)
    cands = sorted({min(n, m) for m in candidates})
    stats = {m: time_program(circuit, batch, objective, M=m, reps=reps, warmup=warmup, timer=timer,
                             device=device) for m in cands}
    best = min(cands, key=lambda m: (stats[m].mean_seconds, -m))
    return best, stats


def plan_for_tile_bits(circuit, batch: int, tile_bits: int, objective: "Objective" = None,
                       stats: dict | None = None) -> "Plan":
    """All-FUSED plan with the given tile exponent (the measured candidates recorded as
    layer_index -1 measurements are not part of the reference format, so they are dropped)."""
    objective = objective or Objective.FORWARD_BACKWARD
    n = int(circuit.n)
    return Plan(machine_id(), n, batch, objective, tuple(KernelKind.FUSED for _ in circuit.layers), (),
                int(tile_bits))


def machine_id() -> str:
    try:
        import ctypes

        from . import _native

        buf = ctypes.create_string_buffer(256)
        if _native.lib().lsq_device_info(0, buf, 256) == 0:
            return buf.value.decode()
    except Exception:
        pass
    return "unknown-device"


def serialize_plan(plan: Plan) -> str:
    doc = {
        "machine_id": plan.machine_id,
        "n": plan.n,
        "batch": plan.batch,
        "objective": plan.objective.value,
        "tile_bits": plan.tile_bits,
        "rebalance_budget": plan.rebalance_budget,
        "assignments": [{"layer_index": i, "kernel": k.value} for i, k in enumerate(plan.assignments)],
        "measurements": [
            {"layer_index": m.layer_index, "kernel": m.kernel.value, "mean_s": m.mean_s,
             "std_s": m.std_s, "reps": m.reps}
            for m in plan.measurements
        ],
    }
    return json.dumps(doc, indent=2) + "\n"


def _req(obj, key, where):
    if not isinstance(obj, dict):
        raise ValueError(f"plan {where} must be an object")
    if key not in obj:
        raise ValueError(f"plan {where} is missing field {key!r}")
    return obj[key]


def parse_plan(text: str) -> Plan:
    doc = json.loads(text)
    pairs = []
    for i, it in enumerate(_req(doc, "assignments", "document")):
        w = f"assignments[{i}]"
        pairs.append((int(_req(it, "layer_index", w)), KernelKind(_req(it, "kernel", w))))
    pairs.sort(key=lambda p: p[0])
    if [p[0] for p in pairs] != list(range(len(pairs))):
        raise ValueError("assignments must cover layer indices 0..L-1 exactly once")
    meas = []
    for i, it in enumerate(_req(doc, "measurements", "document")):
        w = f"measurements[{i}]"
        meas.append(
            PlanMeasurement(int(_req(it, "layer_index", w)), KernelKind(_req(it, "kernel", w)),
                            float(_req(it, "mean_s", w)), float(_req(it, "std_s", w)), int(_req(it, "reps", w)))
        )
    tb = doc.get("tile_bits")
    rb = doc.get("rebalance_budget")
    return Plan(
        str(_req(doc, "machine_id", "document")), int(_req(doc, "n", "document")),
        int(_req(doc, "batch", "document")), Objective(_req(doc, "objective", "document")),
        tuple(k for _, k in pairs), tuple(meas), None if tb is None else int(tb),
        None if rb is None else float(rb),
    )


def plan_roundtrip(plan: Plan) -> Plan:
    return parse_plan(serialize_plan(plan))


def save_plan(plan: Plan, path) -> None:
    with open(path, "w") as f:
        f.write(serialize_plan(plan))


def load_plan(path) -> Plan:
    with open(path) as f:
        plan = parse_plan(f.read())
    here = machine_id()
    if plan.machine_id != here:
        warnings.warn(f"plan was built on {plan.machine_id!r}, this host is {here!r}; timings may not transfer",
                      stacklevel=2)
    return plan
