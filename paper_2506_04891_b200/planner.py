"""Per-layer method choice over CUDA variants (drop-in for reference planner.py:1-309).

The reference times its nine CPU techniques per layer signature and replays the argmin
(`build_plan`, planner.py:165-220). Here the candidates are CUDA execution variants of the
same fused engine:

* per layer: FUSED (the layer's gates join the surrounding tile passes) or ISOLATED (the
  layer gets pass boundaries of its own -- the GPU analogue of one-layer-at-a-time);
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


KERNEL_ORDER = tuple(KernelKind)
_RANK = {k: i for i, k in enumerate(KERNEL_ORDER)}


def kernel_rank(kind: KernelKind) -> int:
    return _RANK[kind]


def applicable_variants(layer, n: int) -> tuple:
    positions(layer, n)  # validates the pattern
    return KERNEL_ORDER


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


def tiling_of(plan, circuit):
    """(M, R) the engine should compile with for this plan (None = defaults)."""
    if plan is None:
        return None, None
    return getattr(plan, "tile_bits", None), None


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
    return Plan(
        str(_req(doc, "machine_id", "document")), int(_req(doc, "n", "document")),
        int(_req(doc, "batch", "document")), Objective(_req(doc, "objective", "document")),
        tuple(k for _, k in pairs), tuple(meas), None if tb is None else int(tb),
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
