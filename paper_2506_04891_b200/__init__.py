"""B200-native (sm_100a) engine for the TQml layer-wise state-vector simulator
(arXiv 2506.04891), behind the reference `layersim` API.

Drop-in surface (reference pkg/src/layersim/__init__.py:10-47, hot path only):
circuits IR (Circuit, Layer, GateKind, WirePattern, Role, patterns), states
(StateBatch, zero_state, random_state, z_weights, expectation_z_sum, expectation_z),
execution (apply_circuit, gradient, backward_sweep, GradResult), planning (build_plan,
Plan, Objective, save/load). The compute path is the CUDA library in `_lib/liblsq.so`;
there is no CPU fallback.
"""

from .circuits import (
    Circuit,
    Layer,
    PatternKind,
    Role,
    WirePattern,
    all_qubits,
    chain_pairs,
    check_parameters,
    explicit,
    positions,
    ring_pairs,
)
from .errors import CapacityError, CorrectnessError, PlanMismatchError
from .gates import GATE_TRAITS, GateKind, TraitFlags, gate_matrix, gate_matrix_derivative


def __getattr__(name):
    # device-dependent modules are imported lazily so that the IR/compiler import on CPU
    lazy = {
        "apply_circuit": ("core", "apply_circuit"),
        "plan_kernels": ("core", "plan_kernels"),
        "gradient": ("grad", "gradient"),
        "backward_sweep": ("grad", "backward_sweep"),
        "GradResult": ("grad", "GradResult"),
        "StateBatch": ("states", "StateBatch"),
        "zero_state": ("states", "zero_state"),
        "random_state": ("states", "random_state"),
        "z_weights": ("states", "z_weights"),
        "expectation_z_sum": ("states", "expectation_z_sum"),
        "expectation_z": ("states", "expectation_z"),
        "Engine": ("engine", "Engine"),
        "engine_for": ("engine", "engine_for"),
        "Objective": ("planner", "Objective"),
        "Plan": ("planner", "Plan"),
        "KernelKind": ("planner", "KernelKind"),
        "build_plan": ("planner", "build_plan"),
        "save_plan": ("planner", "save_plan"),
        "load_plan": ("planner", "load_plan"),
        "plan_roundtrip": ("planner", "plan_roundtrip"),
        "choose_tile_bits": ("planner", "choose_tile_bits"),
        "plan_for_tile_bits": ("planner", "plan_for_tile_bits"),
        "expectation": ("autograd", "expectation"),
        "QuantumLayer": ("autograd", "QuantumLayer"),
    }
    if name in lazy:
        import importlib

        mod, attr = lazy[name]
        return getattr(importlib.import_module(f".{mod}", __name__), attr)
    raise AttributeError(name)


__version__ = "0.1.0"
