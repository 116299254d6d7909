"""Command line over the CUDA engine (reference `cli.py:45-180`).

    python -m paper_2506_04891_b200 run  --circuit C.json [--params P.json] [--plan PLAN.json]
    python -m paper_2506_04891_b200 grad --circuit C.json [--params P.json] [--plan PLAN.json]
    python -m paper_2506_04891_b200 plan --circuit C.json --batch B --out PLAN.json [--objective ...]

File formats are the reference's: circuit JSON {"n", "layers": [{"gate", "pattern", "wires",
"role", "values"}]} (`bench.py:281-319`), params JSON {"trainable", "encoding"}
(`bench.py:322-336`), plan JSON (`planner.py:223-309`, plus `tile_bits`). `run` prints one
<sum Z> per row like the reference; `grad` (an addition) prints value and gradients as JSON.
Exit codes as the reference: 0 ok, 1 correctness failure, 2 invalid arguments or unreadable
inputs, 3 capacity overflow. The reference's benchmark families and CSV harness are out of
scope."""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from .circuits import Circuit, Layer, Role, all_qubits, chain_pairs, explicit, ring_pairs
from .errors import CapacityError, CorrectnessError, PlanMismatchError
from .gates import GateKind

_PATTERNS = {
    "all": lambda item: all_qubits(),
    "ring": lambda item: ring_pairs(),
    "chain": lambda item: chain_pairs(),
    "explicit": lambda item: explicit(*[tuple(w) for w in item.get("wires", [])]),
}


def parse_circuit(text: str) -> Circuit:
    """Circuit from the reference's JSON file form (bench.py:291-314)."""
    doc = json.loads(text)
    if not isinstance(doc, dict) or "n" not in doc or "layers" not in doc:
        raise ValueError("circuit file needs top-level fields 'n' and 'layers'")
    layers = []
    for i, item in enumerate(doc["layers"]):
        try:
            gate = GateKind(item["gate"])
            builder = _PATTERNS[item["pattern"]]
        except (KeyError, ValueError) as exc:
            raise ValueError(f"layer {i}: {exc}") from exc
        role = Role(item["role"]) if "role" in item else None
        try:
            layers.append(Layer(gate, builder(item), role=role, values=item.get("values")))
        except ValueError as exc:
            raise ValueError(f"layer {i}: {exc}") from exc
    return Circuit(int(doc["n"]), layers)


def load_circuit(path) -> Circuit:
    with open(path) as f:
        return parse_circuit(f.read())


def load_params(path):
    """{"trainable": [...], "encoding": [[...]]} (bench.py:322-336)."""
    with open(path) as f:
        doc = json.load(f)
    if not isinstance(doc, dict):
        raise ValueError("params file must be a JSON object")
    tr, en = doc.get("trainable"), doc.get("encoding")
    tr = None if tr is None else np.asarray(tr, dtype=np.float64)
    if en is not None:
        en = np.asarray(en, dtype=np.float64)
        if en.ndim != 2:
            raise ValueError("encoding must be a matrix (batch x inputs)")
    return tr, en


def _parse_qubits(text: str) -> tuple:
    """'5' -> (5,); '4..7' -> (4, 5, 6, 7); '4,6,8' -> (4, 6, 8) (reference cli.py:30-38)."""
    if ".." in text:
        lo, hi = (int(v) for v in text.split("..", 1))
        if hi < lo:
            raise ValueError(f"empty qubit range {text!r}")
        return tuple(range(lo, hi + 1))
    return tuple(int(part) for part in text.split(","))


def _build_parser():
    p = argparse.ArgumentParser(prog="paper_2506_04891_b200",
                                description="B200 layer-wise state-vector engine")
    sub = p.add_subparsers(dest="command", required=True)
    for name, hlp in (("run", "evaluate a circuit file, print <sum Z> per row"),
                      ("grad", "forward + adjoint gradients of a circuit file (JSON out)")):
        s = sub.add_parser(name, help=hlp)
        s.add_argument("--circuit", required=True)
        s.add_argument("--params", default=None)
        s.add_argument("--plan", default=None)
    s = sub.add_parser("plan", help="time the CUDA variants of one circuit and save the plan")
    s.add_argument("--circuit", required=True)
    s.add_argument("--batch", required=True, type=int)
    s.add_argument("--objective", choices=["forward", "forward+backward"], default="forward+backward")
    s.add_argument("--reps", type=int, default=10)
    s.add_argument("--warmup", type=int, default=3)
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--out", required=True)
    s = sub.add_parser("bench", help="timing sweep over a circuit family on the GPU, CSV reports")
    s.add_argument("--family", required=True, choices=("vq", "qdi", "ibm", "ionq"))
    s.add_argument("--qubits", required=True, type=_parse_qubits, metavar="A..B|N[,M...]")
    s.add_argument("--batch", default=(1,), type=lambda t: tuple(int(x) for x in t.split(",")),
                   metavar="B[,B2...]")
    s.add_argument("--blocks", type=int, default=8)
    s.add_argument("--reps", type=int, default=10)
    s.add_argument("--warmup", type=int, default=3)
    s.add_argument("--objective", choices=["forward", "forward+backward"], default="forward")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--out", required=True)
    s.add_argument("--plan", default=None, help="replay a saved plan file")
    s = sub.add_parser("compile", help="compile a circuit into a program artifact for lsq_program_load")
    g = s.add_mutually_exclusive_group(required=True)
    g.add_argument("--circuit", help="reference circuit JSON file")
    g.add_argument("--config", type=int, choices=[1, 2, 3, 4, 5], help="a BASELINE config circuit")
    s.add_argument("--plan", default=None, help="plan JSON (tile exponent, per-layer variants)")
    s.add_argument("--gradient", action="store_true",
                   help="gradient program (synthesized |0..0> prefix, folded observable)")
    s.add_argument("--out", required=True)
    return p


def _inputs(args):
    circuit = load_circuit(args.circuit)
    tr, en = load_params(args.params) if args.params is not None else (None, None)
    from .planner import load_plan

    plan = load_plan(args.plan) if args.plan is not None else None
    batch = en.shape[0] if en is not None else 1
    return circuit, tr, en, plan, batch


def _cmd_run(args) -> int:
    from .core import apply_circuit
    from .states import expectation_z_sum, zero_state

    circuit, tr, en, plan, batch = _inputs(args)
    out = apply_circuit(circuit, tr, en, zero_state(circuit.n, batch), plan)
    for value in np.asarray(expectation_z_sum(out)).reshape(-1):
        print(value)
    return 0


def _cmd_grad(args) -> int:
    from .grad import gradient

    circuit, tr, en, plan, batch = _inputs(args)
    r = gradient(circuit, tr, en, batch=batch, plan=plan)
    print(json.dumps({"value": r.value.tolist(), "grads": r.grads.tolist(),
                      "encoding_grads": r.encoding_grads.tolist(), "grad_sum": r.grad_sum.tolist()}))
    return 0


def _cmd_plan(args) -> int:
    from .planner import Objective, build_plan, save_plan

    circuit = load_circuit(args.circuit)
    plan = build_plan(circuit, args.batch, objective=Objective(args.objective), reps=args.reps,
                      warmup=args.warmup, seed=args.seed)
    save_plan(plan, args.out)
    print(f"wrote plan for n={circuit.n} batch={args.batch} to {args.out}")
    return 0


def _cmd_bench(args) -> int:
    from .harness import BenchConfig, crossover_path, run_benchmark
    from .planner import Objective

    config = BenchConfig(family=args.family, qubits=tuple(args.qubits), batches=tuple(args.batch),
                         blocks=args.blocks, reps=args.reps, warmup=args.warmup,
                         objective=Objective(args.objective), seed=args.seed, out=args.out, plan_path=args.plan)
    rows = run_benchmark(config)
    print(f"wrote {len(rows)} rows to {args.out}")
    print(f"wrote kernel choices to {crossover_path(args.out)}")
    return 0


def _cmd_compile(args) -> int:
    """Host-only (no GPU): circuit -> schedule -> generated kernels -> one artifact file."""
    from . import artifact
    from .planner import KernelKind, load_plan, tiling_of
    from .schedule import DEFAULT_M, DEFAULT_R_SPECIALISED, compile_circuit, default_r

    if args.circuit is not None:
        circuit = load_circuit(args.circuit)
    else:
        from .configs import build_config_circuit

        circuit = build_config_circuit(args.config)
    plan = load_plan(args.plan) if args.plan is not None else None
    M, R = tiling_of(plan, circuit)
    if R is None:
        m = min(circuit.n, M if M is not None else DEFAULT_M)
        R = DEFAULT_R_SPECIALISED if m >= 9 else default_r(m)
    sel = lambda kk: [] if plan is None else [i for i, k in enumerate(plan.assignments) if k is kk]  # noqa: E731
    from .engine import forward_program

    kw = dict(isolate=sel(KernelKind.ISOLATED), prefix=args.gradient, fold=args.gradient, split=True,
              direct=sel(KernelKind.DIRECT), split_layers=sel(KernelKind.SPLIT))
    prog = compile_circuit(circuit, M=M, R=R, **kw)
    size = artifact.write(prog, args.out, forward_program(circuit, prog, M=M, **kw))
    print(f"wrote {args.out}: n={circuit.n}, {len(prog.passes)} passes, {size} bytes")
    return 0


_COMMANDS = {"run": _cmd_run, "grad": _cmd_grad, "plan": _cmd_plan, "compile": _cmd_compile,
             "bench": _cmd_bench}


def main(argv=None) -> int:
    args = _build_parser().parse_args(argv)
    try:
        return _COMMANDS[args.command](args)
    except CorrectnessError as exc:
        print(f"correctness failure: {exc}", file=sys.stderr)
        return 1
    except CapacityError as exc:
        print(f"capacity exceeded: {exc}", file=sys.stderr)
        return 3
    except (ValueError, PlanMismatchError, json.JSONDecodeError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
