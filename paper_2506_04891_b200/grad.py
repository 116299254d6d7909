"""Adjoint gradients (drop-in for reference grad.py:25-218).

`gradient` / `backward_sweep` keep the reference signatures and return a `GradResult`
with the same three fields; the observable defaults to sum_k Z_k and `weights=` selects
sum_q w_q Z_q. Extra fields: per-qubit <Z_q> (`zq`) and the batch-summed shared-angle
gradient (`grad_sum`, what an optimizer step consumes). The backward pass runs on the
device: one coupling matrix per fused gate group, fp64 contraction (see schedule.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .circuits import check_parameters
from .core import _engine
from .states import StateBatch


@dataclass(frozen=True)
class GradResult:
    """value (batch,), grads (batch, trainable_count), encoding_grads (batch, encoding_count)
    -- the reference's GradResult (grad.py:25-37) -- plus zq (batch, n) and grad_sum (T,)."""

    value: np.ndarray
    grads: np.ndarray
    encoding_grads: np.ndarray
    zq: np.ndarray = field(default=None, repr=False)
    grad_sum: np.ndarray = field(default=None, repr=False)


def _np(t, shape):
    if t is None:
        return np.zeros(shape)
    return t.detach().cpu().numpy().reshape(shape)


def gradient(circuit, trainable=None, encoding=None, batch: int = 1, plan=None, weights=None,
             device=None):
    """Expectation values and adjoint gradients from |0...0> (reference grad.py:207-218)."""
    trainable, encoding = check_parameters(circuit, trainable, encoding, None)
    if encoding is not None:
        batch = encoding.shape[0] if batch in (None, 1) and encoding.shape[0] != batch else batch
        if encoding.shape[0] != batch:
            raise ValueError(f"encoding rows {encoding.shape[0]} != batch {batch}")
    if batch < 1:
        raise ValueError(f"batch must be positive, got {batch}")
    eng = _engine(circuit, plan, device)
    # one captured CUDA graph per (batch, weighted) and engine: inputs copied in, graph replayed
    key = ("grad_step", batch, weights is None)
    steps = eng.__dict__.setdefault("_steps", {})
    step = steps.get(key)
    if step is None:
        steps.clear()  # keep one step's static buffers alive per engine
        step = steps[key] = eng.make_step(batch)
    T, E = eng.T, eng.E
    host = not any(type(a).__module__.startswith("torch") for a in (trainable, encoding, weights))
    if host:
        # host arrays in and out: one pinned copy each way around the graph replay
        r = step.run_host(trainable, encoding, np.ones(circuit.n) if weights is None else weights)
        z = lambda k, sh: r[k] if k in r else np.zeros(sh)  # noqa: E731
        return GradResult(value=z("value", (batch,)), grads=z("grads", (batch, T)),
                          encoding_grads=z("encoding_grads", (batch, E)), zq=z("zq", (batch, circuit.n)),
                          grad_sum=z("grad_sum", (T,)))
    r = step.run(trainable, encoding, np.ones(circuit.n) if weights is None else weights)
    return GradResult(
        value=_np(r["value"], (batch,)),
        grads=_np(r["grads"], (batch, T)),
        encoding_grads=_np(r["encoding_grads"], (batch, E)),
        zq=_np(r["zq"], (batch, circuit.n)),
        grad_sum=_np(r["grad_sum"], (T,)),
    )


def backward_sweep(circuit, trainable=None, encoding=None, final_state: StateBatch | None = None,
                   plan=None, weights=None):
    """Reverse sweep from a finished forward state (reference grad.py:169-204)."""
    if final_state is None:
        raise ValueError("backward_sweep needs the forward-pass final state")
    trainable, encoding = check_parameters(circuit, trainable, encoding, final_state.batch)
    eng = _engine(circuit, plan, final_state.amplitudes.device, prefix=False)
    r = eng.backward_from_state(trainable, encoding, final_state.amplitudes, weights=weights)
    b = final_state.batch
    return GradResult(
        value=_np(r["value"], (b,)),
        grads=_np(r["grads"], (b, eng.T)),
        encoding_grads=_np(r["encoding_grads"], (b, eng.E)),
        zq=_np(r["zq"], (b, circuit.n)),
        grad_sum=_np(r["grad_sum"], (eng.T,)),
    )
