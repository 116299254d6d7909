"""PyTorch autograd integration: the engine as a differentiable op.

`expectation(circuit, theta, x, weights)` returns the per-row observable
value_b = sum_q w_q <Z_q>_b (reference grad.py:207-218 with the weighted-Z adapter) as a
float64 CUDA tensor that participates in autograd:

* d value_b / d theta  -> per-row adjoint gradients (B, T), contracted with the upstream
  gradient on the device;
* d value_b / d x_b    -> per-row encoding gradients (B, E) (computed only when x requires
  grad: the adjoint then runs down to the encoding layer);
* d value_b / d w_q    -> <Z_q>_b, a by-product of the same forward.

The forward runs the fused forward + adjoint program once (the adjoint costs about 2x the
forward, so it is done eagerly only when some input requires grad; otherwise the same program
runs and its gradient outputs are ignored). `QuantumLayer` wraps it as an nn.Module with the
trainable angles as a Parameter, for training loops (per-block re-encoding circuits included).
"""

from __future__ import annotations

import numpy as np
import torch

from .circuits import Circuit


def _as_dev(t, device, dtype=torch.float64):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.asarray(t, dtype=np.float64))
    return t.to(device=device, dtype=dtype)


class _Expectation(torch.autograd.Function):
    @staticmethod
    def forward(ctx, theta, x, weights, circuit, plan, batch):
        from .core import _engine

        dev = theta.device if theta is not None and theta.is_cuda else (
            x.device if x is not None and x.is_cuda else torch.device("cuda"))
        eng = _engine(circuit, plan, dev)
        need_t = ctx.needs_input_grad[0]
        need_x = ctx.needs_input_grad[1]
        r = eng.fwd_bwd(theta.detach() if theta.numel() else None,
                        x.detach() if x is not None else None, batch=batch,
                        weights=weights.detach() if weights is not None else None,
                        rows=need_t, encoding_grads=need_x)
        ctx.save_for_backward(r["grads"] if need_t else None,
                              r["encoding_grads"] if need_x else None, r["zq"])
        return r["value"]

    @staticmethod
    def backward(ctx, gout):
        grows, erows, zq = ctx.saved_tensors
        gout = gout.to(torch.float64)
        g_theta = g_x = g_w = None
        if ctx.needs_input_grad[0] and grows is not None:
            g_theta = grows.t() @ gout
        if ctx.needs_input_grad[1] and erows is not None:
            g_x = erows * gout[:, None]
        if ctx.needs_input_grad[2]:
            g_w = zq.t() @ gout
        return g_theta, g_x, g_w, None, None, None


def expectation(circuit, theta=None, x=None, weights=None, batch=None, plan=None, device=None):
    """Differentiable sum_q w_q <Z_q> per row, shape (B,), float64 on the engine's device.

    theta: (T,) trainable angles; x: (B, E) encoding angles; weights: (n,) (default ones).
    Any of them may be tensors requiring grad. `batch` is needed only when E == 0."""
    dev = torch.device(device) if device is not None else None
    for t in (theta, x, weights):
        if dev is None and isinstance(t, torch.Tensor) and t.is_cuda:
            dev = t.device
    dev = dev or torch.device("cuda")
    th = _as_dev(theta, dev)
    xx = _as_dev(x, dev)
    w = _as_dev(weights, dev) if weights is not None else torch.ones(int(circuit.n), dtype=torch.float64, device=dev)
    if batch is None:
        if xx is None:
            raise ValueError("batch is required when the circuit has no encoding angles")
        batch = int(xx.shape[0])
    if th is None:
        th = torch.zeros(0, dtype=torch.float64, device=dev)
    return _Expectation.apply(th, xx, w, circuit, plan, int(batch))


class QuantumLayer(torch.nn.Module):
    """A circuit as a layer: forward(x) -> (B,) weighted <Z> per row; the trainable angles
    are `self.theta` (initialised like the reference bench, U[-pi, pi) seeded), the observable
    weights `self.weights` (trainable when `train_weights`)."""

    def __init__(self, circuit: Circuit, seed: int = 0, weights=None, train_weights: bool = False,
                 device=None, plan=None):
        super().__init__()
        self.circuit = circuit
        self.plan = plan
        rng = np.random.default_rng(seed)
        dev = torch.device(device) if device is not None else torch.device("cuda")
        T = int(circuit.trainable_count)
        self.theta = torch.nn.Parameter(
            torch.as_tensor(rng.uniform(-np.pi, np.pi, T), dtype=torch.float64, device=dev))
        w = np.ones(int(circuit.n)) if weights is None else np.asarray(weights, dtype=np.float64)
        wt = torch.as_tensor(w, dtype=torch.float64, device=dev)
        if train_weights:
            self.weights = torch.nn.Parameter(wt)
        else:
            self.register_buffer("weights", wt)

    def forward(self, x):
        return expectation(self.circuit, self.theta, x, self.weights, plan=self.plan)
