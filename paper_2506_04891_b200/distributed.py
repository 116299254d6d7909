"""Batch-sharded data parallelism: one process per GPU, contiguous row
shards, and ONE collective per step -- an all-reduce (sum) of the T-length shared-angle
gradient in fp64, on the device tensor the adjoint kernels wrote (no host round trip).
Per-row outputs (<Z_q>, values, per-row grads) stay sharded.

A step function can be injected (`step_fn`) so the host logic is testable on CPU with the
gloo backend and an oracle-backed step (tests/test_distributed.py).
"""

from __future__ import annotations

import numpy as np


def shard_rows(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) row range of `rank` (earlier ranks get the extra rows)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def check_shardable(batch: int, world: int) -> None:
    """Every rank needs at least one row. Raised identically on every rank BEFORE any compute
    or collective, so a too-small batch is an error everywhere instead of a hang on the ranks
    that did reach the all-reduce."""
    if batch < 1:
        raise ValueError(f"batch must be positive, got {batch}")
    if world > batch:
        raise ValueError(f"batch of {batch} rows cannot be sharded over {world} ranks (one row each at least)")


def allreduce_grad_sum(grad_sum, group=None):
    """In-place sum over ranks of the shared-angle gradient (torch tensor, fp64)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad_sum, op=dist.ReduceOp.SUM, group=group)
    return grad_sum


def data_parallel_gradient(circuit, trainable, encoding, weights=None, group=None, plan=None,
                           step_fn=None, device=None, batch=None):
    """Each rank evaluates its shard of `encoding` rows (the caller passes the FULL (B, E)
    matrix, every rank slices the same way), then the shared-angle gradient is summed over
    ranks. A circuit without encoding angles has identical rows: `batch` says how many (the
    reference's gradient(batch=...)); they are sharded the same way.

    Returns (rows (start, stop), result of the shard, grad_sum). With the CUDA engine (no
    `step_fn`) the result is the engine's dict of device tensors and grad_sum is the
    all-reduced fp64 device tensor; with `step_fn` (CPU tests) a GradResult and a numpy array.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    enc = None if encoding is None else np.asarray(encoding)
    if enc is not None:
        if batch is not None and batch != enc.shape[0]:
            raise ValueError(f"encoding rows {enc.shape[0]} != batch {batch}")
        batch = enc.shape[0]
    elif batch is None:
        batch = 1
    check_shardable(batch, world)
    start, stop = shard_rows(batch, world, rank)
    shard = None if enc is None else enc[start:stop]
    if step_fn is not None:
        res = step_fn(circuit, trainable, shard, stop - start, weights)
        gs = torch.as_tensor(np.asarray(res.grad_sum, dtype=np.float64).copy())
        allreduce_grad_sum(gs, group)
        return (start, stop), res, gs.numpy()
    from .core import _engine

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    eng = _engine(circuit, plan, dev)
    w = np.ones(circuit.n) if weights is None else weights
    res = eng.fwd_bwd(trainable, shard, batch=stop - start, weights=w)
    gs = res["grad_sum"]
    allreduce_grad_sum(gs, group)  # device tensor, NCCL over NVLink
    return (start, stop), res, gs
