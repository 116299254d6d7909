"""Batch-sharded data parallelism: one process per GPU, contiguous row
shards, and ONE collective per step -- an all-reduce (sum) of the T-length shared-angle
gradient in fp64. Per-row outputs (<Z_q>, values, per-row grads) stay sharded.

The engine is injected (`step_fn`) so the host logic is testable on CPU with the gloo
backend and an oracle-backed step (tests/test_distributed.py).
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


def allreduce_grad_sum(grad_sum, group=None):
    """In-place sum over ranks of the shared-angle gradient (torch tensor, fp64)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad_sum, op=dist.ReduceOp.SUM, group=group)
    return grad_sum


def data_parallel_gradient(circuit, trainable, encoding, weights=None, group=None, plan=None,
                           step_fn=None, device=None):
    """Each rank evaluates its shard of `encoding` rows (the caller passes the FULL
    (B, E) matrix, every rank slices the same way), then the shared-angle gradient is
    summed over ranks. Returns (rows (start, stop), GradResult of the shard, grad_sum)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    enc = None if encoding is None else np.asarray(encoding)
    batch = enc.shape[0] if enc is not None else 1
    start, stop = shard_rows(batch, world, rank)
    shard = None if enc is None else enc[start:stop]
    if step_fn is None:
        from .grad import gradient

        res = gradient(circuit, trainable, shard, batch=stop - start, plan=plan, weights=weights,
                       device=device)
    else:
        res = step_fn(circuit, trainable, shard, stop - start, weights)
    gs = torch.as_tensor(np.asarray(res.grad_sum, dtype=np.float64).copy())
    if dist.is_initialized() and dist.get_backend(group) == "nccl":
        gs = gs.cuda()
    allreduce_grad_sum(gs, group)
    return (start, stop), res, gs.cpu().numpy()
