"""Multi-rank host logic on CPU: world_size 2 over gloo, each rank runs its row shard
through an oracle-backed step and the shared-angle gradient is all-reduced; the result must
equal the single-process full-batch gradient."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2506_04891_b200.distributed import shard_rows


def test_shard_rows_cover_batch():
    for batch in (1, 5, 64, 1024, 1023):
        for world in (1, 2, 3, 4, 8):
            if world > batch:
                continue
            spans = [shard_rows(batch, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_step(circuit, trainable, shard, rows, weights):
    from oracle import layersim_oracle as orc
    from paper_2506_04891_b200.grad import GradResult

    r = orc.gradient(circuit, trainable, shard, batch=rows, weights=weights)
    return GradResult(r["value"], r["grads"], r["encoding_grads"], r["zq"], r["grads"].sum(0))


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_04891_b200.configs import make_workload
    from paper_2506_04891_b200.distributed import data_parallel_gradient

    wl = make_workload(5, n=6, batch=5)
    (s, e), res, gs = data_parallel_gradient(wl.circuit, wl.theta, wl.x, wl.weights, step_fn=_oracle_step)
    out[rank] = (s, e, gs, res.grads)
    dist.destroy_process_group()


def test_gloo_world2_allreduce_matches_single_process():
    from oracle import layersim_oracle as orc
    from paper_2506_04891_b200.configs import make_workload

    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, start_method="fork")
    wl = make_workload(5, n=6, batch=5)
    ref = orc.gradient(wl.circuit, wl.theta, wl.x, batch=5, weights=wl.weights)
    for r in range(world):
        s, e, gs, grads = out[r]
        np.testing.assert_allclose(gs, ref["grads"].sum(0), atol=1e-12)
        np.testing.assert_allclose(grads, ref["grads"][s:e], atol=1e-12)
    assert out[0][:2] == (0, 3) and out[1][:2] == (3, 5)


def _worker_small(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_04891_b200.configs import make_workload
    from paper_2506_04891_b200.distributed import data_parallel_gradient

    wl = make_workload(5, n=5, batch=1)
    try:
        data_parallel_gradient(wl.circuit, wl.theta, wl.x, wl.weights, step_fn=_oracle_step)
        out[rank] = "no error"
    except ValueError as e:
        out[rank] = f"ValueError: {e}"
    # an encoding-free circuit: `batch` identical rows sharded like encoded ones
    from paper_2506_04891_b200.circuits import Circuit, Layer, Role, all_qubits
    from paper_2506_04891_b200.gates import GateKind

    c = Circuit(3, [Layer(GateKind.RY, all_qubits(), Role.TRAINABLE)])
    (s, e), res, gs = data_parallel_gradient(c, np.array([0.3, 0.5, 0.7]), None, None, step_fn=_oracle_step,
                                             batch=4)
    out[f"{rank}_free"] = (s, e, gs)
    dist.destroy_process_group()


def test_gloo_world2_small_batch_errors_everywhere_no_hang():
    """world > batch raises the same ValueError on EVERY rank before any collective (no rank
    is left blocked in the all-reduce); an encoding-free circuit shards its `batch` rows."""
    from oracle import layersim_oracle as orc
    from paper_2506_04891_b200.circuits import Circuit, Layer, Role, all_qubits
    from paper_2506_04891_b200.gates import GateKind

    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker_small, args=(world, port, out), nprocs=world, start_method="fork")
    for r in range(world):
        assert out[r].startswith("ValueError") and "cannot be sharded" in out[r]
    c = Circuit(3, [Layer(GateKind.RY, all_qubits(), Role.TRAINABLE)])
    ref = orc.gradient(c, np.array([0.3, 0.5, 0.7]), None, batch=4)
    assert out["0_free"][:2] == (0, 2) and out["1_free"][:2] == (2, 4)
    for r in range(world):
        np.testing.assert_allclose(out[f"{r}_free"][2], ref["grads"].sum(0), atol=1e-12)
