"""Multi-GPU batch data parallelism over NCCL (world size 2): the engine's device grad_sum is
all-reduced in place and equals the single-process full-batch gradient; per-row results equal
the corresponding rows. Skips on a one-GPU box (the gloo test covers the host logic there)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs two CUDA devices", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from paper_2506_04891_b200.configs import make_workload
    from paper_2506_04891_b200.distributed import data_parallel_gradient

    wl = make_workload(5, n=12, batch=7)
    (s, e), res, gs = data_parallel_gradient(wl.circuit, wl.theta, wl.x, wl.weights, device=f"cuda:{rank}")
    assert gs.is_cuda and gs.device.index == rank
    out[rank] = (s, e, gs.cpu().numpy(), res["grads"].cpu().numpy(), res["zq"].cpu().numpy())
    dist.destroy_process_group()


def test_nccl_world2_matches_single_process():
    from paper_2506_04891_b200 import gradient
    from paper_2506_04891_b200.configs import make_workload

    world = 2
    port = _free_port()
    out = mp.Manager().dict()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, start_method="spawn")
    wl = make_workload(5, n=12, batch=7)
    ref = gradient(wl.circuit, wl.theta, wl.x, batch=7, weights=wl.weights, device="cuda:0")
    for r in range(world):
        s, e, gs, grads, zq = out[r]
        np.testing.assert_allclose(gs, ref.grad_sum, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(grads, ref.grads[s:e], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(zq, ref.zq[s:e], atol=1e-12)
