"""The C ABI on its own (no Engine): a program loaded from an artifact file by
`lsq_program_load` (the path a cgo/JNI host takes) and one program run concurrently from
several host threads on several streams (programs are immutable after construction).
Calls go through ctypes with torch only allocating the buffers."""

import ctypes
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_04891_b200 import _native, artifact  # noqa: E402
from paper_2506_04891_b200.configs import make_workload  # noqa: E402
from paper_2506_04891_b200.engine import Engine  # noqa: E402


def _info(h):
    o = (ctypes.c_int64 * 8)()
    _native.check(_native.lib().lsq_program_info(h, o))
    return {"n": o[0], "T": o[1], "E": o[2], "passes": o[3]}


def _call(h, wl, stream):
    """One lsq_fwd_bwd_ckpt on `stream` with buffers of its own; returns host results and the
    calling thread's launch count."""
    lib = _native.lib()
    inf = _info(h)
    b, n, T, E, L = wl.batch, inf["n"], inf["T"], inf["E"], inf["passes"]
    dev = torch.device("cuda")
    f64 = dict(dtype=torch.float64, device=dev)
    th = torch.as_tensor(wl.theta, **f64)
    x = torch.as_tensor(wl.x, **f64)
    w = torch.as_tensor(wl.weights, **f64)
    lam = torch.empty((b, 1 << n), dtype=torch.complex64, device=dev)
    ck = torch.empty((max(L - 1, 1), b, 1 << n), dtype=torch.complex64, device=dev)
    zq, val = torch.empty((b, n), **f64), torch.empty((b,), **f64)
    gr, gs, er = torch.empty((b, T), **f64), torch.empty((T,), **f64), torch.empty((b, E), **f64)
    ws = torch.empty(int(lib.lsq_workspace_bytes(h, b)), dtype=torch.uint8, device=dev)
    with torch.cuda.stream(stream):
        _native.check(lib.lsq_fwd_bwd_ckpt(h, b, th.data_ptr(), x.data_ptr(), E, w.data_ptr(), lam.data_ptr(),
                                           lam.data_ptr(), ck.data_ptr() if L > 1 else None, zq.data_ptr(),
                                           val.data_ptr(), gr.data_ptr(), gs.data_ptr(), er.data_ptr(),
                                           ws.data_ptr(), ctypes.c_void_p(stream.cuda_stream)))
        count = lib.lsq_last_launch_count(h)
    stream.synchronize()
    return {k: v.cpu().numpy() for k, v in dict(zq=zq, value=val, grads=gr, grad_sum=gs, egrads=er).items()}, count


def test_artifact_program_equals_engine(tmp_path):
    wl = make_workload(2, n=12, batch=5)
    eng = Engine(wl.circuit, M=9)
    assert len(eng.program.passes) > 1
    path = tmp_path / "cfg2_n12.lsqp"
    artifact.write(eng.program, str(path), eng.program_fwd)
    h = ctypes.c_void_p()
    _native.check(_native.lib().lsq_program_load(str(path).encode(), None, ctypes.byref(h)))
    try:
        got, count = _call(h, wl, torch.cuda.Stream())
        ref, count_ref = _call(eng.native.handle, wl, torch.cuda.Stream())
    finally:
        _native.lib().lsq_program_destroy(h)
    for k in ref:
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
    assert count == count_ref > 0


def test_one_program_concurrent_host_threads():
    """4 host threads x 3 calls of ONE program handle on 4 streams, each with its own buffers
    and workspace: every result equals the sequential one bit for bit, and each thread's
    launch count is its own call's."""
    wl = make_workload(5, n=13, batch=3)
    eng = Engine(wl.circuit, M=10)
    h = eng.native.handle
    ref, count_ref = _call(h, wl, torch.cuda.Stream())
    results, errors = [], []

    def worker():
        try:
            s = torch.cuda.Stream()
            for _ in range(3):
                results.append(_call(h, wl, s))
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ths = [threading.Thread(target=worker) for _ in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors
    assert len(results) == 12
    for got, count in results:
        assert count == count_ref
        for k in ref:
            np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
