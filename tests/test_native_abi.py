"""The C-ABI library loads on the CPU host and exports every symbol include/*.h declares
(no compute calls without a GPU)."""

import ctypes
import glob
import os
import re

import pytest

from conftest import ROOT
from paper_2506_04891_b200 import _native


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        syms |= set(re.findall(r"\b(lsq_\w+)\s*\(", text))
    return syms


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("lsq_program_create", "lsq_forward", "lsq_fwd_bwd", "lsq_bwd_from_state", "lsq_last_error"):
        assert s in syms


@pytest.mark.skipif(not os.path.exists(_native.LIB_PATH), reason="library not built (run build())")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in sorted(declared_symbols()) if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_native.EXPORTS) <= declared_symbols()
    loaded = _native.load_library()
    assert loaded.lsq_version() == 1


def test_status_codes_map_to_reference_exceptions():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built")
    from paper_2506_04891_b200.errors import CapacityError, PlanMismatchError

    _native.load_library()
    with pytest.raises(ValueError):
        _native.check(1)
    with pytest.raises(PlanMismatchError):
        _native.check(2)
    with pytest.raises(CapacityError):
        _native.check(3)
    with pytest.raises(RuntimeError):
        _native.check(4)


def test_jit_uses_toolkit_nvrtc_not_first_loaded():
    """The JIT must use the toolkit's NVRTC even when torch's bundled (older) libnvrtc.so.12
    is already loaded in the process: the older ptxas leaves the FFMA2 lane swaps as MOVs."""
    import glob
    import os

    import torch

    for p in glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_nvrtc", "lib",
                                    "libnvrtc.so*")):
        ctypes.CDLL(p, mode=ctypes.RTLD_GLOBAL)
    path, ver, err = _native.jit_compiler().split("|", 2)
    assert not err, err
    maj, mnr = map(int, ver.split("."))
    assert (maj, mnr) >= (12, 9), (path, ver)


def test_program_artifact_roundtrip_and_loader_errors(tmp_path):
    """Artifact format (host side) round-trips; the C loader rejects malformed files with the
    documented status codes before touching the device."""
    from paper_2506_04891_b200 import artifact
    from paper_2506_04891_b200.configs import make_workload
    from paper_2506_04891_b200.schedule import compile_circuit

    wl = make_workload(2, n=10, batch=2)
    prog = compile_circuit(wl.circuit, M=8, R=4, prefix=True, fold=True, split=True)
    blob = artifact.encode(prog)
    d = artifact.decode(blob)
    assert list(d["words"]) == list(prog.words)
    assert len(d["kernels"]) == 2 * len(prog.passes)
    assert all(src.count("__global__") >= 1 for _, _, _, src, _, _ in d["kernels"])
    if not os.path.exists(_native.LIB_PATH):
        return
    lib = _native.load_library()
    h = ctypes.c_void_p()
    bad = tmp_path / "bad.lsqp"
    bad.write_bytes(b"NOPE" + blob[4:])
    assert lib.lsq_program_load(str(bad).encode(), None, ctypes.byref(h)) == 1
    ver = tmp_path / "ver.lsqp"
    ver.write_bytes(blob[:4] + (3).to_bytes(4, "little") + blob[8:])
    assert lib.lsq_program_load(str(ver).encode(), None, ctypes.byref(h)) == 2
    trunc = tmp_path / "trunc.lsqp"
    trunc.write_bytes(blob[: len(blob) // 2])
    assert lib.lsq_program_load(str(trunc).encode(), None, ctypes.byref(h)) == 1
    assert b"truncated" in lib.lsq_last_error() or b"corrupt" in lib.lsq_last_error()
