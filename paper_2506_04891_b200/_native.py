"""ctypes binding of the sm_100a engine (`_lib/liblsq.so`, C ABI in include/layersim_cuda.h).

There is no CPU fallback: if the library is missing or no CUDA device is visible, every
entry point raises. Status codes map onto the reference's exception types
(`pkg/src/layersim/errors.py:4-13`).
"""

from __future__ import annotations

import ctypes
import os

from .errors import CapacityError, PlanMismatchError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "liblsq.so")

_lib = None

_c = ctypes
_P = _c.c_void_p
_I = _c.c_int
_I64 = _c.c_int64

_SIGS = {
    "lsq_version": (_I, []),
    "lsq_last_error": (_c.c_char_p, []),
    "lsq_device_info": (_I, [_I, _c.c_char_p, _I]),
    "lsq_program_create": (_I, [_P, _I64, _P, _I64, _c.POINTER(_P)]),
    "lsq_program_destroy": (None, [_P]),
    "lsq_program_jit": (_I, [_P, _I, _P, _P, _P, _P, _P, _P, _c.c_char_p, _I]),
    "lsq_program_info": (_I, [_P, _P]),
    "lsq_program_load": (_I, [_c.c_char_p, _c.c_char_p, _c.POINTER(_P)]),
    "lsq_workspace_bytes": (_I64, [_P, _I]),
    "lsq_forward": (_I, [_P, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "lsq_fwd_bwd": (_I, [_P, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lsq_fwd_bwd_ckpt": (_I, [_P, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lsq_bwd_from_state": (_I, [_P, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lsq_set_profiling": (_I, [_P, _I]),
    "lsq_last_pass_times": (_I, [_P, _P, _I, _P]),
    "lsq_last_launch_count": (_I, [_P]),
    "lsq_jit_compiler": (_I, [_c.c_char_p, _I]),
}

EXPORTS = tuple(_SIGS)


class NativeUnavailable(RuntimeError):
    pass


def load_library(path: str = LIB_PATH):
    """Load the shared library and declare every C entry point (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"CUDA engine library not built: {path} (run __graft_entry__.build() / make -C "
            "paper_2506_04891_b200/csrc)"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return load_library()


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (lib().lsq_last_error() or b"").decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise PlanMismatchError(msg)
    if rc == 3:
        raise CapacityError(msg)
    raise RuntimeError(f"CUDA engine error: {msg}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible: the engine has no CPU fallback")
    load_library()


def jit_compiler() -> str:
    buf = ctypes.create_string_buffer(1024)
    lib().lsq_jit_compiler(buf, 1024)
    return buf.value.decode()
