"""Program artifacts: a compiled circuit (program words, constants and the generated sm_100a
kernel sources) in one file that the C ABI loads without Python (`lsq_program_load`,
include/layersim_cuda.h). This is how a non-Python host (cgo, JNI, ...) gets a program: the
circuit compiler (schedule.py) and the kernel generator (codegen.py) run once, offline, and
the host only links liblsq.so.

Format (little-endian): b"LSQP", u32 version=2, i64 n_words, i64 n_fvals, i32 n_kernels,
int32 words[n_words], float64 fvals[n_fvals], then per kernel: i32 pass, i32 mode,
i32 stage_vecs, i32 reg_bits, i32 name_len, name, i64 src_len, src (version 1: no reg_bits).
"""

from __future__ import annotations

import struct

import numpy as np

MAGIC = b"LSQP"
VERSION = 2


def encode(prog, prog_fwd=None) -> bytes:
    """Serialize a compiled program (schedule.compile_circuit) with its generated kernels (the
    forward ones from `prog_fwd` when given, engine.forward_program)."""
    from . import codegen

    words = np.ascontiguousarray(prog.words, dtype="<i4")
    fvals = np.ascontiguousarray(prog.fvals, dtype="<f8")
    ks = codegen.kernel_set(prog, prog_fwd)
    out = [MAGIC, struct.pack("<Iqqi", VERSION, words.size, fvals.size, len(ks)), words.tobytes(), fvals.tobytes()]
    for pidx, mode, name, src, stage, rbits in ks:
        nb, sb = name.encode(), src.encode()
        out.append(struct.pack("<iiiii", pidx, mode, stage, rbits, len(nb)) + nb + struct.pack("<q", len(sb)) + sb)
    return b"".join(out)


def decode(blob: bytes) -> dict:
    """Parse an artifact (host-side check of the format the C loader reads)."""
    if blob[:4] != MAGIC:
        raise ValueError("not a program artifact")
    ver, nw, nf, nk = struct.unpack_from("<Iqqi", blob, 4)
    if ver not in (1, 2):
        raise ValueError(f"artifact version {ver} not in (1, 2)")
    off = 4 + struct.calcsize("<Iqqi")
    words = np.frombuffer(blob, "<i4", nw, off)
    off += 4 * nw
    fvals = np.frombuffer(blob, "<f8", nf, off)
    off += 8 * nf
    kernels = []
    for _ in range(nk):
        if ver >= 2:
            pidx, mode, stage, rbits, nl = struct.unpack_from("<iiiii", blob, off)
            off += 20
        else:
            (pidx, mode, stage, nl), rbits = struct.unpack_from("<iiii", blob, off), 0
            off += 16
        name = blob[off : off + nl].decode()
        off += nl
        (sl,) = struct.unpack_from("<q", blob, off)
        off += 8
        kernels.append((pidx, mode, name, blob[off : off + sl].decode(), stage, rbits))
        off += sl
    if off != len(blob):
        raise ValueError("trailing bytes in artifact")
    return {"words": words, "fvals": fvals, "kernels": kernels}


def write(prog, path: str, prog_fwd=None) -> int:
    blob = encode(prog, prog_fwd)
    with open(path, "wb") as f:
        f.write(blob)
    return len(blob)
