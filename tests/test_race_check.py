"""Static shared-memory race check of every generated kernel (tests/race_check.py; the GPU
pool has no compute-sanitizer): no path through any kernel of any BASELINE config, tiling or
random circuit touches a shared buffer across threads without the barrier it needs, and the
check is not vacuous -- deleting any barrier inside the tile loop is reported."""

import re

import numpy as np
import pytest

from paper_2506_04891_b200 import codegen
from paper_2506_04891_b200.configs import make_workload
from paper_2506_04891_b200.schedule import compile_circuit
from race_check import check_kernel_source

CASES = [(1, 8, None), (2, 12, 9), (2, 16, 11), (2, 16, 12), (3, 12, 9), (3, 20, 12), (4, 14, 10),
         (4, 22, 12), (4, 22, 13), (5, 13, 10), (5, 24, 12)]


def _kernels(cfg, n, M, prefix=True):
    wl = make_workload(cfg, n=n, batch=2)
    prog = compile_circuit(wl.circuit, M=M, R=4 if (M or n) >= 9 else None, prefix=prefix, fold=prefix,
                           split=True)
    return prog, codegen.generate_kernels(prog)


def _kernels_r(cfg, n, M, prefix, R):
    wl = make_workload(cfg, n=n, batch=2)
    prog = compile_circuit(wl.circuit, M=M, R=R, prefix=prefix, fold=prefix, split=True)
    return prog, codegen.generate_kernels(prog)


@pytest.mark.parametrize("cfg,n,M", CASES)
def test_generated_kernels_race_free(cfg, n, M):
    for prefix in ((True, False) if n <= 16 else (True,)):
        prog, ks = _kernels(cfg, n, M, prefix)
        if (M or n) >= 10:  # the forward kernels' 2^5-amplitude register tiling (engine.forward_program)
            p5, k5 = _kernels_r(cfg, n, M, prefix, 5)
            ks = ks + [k for k in k5 if k[1] == 0]
        for pi, mode, name, src, _ in ks:
            pp = prog.passes[pi]
            hazards, npaths = check_kernel_source(src, name, pp.M)
            assert npaths > 0
            assert not hazards, f"{name}: {hazards[:3]}"


def test_random_circuit_kernels_race_free():
    import circuit_helpers as h

    for seed in (0, 3, 5, 7, 10):
        rng = np.random.default_rng(100 + seed)
        circ = h.random_circuit(rng, 10, 14)
        for M in (7, 8):
            prog = compile_circuit(circ, M=M, R=None, prefix=True, fold=True, split=True)
            for pi, mode, name, src, _ in codegen.generate_kernels(prog):
                hazards, _ = check_kernel_source(src, name, prog.passes[pi].M)
                assert not hazards, f"seed {seed} M={M} {name}: {hazards[:3]}"


def _tile_loop_span(src, name):
    start = src.index("for (int t = t0; t < t_end; ++t) {", src.index(name))
    depth, i = 0, start
    while True:
        c = src[i]
        if c == "{":
            depth += 1
        elif c == "}":
            depth -= 1
            if depth == 0:
                return start, i
        i += 1


@pytest.mark.parametrize("cfg,n,M", [(4, 22, 12), (2, 16, 11), (5, 13, 10), (3, 12, 9)])
def test_deleting_any_tile_loop_barrier_is_detected(cfg, n, M):
    prog, ks = _kernels(cfg, n, M)
    checked = 0
    # forward, adjoint and turnaround kernels of the first and last passes
    pick = {(0, 0), (0, 2), (1, 0), (1, 2), (len(prog.passes) - 1, 1)}
    for pi, mode, name, src, _ in ks:
        if (pi, mode) not in pick:
            continue
        lo, hi = _tile_loop_span(src, name)
        for m in re.finditer(r"__syncthreads\(\);", src):
            if not lo < m.start() < hi:
                continue
            mutant = src[: m.start()] + "/* removed */" + src[m.end():]
            hazards, _ = check_kernel_source(mutant, name, prog.passes[pi].M)
            assert hazards, f"{name}: barrier at line {src[:m.start()].count(chr(10))} removable undetected"
            checked += 1
    assert checked > 10
