"""Device engine: a compiled circuit program bound to a CUDA device.

Owns the immutable native program (`lsq_program_create`), the device workspace and the
state buffers (torch complex64 tensors, i.e. float2 rows of 2^n amplitudes), and runs the
forward / forward+adjoint drivers of the C ABI on torch's current stream. Rows are
processed in micro-batches when psi+lambda for the whole batch would not fit in HBM
(SURVEY §7.4 H5); the shared-angle gradient is summed over micro-batches in a fixed order.
"""

from __future__ import annotations

import ctypes
import os
import sys
import time

import numpy as np
import torch

from . import _native
from .errors import CapacityError
from .schedule import compile_circuit

_STATE_FRACTION = 0.6  # of free device memory usable for psi + lambda


def _on_device(fn):
    """Run an Engine method with its device current: the native calls launch on the current
    device, with a stream and tables that belong to self.device."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *a, **k):
        with torch.cuda.device(self.device):
            return fn(self, *a, **k)

    return wrapper


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _dev_f64(a, device, shape=None):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        t = a.detach().to(device=device, dtype=torch.float64)
    else:
        t = torch.as_tensor(np.asarray(a, dtype=np.float64), device=device)
    t = t.contiguous()
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"parameter shape {tuple(t.shape)} != {tuple(shape)}")
    return t


class NativeProgram:
    """RAII wrapper of an lsq_program on one device."""

    def __init__(self, prog, device: torch.device):
        _native.require_cuda()
        self.prog = prog
        self.device = device
        lib = _native.lib()
        words = np.ascontiguousarray(prog.words, dtype=np.int32)
        fvals = np.ascontiguousarray(prog.fvals, dtype=np.float64)
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            _native.check(
                lib.lsq_program_create(
                    words.ctypes.data, words.size, fvals.ctypes.data, fvals.size, ctypes.byref(h)
                )
            )
        self.handle = h
        self._ws = {}
        self.jit = False
        self.profiling = False
        self.profile = []

    def attach_jit(self, cache_dir=None, prog_fwd=None):
        """Compile the per-pass specialised kernels (codegen.py) with NVRTC for sm_100a; with
        `prog_fwd` the forward kernels come from that register tiling (engine.forward_program)."""
        from . import codegen

        ks = codegen.kernel_set(self.prog, prog_fwd)
        n = len(ks)
        srcs = (ctypes.c_char_p * n)(*[k[3].encode() for k in ks])
        names = (ctypes.c_char_p * n)(*[k[2].encode() for k in ks])
        pidx = (ctypes.c_int * n)(*[k[0] for k in ks])
        modes = (ctypes.c_int * n)(*[k[1] for k in ks])
        stages = (ctypes.c_int * n)(*[k[4] for k in ks])
        regs = (ctypes.c_int * n)(*[k[5] for k in ks])
        if cache_dir is None:
            cache_dir = os.environ.get("LSQ_CACHE_DIR", os.path.join(os.path.expanduser("~"), ".cache", "lsq_jit"))
        if cache_dir:
            os.makedirs(cache_dir, exist_ok=True)
        with torch.cuda.device(self.device):
            _native.check(
                _native.lib().lsq_program_jit(
                    self.handle, n, ctypes.cast(srcs, ctypes.c_void_p), ctypes.cast(pidx, ctypes.c_void_p),
                    ctypes.cast(modes, ctypes.c_void_p), ctypes.cast(stages, ctypes.c_void_p),
                    ctypes.cast(regs, ctypes.c_void_p), ctypes.cast(names, ctypes.c_void_p),
                    cache_dir.encode() if cache_dir else None, 0,
                )
            )
        self.jit = True

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _native.lib().lsq_program_destroy(h)
            except Exception:
                pass
            self.handle = None

    def workspace_bytes(self, batch: int) -> int:
        nbytes = int(_native.lib().lsq_workspace_bytes(self.handle, batch))
        if nbytes < 0:
            raise ValueError("invalid batch for workspace")
        return nbytes

    def workspace(self, *batches: int) -> torch.Tensor:
        """One workspace large enough for every chunk size in `batches` (the carve of a chunk
        depends on its row count through the launch geometry and is not monotone in it, so a
        short last chunk can need more than a full one). The cached tensor is replaced when a
        larger one is needed; callers that capture it in a CUDA graph keep their own reference
        (GradStep), so a replaced workspace stays alive as long as a graph uses it."""
        nbytes = max(256, max(self.workspace_bytes(b) for b in batches if b > 0))
        ws = self._ws.get("ws")
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self._ws = {"ws": ws}
        return ws

    def set_profiling(self, on: bool):
        _native.check(_native.lib().lsq_set_profiling(self.handle, int(on)))
        self.profiling = bool(on)
        self.profile = []  # (kind, ms, rows) for every pass launch since profiling was enabled

    def pass_times(self):
        cap = 4096
        ms = (ctypes.c_float * cap)()
        kinds = (ctypes.c_int * cap)()
        n = _native.lib().lsq_last_pass_times(self.handle, ms, cap, kinds)
        return [(int(kinds[i]), float(ms[i])) for i in range(min(n, cap))]

    def launch_count(self) -> int:
        return int(_native.lib().lsq_last_launch_count(self.handle))


def forward_register_bits(M: int) -> int | None:
    """Register bits of the forward kernels when they differ from the program's (LSQ_R_FWD:
    0 = same as the adjoint's): one vector per thread leaves room for 2^5 amplitudes, which
    means fewer phase transposes; needs tiles of >= 2^10 amplitudes (>= 32 threads)."""
    r = int(os.environ.get("LSQ_R_FWD", "5"))
    return r if r > 0 and M - r >= 5 else None


def forward_program(circuit, prog, M=None, **kw):
    """The same pass partition compiled with the forward register tiling (or None): identical
    groups and tile wires per pass -- only the phase plans differ -- so its forward kernels run
    against the program's tables and checkpoints unchanged."""
    if not prog.passes:
        return None
    rf = forward_register_bits(prog.passes[0].M)
    if rf is None or rf == prog.passes[0].R or any(pp.M != prog.passes[0].M for pp in prog.passes):
        return None
    pf = compile_circuit(circuit, M=M, R=rf, fwd_only=True, **kw)
    same = len(pf.passes) == len(prog.passes) and all(
        a.groups == b.groups and a.tile_wires == b.tile_wires for a, b in zip(pf.passes, prog.passes))
    return pf if same else None


class Engine:
    """A circuit compiled for the device; the object behind the drop-in API."""

    def __init__(self, circuit, M: int | None = None, R: int | None = None, device=None, jit=None,
                 isolate=(), prefix=None, fold=None, split=None, direct=(), split_layers=(),
                 rebalance_budget=None):
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.type != "cuda":
            raise ValueError("the engine runs on CUDA devices only")
        if jit is False or os.environ.get("LSQ_JIT", "1") == "0":
            raise ValueError("the engine has one kernel family: the per-circuit specialised sm_100a kernels "
                             "(the run-time interpreting kernel was removed)")
        self.circuit = circuit
        self.n = int(circuit.n)
        if R is None:
            # 16 amplitudes per thread per vector once tiles are >= 9 bits (measured best,
            # profiles/r01)
            from .schedule import DEFAULT_M, DEFAULT_R_SPECIALISED, default_r

            m = min(self.n, M if M is not None else DEFAULT_M)
            R = DEFAULT_R_SPECIALISED if m >= 9 else default_r(m)
        if prefix is None:
            prefix = os.environ.get("LSQ_PREFIX", "1") != "0"
        # trailing diagonal / permutation groups folded into the observable: gradient-type
        # programs only
        if fold is None:
            fold = bool(prefix) and os.environ.get("LSQ_FOLD", "1") != "0"
        # diagonal gates split out of one-qubit groups when the remainder is cheaper
        if split is None:
            split = os.environ.get("LSQ_SPLIT", "1") != "0"
        kw = dict(isolate=isolate, prefix=prefix, fold=fold, split=split, direct=direct, split_layers=split_layers,
                  rebalance_budget=rebalance_budget)
        self.program = compile_circuit(circuit, M=M, R=R, **kw)
        self.program_fwd = forward_program(circuit, self.program, M=M, **kw)
        self.prefix = bool(self.program.prefix) or bool(self.program.obs)
        self.native = NativeProgram(self.program, self.device)
        self.native.attach_jit(prog_fwd=self.program_fwd)
        self.variant = "jit"
        self.T = self.program.trainable_count
        self.E = self.program.encoding_count

    # -- helpers ---------------------------------------------------------------------------
    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _params(self, trainable, encoding, weights, batch):
        th = _dev_f64(trainable, self.device, (self.T,)) if self.T else None
        if self.T and th is None:
            raise ValueError("circuit has trainable parameters but none given")
        x = None
        if self.E:
            if encoding is None:
                raise ValueError("circuit has encoding parameters but none given")
            x = _dev_f64(encoding, self.device)
            if x.ndim != 2 or x.shape != (batch, self.E):
                raise ValueError(f"encoding shape {tuple(x.shape)} != ({batch}, {self.E})")
        w = _dev_f64(weights, self.device, (self.n,)) if weights is not None else None
        return th, x, w

    def row_bytes(self, nvec: int) -> int:
        return nvec * (8 << self.n)

    def micro_batch(self, batch: int, nvec: int) -> int:
        # cudaMemGetInfo costs ~4 ms per call on B200: query once per (batch, nvec)
        key = (batch, nvec)
        cache = self.__dict__.setdefault("_mb_cache", {})
        if key in cache:
            return cache[key]
        free, _ = torch.cuda.mem_get_info(self.device)
        # buffers this engine already holds for a previous call count as available
        held = 0
        seen = set()
        for t in self.__dict__.get("_held_buffers") or ():
            if t is not None and t.data_ptr() not in seen:
                seen.add(t.data_ptr())
                held += t.numel() * t.element_size()
        cap = int((free + held) * _STATE_FRACTION) // self.row_bytes(nvec)
        if cap < 1:
            raise CapacityError(
                f"one row of 2^{self.n} amplitudes x {nvec} vectors does not fit in device memory"
            )
        cache[key] = min(batch, cap)
        return cache[key]

    # -- forward ----------------------------------------------------------------------------
    @_on_device
    def forward(self, trainable=None, encoding=None, state=None, batch=None, weights=None, want_z=False):
        """Evolve `state` ((B, 2^n) complex64 CUDA tensor, or None = |0..0> with `batch` rows)
        through the circuit into a NEW tensor. Returns (psi, zq, value)."""
        if self.program.obs:
            raise ValueError("this program folds its trailing permutations/diagonals into the "
                             "observable (gradient programs); compile with fold=False to get states")
        if state is not None:
            if self.prefix:
                raise ValueError("this program synthesizes its |0..0> prefix; compile with prefix=False "
                                 "to evolve an arbitrary input state")
            if not isinstance(state, torch.Tensor) or state.dtype != torch.complex64:
                raise ValueError("state must be a complex64 torch tensor")
            if state.device != self.device:
                state = state.to(self.device)
            state = state.contiguous()
            batch = state.shape[0]
            if state.shape[1] != (1 << self.n):
                raise ValueError(f"state has {state.shape[1]} amplitudes, expected 2^{self.n}")
        if batch is None or batch < 1:
            raise ValueError("batch must be positive")
        th, x, w = self._params(trainable, encoding, weights, batch)
        out = torch.empty((batch, 1 << self.n), dtype=torch.complex64, device=self.device)
        zq = torch.empty((batch, self.n), dtype=torch.float64, device=self.device) if want_z else None
        val = torch.empty((batch,), dtype=torch.float64, device=self.device) if want_z else None
        lib = _native.lib()
        mb = batch  # output buffer is the full batch already; process in one call
        ws = self.native.workspace(mb)
        _native.check(
            lib.lsq_forward(
                self.native.handle, batch, _ptr(th), _ptr(x), self.E, _ptr(w), _ptr(state),
                out.data_ptr(), _ptr(zq), _ptr(val), ws.data_ptr(), self._stream(),
            )
        )
        return out, zq, val

    # -- forward + adjoint ------------------------------------------------------------------------
    def adjoint_mode(self, batch: int, checkpoint=None) -> str:
        """'ckpt' (forward checkpoints, adjoint writes lambda only) when every pass output fits
        for a micro-batch of >= min(batch, 16) rows, else 'recompute' (psi un-computed in place)."""
        L = len(self.program.passes)
        if L == 1 or checkpoint is False:
            return "recompute"
        if checkpoint is True:
            return "ckpt"
        env = os.environ.get("LSQ_ADJOINT")
        if env in ("ckpt", "recompute"):
            return env
        return "ckpt" if self.micro_batch(batch, L) >= min(batch, 16) else "recompute"

    @_on_device
    def fwd_bwd(self, trainable=None, encoding=None, batch=1, weights=None, rows=True,
                encoding_grads=True, micro_batch=None, buffers=None, checkpoint=None, out=None):
        """Forward from |0..0> plus adjoint backward. Returns a dict of CUDA tensors:
        value (B,), zq (B,n), grads (B,T) if rows, grad_sum (T,), encoding_grads (B,E).
        `out`: optional preallocated float64 tensors with those keys (written in place)."""
        th, x, w = self._params(trainable, encoding, weights, batch)
        mode = self.adjoint_mode(batch, checkpoint)
        L = len(self.program.passes)
        nvec = L if mode == "ckpt" else 2
        env_mb = int(os.environ.get("LSQ_MICRO_BATCH", "0"))  # experiments (L2-resident micro-batches)
        mb = micro_batch or (min(env_mb, batch) if env_mb > 0 else self.micro_batch(batch, nvec))
        self.last_micro_batch, self.last_adjoint = mb, mode
        dev = self.device
        f64 = dict(dtype=torch.float64, device=dev)
        o = out or {}
        value = o["value"] if "value" in o else torch.empty((batch,), **f64)
        zq = o["zq"] if "zq" in o else torch.empty((batch, self.n), **f64)
        grows = None
        if rows and self.T:
            grows = o["grads"] if o.get("grads") is not None else torch.empty((batch, self.T), **f64)
        erows = None
        if encoding_grads and self.E:
            erows = (o["encoding_grads"] if o.get("encoding_grads") is not None
                     else torch.empty((batch, self.E), **f64))
        nchunk = (batch + mb - 1) // mb
        if nchunk == 1 and o.get("grad_sum") is not None and self.T:
            gparts = o["grad_sum"].view(1, self.T)
        else:
            gparts = torch.zeros((nchunk, max(self.T, 1)), **f64)
        def fits(bufs):
            if bufs is None or bufs[0].shape[0] < mb:
                return False
            if mode == "recompute":  # separate psi and lambda, no checkpoint slots
                return bufs[2] is None and bufs[0] is not bufs[1]
            return bufs[2] is not None and bufs[2].shape[1] >= mb and bufs[2].shape[0] >= L - 1

        held = self.__dict__.get("_held_buffers")
        if buffers is not None and len(buffers) == 3 and fits(buffers):
            psi, lam, ck = buffers
        elif held is not None and fits(held):
            psi, lam, ck = held
        else:
            self._held_buffers = None
            lam = torch.empty((mb, 1 << self.n), dtype=torch.complex64, device=dev)
            if mode == "ckpt":
                ck = torch.empty((L - 1, mb, 1 << self.n), dtype=torch.complex64, device=dev)
                psi = lam  # psi is not stored by any pass in checkpoint mode (L > 1)
            else:
                ck = None
                psi = torch.empty_like(lam)
            self._held_buffers = (psi, lam, ck)
        ws = self.native.workspace(mb, batch - (nchunk - 1) * mb)
        lib = _native.lib()
        for c in range(nchunk):
            r0 = c * mb
            b = min(mb, batch - r0)
            xc = x[r0 : r0 + b] if x is not None else None
            ck_ptr = None
            if ck is not None:
                # the checkpoint layout is (L-1) slots of b rows each: compact view for this chunk
                ck_ptr = ck.data_ptr() if b == ck.shape[1] else ck.view(-1)[: (L - 1) * (b << self.n)].data_ptr()
            _native.check(
                lib.lsq_fwd_bwd_ckpt(
                    self.native.handle, b, _ptr(th), _ptr(xc), self.E, _ptr(w),
                    psi.data_ptr(), lam.data_ptr(), ck_ptr, zq[r0].data_ptr(), value[r0].data_ptr(),
                    grows[r0].data_ptr() if grows is not None else None,
                    gparts[c].data_ptr() if self.T else None,
                    erows[r0].data_ptr() if erows is not None else None,
                    ws.data_ptr(), self._stream(),
                )
            )
            if self.native.profiling:
                self.native.profile += [(k, ms, b) for k, ms in self.native.pass_times()]
        gsum = gparts.sum(dim=0)[: self.T] if nchunk > 1 else gparts[0, : self.T]
        if o.get("grad_sum") is not None and gsum.data_ptr() != o["grad_sum"].data_ptr():
            o["grad_sum"].copy_(gsum)
            gsum = o["grad_sum"]
        return {"value": value, "zq": zq, "grads": grows, "grad_sum": gsum, "encoding_grads": erows,
                "buffers": (psi, lam, ck), "workspace": ws, "adjoint": mode,
                "native_mode": "ckpt" if ck is not None else "recompute"}

    def make_step(self, batch, rows=True, encoding_grads=True, checkpoint=None, graph=None):
        """A reusable forward+adjoint step with static device inputs/outputs, replayed as one
        CUDA graph (the whole launch sequence: tables, passes, reductions, contraction)."""
        return GradStep(self, batch, rows, encoding_grads, checkpoint, graph)

    @_on_device
    def backward_from_state(self, trainable, encoding, final_state, weights=None):
        """Adjoint sweep from a given final state (reference backward_sweep)."""
        if self.prefix:
            raise ValueError("backward_from_state needs a program compiled with prefix=False")
        if not isinstance(final_state, torch.Tensor) or final_state.dtype != torch.complex64:
            raise ValueError("final state must be a complex64 torch tensor")
        final_state = final_state.to(self.device).contiguous()
        batch = final_state.shape[0]
        th, x, w = self._params(trainable, encoding, weights, batch)
        f64 = dict(dtype=torch.float64, device=self.device)
        value = torch.empty((batch,), **f64)
        zq = torch.empty((batch, self.n), **f64)
        grows = torch.empty((batch, max(self.T, 1)), **f64)
        erows = torch.empty((batch, max(self.E, 1)), **f64)
        gsum = torch.empty((max(self.T, 1),), **f64)
        psi = torch.empty_like(final_state)
        lam = torch.empty_like(final_state)
        ws = self.native.workspace(batch)
        _native.check(
            _native.lib().lsq_bwd_from_state(
                self.native.handle, batch, _ptr(th), _ptr(x), self.E, _ptr(w), final_state.data_ptr(),
                psi.data_ptr(), lam.data_ptr(), zq.data_ptr(), value.data_ptr(),
                grows.data_ptr() if self.T else None, gsum.data_ptr() if self.T else None,
                erows.data_ptr() if self.E else None, ws.data_ptr(), self._stream(),
            )
        )
        return {"value": value, "zq": zq, "grads": grows[:, : self.T], "grad_sum": gsum[: self.T],
                "encoding_grads": erows[:, : self.E]}


_TRACE = os.environ.get("LSQ_E2E_TRACE") == "1"


class GradStep:
    """Static-buffer forward+adjoint step captured in a CUDA graph.

    `run(theta, x, w)` copies new inputs (host or device) into the static buffers and replays
    the graph; `out` holds the static output tensors (value, zq, grads, grad_sum,
    encoding_grads). Graphs are disabled with LSQ_GRAPHS=0 (eager replay of the same calls).
    """

    def __init__(self, eng, batch, rows=True, encoding_grads=True, checkpoint=None, graph=None):
        self.eng = eng
        self.batch = int(batch)
        dev = eng.device
        f64 = dict(dtype=torch.float64, device=dev)
        B, T, E, n = self.batch, eng.T, eng.E, eng.n
        # one flat input buffer (theta | x | w) and one flat output buffer (value | zq | grads |
        # grad_sum | encoding_grads): host I/O is one pinned copy each way (run_host)
        nT, nE = max(T, 1), max(E, 1)
        self.d_in = torch.zeros((nT + B * nE + n,), **f64)
        self.theta = self.d_in[:nT]
        self.x = self.d_in[nT : nT + B * nE].view(B, nE)
        self.w = self.d_in[nT + B * nE :]
        self.w.fill_(1.0)
        sizes = [("value", (B,)), ("zq", (B, n))]
        if rows and T:
            sizes.append(("grads", (B, T)))
        if T:
            sizes.append(("grad_sum", (T,)))
        if encoding_grads and E:
            sizes.append(("encoding_grads", (B, E)))
        tot = sum(int(np.prod(sh)) for _, sh in sizes)
        self.d_out = torch.zeros((tot,), **f64)
        self.out_views, off = {}, 0
        for k, sh in sizes:
            m = int(np.prod(sh))
            self.out_views[k] = (off, sh)
            off += m
        self.outbuf = {k: self.d_out[o : o + int(np.prod(sh))].view(sh) for k, (o, sh) in self.out_views.items()}
        self.h_in = self.h_out = None
        self.kw = dict(batch=self.batch, rows=rows, encoding_grads=encoding_grads, checkpoint=checkpoint)
        if graph is None:
            graph = os.environ.get("LSQ_GRAPHS", "1") != "0"
        self.graph = None
        self.out = self._call()  # warm-up: JIT, workspace, buffers, micro-batch sizing
        if graph:
            torch.cuda.synchronize(dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.device(dev), torch.cuda.graph(g):
                self.out = self._call()
            self.graph = g
        # the graph holds raw addresses of the workspace and state buffers it captured: keep
        # them alive for the step's lifetime, whatever later calls on the engine allocate
        self._captured = (self.out.get("workspace"), self.out.get("buffers"))

    def _call(self):
        e = self.eng
        th = self.theta[: e.T] if e.T else None
        x = self.x[:, : e.E] if e.E else None
        return e.fwd_bwd(th, x, weights=self.w, out=self.outbuf, **self.kw)

    def set_inputs(self, theta=None, x=None, w=None):
        e = self.eng
        if theta is not None and e.T:
            self.theta[: e.T].copy_(torch.as_tensor(np.asarray(theta, dtype=np.float64)) if not isinstance(theta, torch.Tensor) else theta)
        if x is not None and e.E:
            self.x[:, : e.E].copy_(torch.as_tensor(np.asarray(x, dtype=np.float64)) if not isinstance(x, torch.Tensor) else x)
        if w is not None:
            self.w.copy_(torch.as_tensor(np.asarray(w, dtype=np.float64)) if not isinstance(w, torch.Tensor) else w)

    def run(self, theta=None, x=None, w=None):
        self.set_inputs(theta, x, w)
        if self.graph is not None:
            self.graph.replay()
        else:
            self.out = self._call()
        return self.out

    def run_host(self, theta=None, x=None, w=None) -> dict:
        """Host numpy in, host numpy out: the inputs are packed into a pinned staging buffer and
        sent with ONE host-to-device copy, the graph is replayed, and every output comes back
        with ONE device-to-host copy (then copied out of the reused pinned buffer)."""
        e = self.eng
        if self.h_in is None:
            self.h_in = torch.empty(self.d_in.shape, dtype=torch.float64, pin_memory=True)
            self.h_out = torch.empty(self.d_out.shape, dtype=torch.float64, pin_memory=True)
            self.h_in.copy_(self.d_in)
        hi = self.h_in.numpy()
        nT, nE = self.theta.shape[0], self.x.shape[1]
        if theta is not None and e.T:
            hi[: e.T] = np.asarray(theta, dtype=np.float64).reshape(-1)
        if x is not None and e.E:
            hi[nT : nT + self.batch * nE].reshape(self.batch, nE)[:, : e.E] = np.asarray(x, dtype=np.float64)
        if w is not None:
            hi[nT + self.batch * nE :] = np.asarray(w, dtype=np.float64).reshape(-1)
        stream = torch.cuda.current_stream(e.device)
        t0 = time.perf_counter() if _TRACE else 0.0
        self.d_in.copy_(self.h_in, non_blocking=True)
        if self.graph is not None:
            self.graph.replay()
        else:
            self.out = self._call()
        self.h_out.copy_(self.d_out, non_blocking=True)
        t1 = time.perf_counter() if _TRACE else 0.0
        stream.synchronize()
        t2 = time.perf_counter() if _TRACE else 0.0
        ho = self.h_out.numpy()
        out = {k: ho[o : o + int(np.prod(sh))].reshape(sh).copy() for k, (o, sh) in self.out_views.items()}
        if _TRACE:
            t3 = time.perf_counter()
            print(f"run_host: launch {1e3 * (t1 - t0):.3f} ms, wait {1e3 * (t2 - t1):.3f} ms, "
                  f"unpack {1e3 * (t3 - t2):.3f} ms", file=sys.stderr)
        return out


_CACHE: "OrderedDict" = None
_CACHE_MAX = 8  # engines (programs + held state buffers) kept alive, least recently used evicted


def engine_for(circuit, device=None, M=None, R=None, jit=None, isolate=(), prefix=None, direct=(),
               split_layers=(), rebalance_budget=None) -> Engine:
    """Cached Engine per (circuit layers, n, tiling, variant, device)."""
    dev = torch.device(device if device is not None else "cuda")
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    global _CACHE
    if _CACHE is None:
        from collections import OrderedDict

        _CACHE = OrderedDict()
    isolate = tuple(sorted(set(int(i) for i in isolate)))
    direct = tuple(sorted(set(int(i) for i in direct)))
    split_layers = tuple(sorted(set(int(i) for i in split_layers)))
    key = (_circuit_key(circuit), M, R, jit, isolate, prefix, direct, split_layers, rebalance_budget, str(dev))
    eng = _CACHE.get(key)
    if eng is None:
        eng = Engine(circuit, M=M, R=R, device=dev, jit=jit, isolate=isolate, prefix=prefix, direct=direct,
                     split_layers=split_layers, rebalance_budget=rebalance_budget)
        _CACHE[key] = eng
        while len(_CACHE) > _CACHE_MAX:
            _CACHE.popitem(last=False)
    else:
        _CACHE.move_to_end(key)
    return eng


def _circuit_key(circuit):
    layers = []
    for l in circuit.layers:
        layers.append(
            (l.gate.value, l.pattern.kind.value, tuple(map(tuple, l.pattern.wires)),
             None if l.role is None else l.role.value, l.values)
        )
    return (int(circuit.n), tuple(layers))
