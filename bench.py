#!/usr/bin/env python
"""Benchmark: batched forward + adjoint-backward circuit evaluations per second.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One JSON line (rank 0). A step = one forward + adjoint backward of this GPU's row shard
(inputs resident in HBM) plus, for N > 1, the NCCL all-reduce of the shared-angle gradient.
Default workload: BASELINE cfg4 (n=22, batch 256), the largest config that fits one B200
without micro-batching; every config runs its BASELINE global batch split over the GPUs
(strong scaling; cfg5's 1024 rows are micro-batched at N=1). Before timing, the same compiled
engine must reproduce the reference-generated golden rows (`parity_gate`). `--impl reference`
times the reference itself (baseline/_ref, compiled backend, its own gradient() path) on the
host cores, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2506_04891_b200.configs import CONFIG_NAMES, CONFIG_SHAPES, make_workload  # noqa: E402

METRIC = "batched fwd+bwd circuit evals/s"
UNIT = "evals/s"
FALLBACK_HBM = 6650.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


FP32_PEAK_TFLOPS = 74.0  # measured: profiles/micro/ffma2_rate (packed FFMA2, B200, 1965 MHz)


def _fp32_view(per_kernel, dom_key):
    """FP32-pipe view of the roofline: the pass kernels are issue/FMA bound once fused, so
    the HBM fraction alone under-states how busy they are. achieved = executed FP32 flops of
    the launches (per-row counts from ncu source counters) / their CUDA-event time."""
    def one(v):
        if v.get("flops_missing") or not v.get("flops"):
            return None
        t = v["flops"] / (v["ms"] / 1e3) / 1e12
        return {"achieved": round(t, 2), "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(t / FP32_PEAK_TFLOPS, 4)}
    dom = one(per_kernel[dom_key])
    if dom is None:
        return None
    tot = {"flops": sum(v.get("flops", 0.0) for v in per_kernel.values()),
           "ms": sum(v["ms"] for v in per_kernel.values()),
           "flops_missing": any(v.get("flops_missing") for v in per_kernel.values())}
    return {"kernel": dom_key, **dom, "all_pass_kernels": one(tot),
            "peak_source": "profiles/micro/ffma2_rate.cu (measured)",
            "flops_source": "profiles/ncu_fp32.json (ncu source counters, executed FFMA2/FMUL2/FFMA/FMUL/FADD)"}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _workload_rows(cfg, world, rank, batch=None):
    """(workload, start, stop, global_batch, scaling) for this rank: the BASELINE global batch
    of the config, drawn once (independent of the world size) and split into contiguous
    balanced row shards -- strong scaling, as BASELINE.json's 1/2/4/8-GPU runs specify."""
    from paper_2506_04891_b200.distributed import check_shardable, shard_rows

    n, b = CONFIG_SHAPES[cfg]
    if batch is not None:  # experiments only: a reduced batch of the same circuit per GPU
        wl = make_workload(cfg, batch=batch * world)
        return wl, rank * batch, (rank + 1) * batch, batch * world, "weak"
    wl = make_workload(cfg)
    check_shardable(b, world)
    s, e = shard_rows(b, world, rank)
    return wl, s, e, b, "strong"


# ------------------------------------------------------------------------------ CPU legs
#
# The reference itself (arXiv 2506.04891's `layersim`, pip-installed UNMODIFIED into
# baseline/_ref with its compiled Cython backend) runs its own public `gradient()` path
# (reference grad.py:207-218) on the host cores: one process per core, one BLAS thread each,
# every process on a contiguous shard of the same seeded rows. Adapters (no reference file is
# modified): the weighted observable sum_q w_q Z_q by rebinding the module
# attributes `layersim.grad.z_weights` / `layersim.states.z_weights`; GPi/GPi2/MS angles are
# already in turns in the workload. The numpy oracle port is used only when baseline/_ref is
# absent, and is labelled "port".

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _ref_layersim():
    """The installed reference package, or None when baseline/_ref is absent."""
    if not os.path.isfile(os.path.join(REF_DIR, "layersim", "__init__.py")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import layersim

    if not os.path.abspath(layersim.__file__).startswith(os.path.abspath(REF_DIR)):
        raise RuntimeError(f"layersim imported from {layersim.__file__}, not {REF_DIR}")
    return layersim


def _to_ref_circuit(ls, circ):
    layers = []
    for layer in circ.layers:
        pat = ls.WirePattern(ls.PatternKind(layer.pattern.kind.value), layer.pattern.wires)
        role = None if layer.role is None else ls.Role(layer.role.value)
        layers.append(ls.Layer(ls.GateKind(layer.gate.value), pat, role, layer.values))
    return ls.Circuit(circ.n, layers)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or platform.machine()


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _sub_circuit(cfg, circ, nblocks):
    """Encoding prefix + the first `nblocks` repeated blocks of a BASELINE config circuit (the
    n >= 24 sample: whole blocks, never a partial layer prefix)."""
    from paper_2506_04891_b200.circuits import Circuit
    from paper_2506_04891_b200.configs import BLOCK_LAYOUT

    head, per, _ = BLOCK_LAYOUT[cfg]
    return Circuit(circ.n, list(circ.layers[: head + nblocks * per]))


def _ref_worker(args):
    """One process: `rows` (a contiguous shard) through the reference's gradient(), `reps` times.
    Returns the wall seconds of each rep."""
    cfg, rows, plan_text, reps, nblocks = args
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    wl = make_workload(cfg)
    circ = wl.circuit if nblocks is None else _sub_circuit(cfg, wl.circuit, nblocks)
    T, E = circ.trainable_count, circ.encoding_count
    ls = _ref_layersim()
    if ls is None:  # no reference install: the oracle port (labelled "port")
        from oracle import layersim_oracle as orc

        run = lambda xs: orc.gradient(circ, wl.theta[:T], xs, batch=xs.shape[0], weights=wl.weights)  # noqa: E731
    else:
        import layersim.grad as rg
        import layersim.states as rs
        from layersim.planner import parse_plan

        n = circ.n
        idx = np.arange(1 << n)
        d = np.zeros(1 << n)
        for q in range(n):
            d += wl.weights[q] * (1.0 - 2.0 * ((idx >> (n - 1 - q)) & 1))
        d.setflags(write=False)
        orig = rg.z_weights
        rg.z_weights = rs.z_weights = lambda m: d if m == n else orig(m)
        rc = _to_ref_circuit(ls, circ)
        plan = parse_plan(plan_text) if plan_text else None
        run = lambda xs: ls.gradient(rc, wl.theta[:T] if T else None, xs if E else None,  # noqa: E731
                                     batch=xs.shape[0], plan=plan)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for r0, r1 in rows:
            run(wl.x[r0:r1, :E])
        times.append(time.perf_counter() - t0)
    return times


class RefCPU:
    """Pool of one process per host core running the reference (or, absent, the port) on a
    bounded sample of the workload's rows. A step = every process runs its shard once; the
    step time is the wall time until the last process finishes."""

    def __init__(self, cfg):
        import multiprocessing as mp

        n, B = CONFIG_SHAPES[cfg]
        self.cfg, self.n = cfg, n
        self.kind = "reference" if _ref_layersim() is not None else "port"
        cores = _host_cores()
        # memory guard: ~8 complex128 state copies per process (state, lambda, einsum temporaries)
        try:
            import psutil

            avail = psutil.virtual_memory().available
            cores = max(1, min(cores, int(avail * 0.7) // (8 * (16 << n))))
        except Exception:
            pass
        self.nblocks = None
        if n <= 16:  # the whole BASELINE batch, contiguous shards
            rows = B
        else:  # one row per process
            rows = cores
        self.procs = min(cores, rows)
        base, extra = divmod(rows, self.procs)
        self.shards, s = [], 0
        for i in range(self.procs):
            e = s + base + (1 if i < extra else 0)
            self.shards.append([(s, e)])
            s = e
        self.rows = rows
        self.scale = 1.0
        if n >= 24:  # a full n=24 row takes minutes: time encoding + 1 block, scale to 6
            from paper_2506_04891_b200.configs import BLOCK_LAYOUT

            self.total_blocks = BLOCK_LAYOUT[cfg][2]
            self.nblocks = 1
        self.pool = mp.get_context("fork").Pool(self.procs)
        self.plan_text = None

    def step(self, reps=1):
        args = [(self.cfg, sh, self.plan_text, reps, self.nblocks) for sh in self.shards]
        t0 = time.perf_counter()
        per_proc = self.pool.map(_ref_worker, args)
        wall = time.perf_counter() - t0
        return wall, per_proc

    def build_autotuned_plan(self):
        """The reference's own planner, Objective.FORWARD_BACKWARD, at the per-process batch
        (reference planner.py:165-220); plan build is excluded from every timed region."""
        ls = _ref_layersim()
        if ls is None:
            return None
        from layersim.planner import Objective, build_plan, serialize_plan

        wl = make_workload(self.cfg, batch=1)
        circ = wl.circuit if self.nblocks is None else _sub_circuit(self.cfg, wl.circuit, self.nblocks)
        b = max(e - s for sh in self.shards for s, e in sh)
        t0 = time.perf_counter()
        # reps=3, warmup=1 instead of the defaults 10/3: the n=22 build takes ~4 min with the
        # defaults on one core; both settings pick the same kernels for the cfg4 circuit at n=16
        plan = build_plan(_to_ref_circuit(ls, circ), b, Objective.FORWARD_BACKWARD, reps=3, warmup=1)
        return serialize_plan(plan), time.perf_counter() - t0

    def describe(self):
        what = (f"{self.rows} rows of {CONFIG_NAMES[self.cfg]} in {self.procs} contiguous shards"
                if self.n <= 16 else f"{self.rows} rows of {CONFIG_NAMES[self.cfg]}, one per process")
        if self.nblocks is not None:
            what += (f"; each row runs the encoding + {self.nblocks} of {self.total_blocks} blocks"
                     f" (scaled by the measured per-block time, see `block_scaling`)")
        return what

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_baseline(cfg):
    """Our arm's reported CPU baseline: the reference on every host core, the same protocol as
    the reference arm with one timed step -- warm-up (cold), default plan, the reference's
    FORWARD_BACKWARD-autotuned plan; the faster of the two is the value."""
    rc = RefCPU(cfg)
    try:
        rc.step()  # warm-up: imports, the reference's constant caches
        wall, per = rc.step()
        plan_name = "default"
        built = rc.build_autotuned_plan()
        if built is not None:
            rc.plan_text = built[0]
            wall2, per2 = rc.step()
            if wall2 < wall:
                wall, per, plan_name = wall2, per2, "autotuned"
        out = {"value": rc.rows / wall, "unit": UNIT, "cores": rc.procs, "kind": rc.kind,
               "sample": rc.describe() + f"; {plan_name} plan (the faster of default and autotuned), "
                                         "1 BLAS thread per process",
               "cpu_model": _cpu_model(), "seconds_per_step": wall, "plan": plan_name,
               "one_core_evals_per_s": sum(e - s for sh in rc.shards[:1] for s, e in sh) / min(t[0] for t in per)}
        if rc.nblocks is not None:
            sc = _block_scaling(rc)
            out["value"] *= sc["row_scale_inverse"]
            out["one_core_evals_per_s"] *= sc["row_scale_inverse"]
            out["block_scaling"] = sc
        return out
    finally:
        rc.close()


def run_reference(args, world, rank):
    """`--impl reference`: the reference's own CPU path on the host cores (rank 0 only)."""
    if rank != 0:
        return
    cfg = args.config
    n, b = CONFIG_SHAPES[cfg]
    rc = RefCPU(cfg)
    try:
        rates = {}
        plan_build_s = None
        # warm-up 1: cold (imports, the reference's constant caches); warm-up 2: default plan;
        # warm-up 3: the reference's autotuned plan; the faster plan is the one timed
        rc.step()
        wall, _ = rc.step()
        rates["default"] = rc.rows / wall
        built = rc.build_autotuned_plan()
        chosen = "default"
        if built is not None:
            text, plan_build_s = built
            rc.plan_text = text
            wall, _ = rc.step()
            rates["autotuned"] = rc.rows / wall
            if rates["autotuned"] > rates["default"]:
                chosen = "autotuned"
            else:
                rc.plan_text = None
        for _ in range(max(0, args.warmup - 3)):
            rc.step()
        walls, one = [], []
        for _ in range(args.steps):
            wall, per = rc.step()
            walls.append(wall)
            one.append(min(t[0] for t in per))
        el = sum(walls)
        value = rc.rows * args.steps / el
        scale = None
        if rc.nblocks is not None:
            scale = _block_scaling(rc)
            value *= scale["row_scale_inverse"]
        desc = rc.describe() + f"; {chosen} plan, 1 BLAS thread per process"
        shard0 = sum(e - s for s, e in rc.shards[0])
        cpu = {"value": value, "unit": UNIT, "cores": rc.procs, "kind": rc.kind, "sample": desc,
               "cpu_model": _cpu_model(), "plan": chosen,
               "warmup_rates": {k: round(v, 6) for k, v in rates.items()},
               "plan_build_s": plan_build_s,
               "one_core_evals_per_s": shard0 / statistics.median(one) * (scale["row_scale_inverse"] if scale else 1.0),
               "step_seconds": {"mean": statistics.mean(walls), "std": statistics.pstdev(walls)}}
        if scale:
            cpu["block_scaling"] = scale
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128 (reference numpy/Cython, complex128)",
            "data": "synthetic (seeded BASELINE inputs, A5 draw order)",
            "config": {"workload": CONFIG_NAMES[cfg], "n_qubits": n, "global_batch": b,
                       "sample_rows": rc.rows, "parallelism": f"{rc.procs} host processes"},
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
    finally:
        rc.close()


def _block_scaling(rc):
    """n >= 24 sample: per-row time of (encoding + 1 block) and (encoding + 2 blocks), both
    measured on one process, extrapolated linearly to the config's block count."""
    r = (0, 1)
    t1 = min(_ref_worker((rc.cfg, [r], rc.plan_text, 1, 1)))
    t2 = min(_ref_worker((rc.cfg, [r], rc.plan_text, 1, 2)))
    per_block = max(t2 - t1, 1e-9)
    full = t1 + (rc.total_blocks - 1) * per_block
    return {"t_enc_plus_1_block_s": t1, "t_enc_plus_2_blocks_s": t2, "blocks": rc.total_blocks,
            "row_scale_inverse": t1 / full}


# ------------------------------------------------------------------------------ GPU leg


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 20 ms while the timed region runs.
    Samples are time-stamped and kept if they fall inside [mark_start, mark_end] (+-150 ms
    when the region is shorter than the sampling period)."""

    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_indices):
        self.idx = ",".join(str(i) for i in gpu_indices)
        self.proc = None
        self.t0 = self.t1 = None

    def _nvml_loop(self):
        """NVML poll every 2 ms (same counters as nvidia-smi, denser inside short regions)"""
        import pynvml

        bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
        hs = [pynvml.nvmlDeviceGetHandleByIndex(int(i)) for i in self.idx.split(",")]
        while not self.stop:
            now = time.time()
            if self.w0 is not None and (self.w1 is None or now <= self.w1):
                for h in hs:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.nv.append((sm, mx, sorted(k for k, b in bits.items() if r & b)))
            time.sleep(0.002)

    def __enter__(self):
        self.nv, self.stop, self.w0, self.w1 = [], False, None, None
        try:
            import threading

            import pynvml

            pynvml.nvmlInit()
            self.th = threading.Thread(target=self._nvml_loop, daemon=True)
            self.th.start()
        except Exception:
            self.th = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.idx, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the sampler start before the timed region
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        import datetime

        self.t0 = datetime.datetime.now()
        self.w0 = time.time()

    def mark_end(self):
        import datetime

        self.t1 = datetime.datetime.now()
        self.w1 = time.time()
        time.sleep(0.05)

    def __exit__(self, *a):
        self.stop = True
        if getattr(self, "th", None) is not None:
            self.th.join(timeout=1)
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        import datetime

        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        samples = []
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            if len(p) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f")
                samples.append((ts, float(p[2]), float(p[3]), p[5:9]))
            except ValueError:
                continue
        nv = list(getattr(self, "nv", []))
        if len(nv) >= 3:  # dense NVML samples inside the timed region
            reasons = sorted({r for x in nv for r in x[2]})
            return {"sm_mhz": statistics.median(x[0] for x in nv), "sm_max_mhz": max(x[1] for x in nv),
                    "reasons": reasons, "samples": len(nv), "source": "nvml, 2 ms"}
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        win = samples
        if self.t0 and self.t1:
            inside = [x for x in samples if self.t0 <= x[0] <= self.t1]
            if not inside:
                pad = datetime.timedelta(milliseconds=150)
                inside = [x for x in samples if self.t0 - pad <= x[0] <= self.t1 + pad]
            win = inside or samples
        reasons = set()
        for x in win:
            for nm, v in zip(names, x[3]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(x[1] for x in win), "sm_max_mhz": max(x[2] for x in win),
                "reasons": sorted(reasons), "samples": len(win), "source": "nvidia-smi, 20 ms"}


def _pass_vectors(prog, mode, pidx, adjoint="recompute"):
    """State-vector transfers (reads + writes of one (rows, 2^n) vector) of one launch."""
    L = len(prog.passes)
    if mode == 0:  # forward: read psi (not for the synthesized first pass) + write psi
        return (0 if pidx == 0 else 1) + 1
    if mode == 1:  # turnaround: read psi (unless synthesized), write lambda (unless last)
        return (0 if L == 1 else 1) + (1 if L > 1 else 0)
    # adjoint: read psi, lambda; write lambda (+ psi when un-computing) unless pass 0
    writes = 0 if pidx == 0 else (1 if adjoint == "ckpt" else 2)
    return 2 + writes


MODE_NAMES = {0: "forward", 1: "turnaround", 2: "adjoint"}


def _kernel_label(eng, mode, pidx):
    """Kernel family of one pass launch: the specialised kernels are lsq_jit_p<pass>_m<mode>
    (NVRTC, one per pass and mode), the generic ones lsq_pass_kernel<M, NV>."""
    M = eng.program.passes[pidx].M
    if eng.variant == "jit":
        return "lsq_jit_p*_m%d (%s, M=%d)" % (mode, MODE_NAMES[mode], M)
    return "lsq_pass_kernel<M=%d,NV=%d>" % (M, 1 if mode == 0 else 2)


GOLDEN_TAG = {1: "cfg1_full", 2: "cfg2_rows4", 3: "cfg3_rows2", 4: "cfg4_rows1", 5: "cfg5_rows1"}


def correctness_gate(eng, cfg, checkpoint):
    """Before timing: the SAME compiled engine (program, tile exponent, generated kernels,
    adjoint variant) runs the reference-generated golden rows of this config (the first rows of
    the seeded workload, tests/golden/make_golden.py) and must match them -- <Z_q> within 1e-5
    absolute, every per-row angle gradient (trainable and encoding) and the loss gradient within
    1e-4 relative under SURVEY §0.2 A2 (floor 1e-2 * max |g_ref| of the compared array). A mismatch raises CorrectnessError, as the reference's own bench
    aborts a planned run that disagrees with the default one (reference bench.py:200-207)."""
    import torch

    from paper_2506_04891_b200.errors import CorrectnessError

    g = dict(np.load(os.path.join(ROOT, "tests", "golden", GOLDEN_TAG[cfg] + ".npz")))
    b = int(g["batch"])
    dev = eng.device
    r = eng.fwd_bwd(torch.as_tensor(g["theta"], device=dev), torch.as_tensor(g["x"], device=dev), batch=b,
                    weights=torch.as_tensor(g["weights"], device=dev), checkpoint=checkpoint)
    zq = r["zq"].cpu().numpy()
    ang = np.concatenate([r["grads"].cpu().numpy(), r["encoding_grads"].cpu().numpy()], 1)
    ref = np.concatenate([g["grads"], g["encoding_grads"]], 1)
    zerr = float(np.abs(zq - g["zq"]).max())
    scale = np.maximum(np.abs(ref), 1e-2 * np.abs(ref).max())
    a2 = float((np.abs(ang - ref) / scale).max())
    norm = float(np.abs(ang - ref).max() / np.abs(ref).max())
    gs, gs_ref = r["grad_sum"].cpu().numpy(), g["grads"].sum(0)
    a2s = float((np.abs(gs - gs_ref) / np.maximum(np.abs(gs_ref), 1e-2 * np.abs(gs_ref).max())).max())
    out = {"golden": GOLDEN_TAG[cfg], "rows": b, "zq_abs_err": zerr, "grad_a2_rel_err": a2,
           "grad_normwise_err": norm, "grad_sum_a2_rel_err": a2s, "adjoint": r["native_mode"], "tile_bits": eng.program.passes[0].M,
           "tol": {"zq_abs": 1e-5, "grad_a2_rel": 1e-4}}
    if not (zerr <= 1e-5 and a2 <= 1e-4 and a2s <= 1e-4):
        raise CorrectnessError(f"bench program disagrees with the reference goldens: {out}")
    return out


def run_ours(args, world, rank, local):
    import torch

    from paper_2506_04891_b200 import gradient
    from paper_2506_04891_b200.engine import Engine

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    cfg = args.config
    wl, r0, r1, gbatch, scaling = _workload_rows(cfg, world, rank, args.batch)
    b = r1 - r0
    n = wl.n
    # the per-layer CUDA-variant plan: the one build_plan made for this config on a B200
    # (profiles/plans/cfg<C>.json, profiles/build_plans.py) when present, else the tile exponent
    # measured here by choose_tile_bits on a bounded row sample (plan build is excluded from the
    # timed region, as in the reference's bench); --M forces an all-FUSED plan
    from paper_2506_04891_b200.planner import KernelKind, load_plan, plan_for_tile_bits

    plan, tile_choice, plan_src = None, None, None
    plan_path = os.path.join(ROOT, "profiles", "plans", f"cfg{cfg}.json")
    if args.M is not None:
        plan, plan_src = plan_for_tile_bits(wl.circuit, b, args.M), f"--M {args.M}"
    elif os.path.exists(plan_path) and not args.no_plan:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")  # machine id of the box that built it
            plan = load_plan(plan_path)
        plan_src = os.path.relpath(plan_path, ROOT)
    else:
        from paper_2506_04891_b200.planner import Objective, choose_tile_bits

        prow = max(1, min(b, (2 << 30) // (8 << wl.n)))
        M_best, st = choose_tile_bits(wl.circuit, prow, Objective.FORWARD_BACKWARD, device=dev)
        if world > 1:  # one tiling for every rank (rank 0's measurement)
            import torch.distributed as dist

            mt = torch.tensor([M_best], device=dev, dtype=torch.int64)
            dist.broadcast(mt, src=0)
            M_best = int(mt.item())
        tile_choice = {"rows": prow, "ms": {str(m): round(v.mean_seconds * 1e3, 3) for m, v in st.items()}}
        plan, plan_src = plan_for_tile_bits(wl.circuit, b, M_best), "choose_tile_bits"
    from paper_2506_04891_b200.core import plan_kernels

    kinds = plan_kernels(wl.circuit, plan)  # validates the plan against the circuit
    sel = lambda kk: [i for i, k in enumerate(kinds) if k is kk]  # noqa: E731
    args.M = plan.tile_bits
    if args.R is None:
        # the engine the public gradient(plan=...) call resolves to (the same cached object), so
        # the e2e leg below runs the timed program with the same buffers and micro-batching
        from paper_2506_04891_b200.core import _engine

        eng = _engine(wl.circuit, plan, dev)
    else:
        eng = Engine(wl.circuit, device=dev, M=args.M, R=args.R, isolate=sel(KernelKind.ISOLATED),
                     direct=sel(KernelKind.DIRECT), split_layers=sel(KernelKind.SPLIT),
                     rebalance_budget=plan.rebalance_budget)
    ck = None if args.checkpoint is None else bool(args.checkpoint)
    gate = None
    if args.batch is None:  # BASELINE workloads only (golden rows are the first rows of the batch)
        gate = correctness_gate(eng, cfg, eng.adjoint_mode(b, ck) == "ckpt")
    theta = torch.as_tensor(wl.theta, device=dev)
    x = torch.as_tensor(wl.x[r0:r1], device=dev)
    w = torch.as_tensor(wl.weights, device=dev)
    # one forward+adjoint step = one CUDA-graph replay of the engine's launch sequence
    gstep = eng.make_step(b, rows=False, encoding_grads=False, checkpoint=ck,
                          graph=not args.no_graph)
    gstep.set_inputs(theta, x, w)
    bufs = None

    def step():
        r = gstep.run()
        if world > 1:
            import torch.distributed as dist

            dist.all_reduce(r["grad_sum"])
        return r

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    launches = eng.native.launch_count()
    mb = eng.last_micro_batch
    nchunks = (b + mb - 1) // mb
    with ClockSampler([local] if world == 1 else list(range(world))) as clk:
        barrier()
        clk.mark_start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        barrier()
        clk.mark_end()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = gbatch * args.steps / (ms / 1e3)

    # ---- roofline: per-launch CUDA events on the engine's stream (separate profiled steps)
    eng.native.set_profiling(True)
    per_kernel = {}
    sol = []  # (speed-of-light seconds, measured seconds, flops known) per profiled pass launch
    nprof = max(2, min(args.steps, 5))
    # executed FP32 flops per row of each pass kernel, from ncu source counters of the same
    # kernels (profiles/ncu_fp32.py); the launch times below are this run's own CUDA events
    fp32_key = f"cfg{cfg}_M{eng.program.passes[0].M}_R{eng.program.passes[0].R}"
    try:
        fp32_tab = json.load(open(os.path.join(ROOT, "profiles", "ncu_fp32.json")))
    except Exception:
        fp32_tab = {}
    for _ in range(nprof):
        eng.native.profile = []
        eng.fwd_bwd(theta, x, batch=b, weights=w, rows=False, encoding_grads=False, micro_batch=mb,
                    checkpoint=ck)
        for kind, t, rows_launch in eng.native.profile:
            mode, pidx = divmod(kind, 1000)
            vec = _pass_vectors(eng.program, mode, pidx, eng.last_adjoint)
            key = _kernel_label(eng, mode, pidx)
            d = per_kernel.setdefault(key, {"bytes": 0.0, "ms": 0.0, "launches": 0, "rows": 0})
            d["rows"] += rows_launch
            d["bytes"] += vec * rows_launch * (8 << n)
            d["ms"] += t
            d["launches"] += 1
            fl = fp32_tab.get(f"{fp32_key}|lsq_jit_p{pidx}_m{mode}", {}).get("flops_per_row")
            if fl is not None and eng.variant == "jit":
                d["flops"] = d.get("flops", 0.0) + fl * rows_launch
            else:
                d["flops_missing"] = True
            # per-launch speed of light: the larger of its FP32 and its HBM time at the peaks
            sol.append((max((fl or 0.0) * rows_launch / (FP32_PEAK_TFLOPS * 1e12),
                            vec * rows_launch * (8 << n) / (_peaks()[0] * 1e9)), t / 1e3, fl is not None))
    eng.native.set_profiling(False)
    peak, peak_src = _peaks()
    dom = max(per_kernel.items(), key=lambda kv: kv[1]["ms"])
    ach = dom[1]["bytes"] / (dom[1]["ms"] / 1e3) / 1e9
    all_b = sum(v["bytes"] for v in per_kernel.values())
    all_ms = sum(v["ms"] for v in per_kernel.values())
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            tab = json.load(open(prof))
            traffic = tab.get(f"{CONFIG_NAMES[cfg]}|{dom[0]}")
            cap_rows = tab.get(f"{CONFIG_NAMES[cfg]}|rows")  # rows per launch of the ncu capture
            if traffic is not None and cap_rows:
                traffic = round(traffic * (dom[1]["rows"] / dom[1]["launches"]) / cap_rows)
        except Exception:
            traffic = None
    roofline = {
        "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
        "frac": round(ach / peak, 4), "traffic": traffic, "peak_source": peak_src,
        "kernel": dom[0], "avg_launch_ms": dom[1]["ms"] / dom[1]["launches"],
        "bytes_per_launch": dom[1]["bytes"] / dom[1]["launches"],
        "all_pass_kernels": {"achieved": round(all_b / (all_ms / 1e3) / 1e9, 1),
                             "frac": round(all_b / (all_ms / 1e3) / 1e9 / peak, 4),
                             "share_of_step": round((all_ms / nprof) / (ms / args.steps), 4)},
        "fp32": _fp32_view(per_kernel, dom[0]),
        # every pass launch bounded by whichever of FP32 and HBM it needs more time for
        "speed_of_light": ({"frac": round(sum(a for a, _, _ in sol) / sum(b for _, b, _ in sol), 4),
                            "bound": "per launch max(executed FP32 flops / FP32 peak, algorithmic bytes / HBM peak)",
                            "fp32_peak_tflops": FP32_PEAK_TFLOPS, "hbm_peak_gbs": peak}
                           if sol and all(k for _, _, k in sol) else None),
        "per_kernel": {k: {"GBps": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1),
                           "ms_per_step": v["ms"] / nprof,
                           "launches_per_step": v["launches"] // nprof}
                       for k, v in per_kernel.items()},
    }

    # ---- e2e through the public API, host buffers in and out
    x_host = np.ascontiguousarray(wl.x[r0:r1])
    h2d = wl.theta.nbytes + x_host.nbytes + wl.weights.nbytes
    res = None
    for _ in range(1):
        res = gradient(wl.circuit, wl.theta, x_host, batch=b, weights=wl.weights, device=dev, plan=plan)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tq = time.perf_counter()
        res = gradient(wl.circuit, wl.theta, x_host, batch=b, weights=wl.weights, device=dev, plan=plan)
        if os.environ.get("LSQ_E2E_TRACE") == "1":
            print(f"gradient(): {1e3 * (time.perf_counter() - tq):.3f} ms", file=sys.stderr)
        if world > 1:
            import torch.distributed as dist

            gs = torch.as_tensor(res.grad_sum, device=dev)
            dist.all_reduce(gs)
            gs.cpu()
    barrier()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    d2h = res.value.nbytes + res.grads.nbytes + res.encoding_grads.nbytes + res.zq.nbytes + res.grad_sum.nbytes
    e2e = {"value": gbatch * args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h)}

    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline(cfg)
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "error": str(e)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "c64 (fp32 complex; fp64 reductions)",
        "data": "synthetic (seeded BASELINE inputs, A5 draw order)",
        "config": {"workload": CONFIG_NAMES[cfg], "n_qubits": n, "global_batch": gbatch,
                   "rows_per_gpu": b, "micro_batch": mb, "adjoint": eng.last_adjoint,
                   "parallelism": f"dp{world}",
                   "passes": len(eng.program.passes), "tile_bits": eng.program.passes[0].M,
                   "tile_bits_choice": tile_choice, "plan": plan_src,
                   "plan_variants": {k.value: sum(1 for x in kinds if x is k) for k in set(kinds)},
                   "rebalance_budget": plan.rebalance_budget,
                   "cuda_graph": gstep.graph is not None,
                   "reg_bits": eng.program.passes[0].R, "variant": eng.variant,
                   "l2": f"working set {2 * b * (8 << n) / 2**20:.0f} MiB (psi+lambda) vs 126 MB L2"
                         + (" -> inputs larger than L2" if 2 * b * (8 << n) > 126e6 else " (L2-resident)")},
        "parity_gate": gate,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--M", type=int, default=None, help="tile bits per pass (default: planner/engine)")
    ap.add_argument("--R", type=int, default=None, help="register bits per thread")
    ap.add_argument("--batch", type=int, default=None, help="experiments: rows per GPU (not a bench line)")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    ap.add_argument("--no-plan", action="store_true", help="ignore profiles/plans/cfg<C>.json (tile choice only)")
    ap.add_argument("--checkpoint", type=int, default=None, choices=[0, 1],
                    help="adjoint with forward checkpoints (1) or in-place un-computation (0); default: engine")
    args = ap.parse_args()
    world, rank, local = _dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
