#!/usr/bin/env python
"""Benchmark: batched forward + adjoint-backward circuit evaluations per second.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One JSON line (rank 0). A step = one forward + adjoint backward of this GPU's batch
(inputs resident in HBM) plus, for N > 1, the NCCL all-reduce of the shared-angle
gradient. Default workload: BASELINE configs[1] (cfg2, n=16, batch 512 per GPU, weak
scaling); --config 5 runs the 24-qubit, batch-1024 config sharded over the GPUs (strong
scaling). `--impl reference` times the reference algorithm on the host cores (the CPU
oracle port) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

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
    """(workload, start, stop, global_batch, scaling) for this rank."""
    n, b = CONFIG_SHAPES[cfg]
    if batch is not None:  # experiments only: reduced batch of the same circuit
        wl = make_workload(cfg, batch=batch * world)
        return wl, rank * batch, (rank + 1) * batch, batch * world, "weak"
    if cfg == 5:  # BASELINE: 1024 rows sharded over the GPUs
        from paper_2506_04891_b200.distributed import shard_rows

        wl = make_workload(cfg)
        s, e = shard_rows(b, world, rank)
        return wl, s, e, b, "strong"
    wl = make_workload(cfg, batch=b * world)  # b rows per GPU
    return wl, rank * b, (rank + 1) * b, b * world, "weak"


# ------------------------------------------------------------------------------ CPU leg


def _cpu_rows_worker(args):
    cfg, rows, prefix = args
    from oracle import layersim_oracle as orc

    wl = make_workload(cfg, batch=max(rows) + 1)
    out = 0
    for r in rows:
        c = wl.circuit
        if prefix is not None:
            from paper_2506_04891_b200.circuits import Circuit

            c = Circuit(c.n, c.layers[:prefix])
            th = wl.theta[: c.trainable_count]
            orc.gradient(c, th, wl.x[r : r + 1, : c.encoding_count], batch=1, weights=wl.weights)
        else:
            orc.gradient(c, wl.theta, wl.x[r : r + 1], batch=1, weights=wl.weights)
        out += 1
    return out


def _cpu_sample_plan(cfg):
    """(rows, layer prefix or None, extrapolation factor, description)."""
    n, _ = CONFIG_SHAPES[cfg]
    ncores = os.cpu_count() or 1
    if n <= 16:
        rows = ncores if n == 16 else 64 * ncores
        return rows, None, 1.0, f"{rows} full rows of cfg{cfg} (1 row per task, {ncores} processes)"
    # n >= 20: one full row takes minutes on one core; time a layer prefix of one row per
    # core and scale by the layer count (per-layer cost of the reference is uniform).
    wl = make_workload(cfg, batch=1)
    L = len(wl.circuit.layers)
    prefix = 1 + (L - 1) // (8 if n >= 22 else 4)
    return ncores, prefix, L / prefix, (
        f"{ncores} rows x first {prefix}/{L} layers of cfg{cfg} (fwd+adjoint of the prefix),"
        f" scaled by {L}/{prefix}"
    )


def cpu_baseline(cfg, steps=1):
    """Oracle port (reference algorithm, complex128 numpy) on all host cores."""
    import multiprocessing as mp

    rows, prefix, scale, desc = _cpu_sample_plan(cfg)
    ncores = os.cpu_count() or 1
    procs = min(ncores, rows)
    tasks = [(cfg, list(range(i, rows, procs)), prefix) for i in range(procs)]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            done = sum(pool.map(_cpu_rows_worker, tasks))
            times.append(time.perf_counter() - t0)
    per = statistics.mean(times) * scale
    return {"value": done / per, "unit": UNIT, "cores": procs, "kind": "port", "sample": desc,
            "seconds_per_sample": per}


def run_reference(args, world, rank):
    if rank != 0:
        return
    cfg = args.config
    n, b = CONFIG_SHAPES[cfg]
    import multiprocessing as mp

    rows, prefix, scale, desc = _cpu_sample_plan(cfg)
    ncores = os.cpu_count() or 1
    procs = min(ncores, rows)
    tasks = [(cfg, list(range(i, rows, procs)), prefix) for i in range(procs)]
    with mp.get_context("fork").Pool(procs) as pool:
        for _ in range(args.warmup):
            pool.map(_cpu_rows_worker, tasks)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_cpu_rows_worker, tasks)
        el = (time.perf_counter() - t0) * scale
    value = rows * args.steps / el
    _, _, gb, scaling = (None, None, b, "weak" if cfg != 5 else "strong")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded BASELINE inputs)",
        "config": {"workload": CONFIG_NAMES[cfg], "n_qubits": n, "global_batch": b, "sample_rows": rows},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    # tile exponent: measured by the planner on a bounded row sample (plan build excluded from
    # the timed region, as the reference's bench does), unless --M is given
    plan, tile_choice = None, None
    if args.M is None:
        from paper_2506_04891_b200.planner import Objective, choose_tile_bits, plan_for_tile_bits

        prow = max(1, min(b, (2 << 30) // (8 << wl.n)))
        M_best, st = choose_tile_bits(wl.circuit, prow, Objective.FORWARD_BACKWARD, device=dev)
        if world > 1:  # one tiling for every rank (rank 0's measurement)
            import torch.distributed as dist

            mt = torch.tensor([M_best], device=dev, dtype=torch.int64)
            dist.broadcast(mt, src=0)
            M_best = int(mt.item())
        tile_choice = {"rows": prow, "ms": {str(m): round(v.mean_seconds * 1e3, 3) for m, v in st.items()}}
        plan = plan_for_tile_bits(wl.circuit, b, M_best)
        args.M = M_best
    else:
        from paper_2506_04891_b200.planner import plan_for_tile_bits

        plan = plan_for_tile_bits(wl.circuit, b, args.M)  # the e2e leg compiles the same tiling
    eng = Engine(wl.circuit, device=dev, M=args.M, R=args.R)
    theta = torch.as_tensor(wl.theta, device=dev)
    x = torch.as_tensor(wl.x[r0:r1], device=dev)
    w = torch.as_tensor(wl.weights, device=dev)
    ck = None if args.checkpoint is None else bool(args.checkpoint)
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
            d = per_kernel.setdefault(key, {"bytes": 0.0, "ms": 0.0, "launches": 0})
            d["bytes"] += vec * rows_launch * (8 << n)
            d["ms"] += t
            d["launches"] += 1
            fl = fp32_tab.get(f"{fp32_key}|lsq_jit_p{pidx}_m{mode}", {}).get("flops_per_row")
            if fl is not None and eng.variant == "jit":
                d["flops"] = d.get("flops", 0.0) + fl * rows_launch
            else:
                d["flops_missing"] = True
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
            traffic = json.load(open(prof)).get(f"{CONFIG_NAMES[cfg]}|{dom[0]}")
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
                   "tile_bits_choice": tile_choice,
                   "cuda_graph": gstep.graph is not None,
                   "reg_bits": eng.program.passes[0].R, "variant": eng.variant,
                   "l2": f"working set {2 * b * (8 << n) / 2**20:.0f} MiB (psi+lambda) vs 126 MB L2"
                         + (" -> inputs larger than L2" if 2 * b * (8 << n) > 126e6 else " (L2-resident)")},
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
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--M", type=int, default=None, help="tile bits per pass (default: planner/engine)")
    ap.add_argument("--R", type=int, default=None, help="register bits per thread")
    ap.add_argument("--batch", type=int, default=None, help="experiments: rows per GPU (not a bench line)")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
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
