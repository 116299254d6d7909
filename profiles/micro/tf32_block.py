"""Measurement behind the tensor-core decision: a dense k-qubit block on the
tensor cores against the packed-FP32 one-qubit kernels.

A k-qubit block on complex64 amplitudes is a real (2 * 2^k) x (2 * 2^k) matrix applied to
(2 * 2^k) x N real columns. B200 has no FP32 tensor path: the candidates are one TF32 GEMM
(10-bit mantissa: does it meet the 1e-5 / 1e-4 tolerances?) and the 3xTF32 split (hi/lo parts,
three GEMMs). cuBLAS through torch.matmul stands in for a hand-written tcgen05 kernel (an upper
bound on what the library reaches for these skinny shapes, not a product path).

Prints, per k: the worst error of the variants against fp64 relative to the rms amplitude of a
unit-norm state of 2^22 amplitudes, their time per amplitude, and the time per amplitude of k one-qubit groups at the
packed-FP32 rates the engine measures (4 packed ops per amplitude forward in the direct form, 2.3
in the merged Euler form, at 74 TFLOP/s peak and at the 55% the heavy kernels sustain).
usage: python profiles/micro/tf32_block.py"""
import torch

assert torch.cuda.is_available()
dev = torch.device("cuda")
n = 22
torch.manual_seed(0)


def tf32_round(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)  # keep 10 mantissa bits


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print(f"{'k':>2} {'variant':>8} {'err / rms amp':>13} {'ps/amplitude':>13} | k one-qubit groups on packed FP32 (ps/amplitude)")
for k in (3, 4, 5, 6):
    d = 1 << k
    N = (1 << n) // d
    # random unitary block, as the real 2d x 2d matrix acting on (re; im)
    q, _ = torch.linalg.qr(torch.randn(d, d, dtype=torch.complex128, device=dev))
    W = torch.cat([torch.cat([q.real, -q.imag], 1), torch.cat([q.imag, q.real], 1)], 0)
    x = torch.randn(2 * d, N, dtype=torch.float64, device=dev)
    x /= x.norm()  # unit-norm state
    ref = W @ x
    W32, x32 = W.float().contiguous(), x.float().contiguous()
    Wh, xh = tf32_round(W32), tf32_round(x32)
    Wl, xl = tf32_round(W32 - Wh), tf32_round(x32 - xh)
    torch.backends.cuda.matmul.allow_tf32 = True
    one = lambda: W32 @ x32  # noqa: E731
    three = lambda: Wh @ xh + (Wh @ xl + Wl @ xh)  # noqa: E731
    torch.backends.cuda.matmul.allow_tf32 = False
    fp32 = lambda: W32 @ x32  # noqa: E731
    rows = []
    for name, fn, tf in (("tf32", one, True), ("3xtf32", three, True), ("fp32", fp32, False)):
        torch.backends.cuda.matmul.allow_tf32 = tf
        err = (fn().double() - ref).abs().max().item() / ref.pow(2).mean().sqrt().item()
        ms = timed(fn)
        rows.append((name, err, ms * 1e9 / (1 << n)))
    peak = 74e12 / 4  # packed ops per second (one FFMA2 = 4 flop)
    cuda_cores = {f"{ops} ops/group": (k * ops / peak * 1e12, k * ops / (0.55 * peak) * 1e12) for ops in (4.0, 2.3)}
    cc = ", ".join(f"{nm}: {a:.2f} peak / {b:.2f} at 55%" for nm, (a, b) in cuda_cores.items())
    for i, (name, err, ps) in enumerate(rows):
        print(f"{k:2d} {name:>8} {err:13.3e} {ps:13.2f} | {cc if i == 0 else ''}")
print("amplitude scale of a unit-norm 2^22 state: %.1e; tolerance on <Z>: 1e-5 absolute" % (2.0 ** (-n / 2)))
