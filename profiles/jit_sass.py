"""Offline SASS check of the JIT kernels (no GPU): generate a config's per-pass kernels, compile
them with the toolkit NVRTC for sm_100a, print per-kernel opcode histograms.
usage: python profiles/jit_sass.py CFG [M] [R] [--dump DIR] [--only p1_m2,...]"""
import argparse, collections, ctypes, os, re, subprocess, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04891_b200 import codegen
from paper_2506_04891_b200.configs import make_workload
from paper_2506_04891_b200.schedule import compile_circuit

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("M", type=int, nargs="?", default=12)
ap.add_argument("R", type=int, nargs="?", default=4)
ap.add_argument("--dump", default=None)
ap.add_argument("--only", default=None)
ap.add_argument("--no-prefix", action="store_true")
ap.add_argument("--no-split", action="store_true")
a = ap.parse_args()

lib = ctypes.CDLL(os.path.realpath("/usr/local/cuda/lib64/libnvrtc.so.12"))
OPTS = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo", b"-DNDEBUG"]


def compile_cubin(src):
    prog = ctypes.c_void_p()
    assert lib.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), b"k.cu", 0, None, None) == 0
    arr = (ctypes.c_char_p * len(OPTS))(*OPTS)
    rc = lib.nvrtcCompileProgram(prog, len(OPTS), arr)
    n = ctypes.c_size_t()
    lib.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
    log = ctypes.create_string_buffer(n.value)
    lib.nvrtcGetProgramLog(prog, log)
    if rc:
        raise RuntimeError(log.value.decode()[:3000])
    lib.nvrtcGetCUBINSize(prog, ctypes.byref(n))
    buf = ctypes.create_string_buffer(n.value)
    lib.nvrtcGetCUBIN(prog, buf)
    return buf.raw


wl = make_workload(a.cfg)
pre = not a.no_prefix
prog = compile_circuit(wl.circuit, M=a.M, R=a.R, prefix=pre, fold=pre, split=not a.no_split)
print(len(prog.passes), "passes")
only = set(a.only.split(",")) if a.only else None
tot = collections.Counter()
for pi, mode, name, src, sv in codegen.generate_kernels(prog):
    short = name.replace("lsq_jit_", "")
    if only and short not in only:
        continue
    cub = compile_cubin(src)
    with tempfile.NamedTemporaryFile(suffix=".cubin", delete=False) as f:
        f.write(cub)
    sass = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", f.name], capture_output=True, text=True).stdout
    os.unlink(f.name)
    ops = collections.Counter(m.group(1).split(".")[0] for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", sass))
    tot.update(ops)
    reg = re.search(r"REG:(\d+)", res)
    spill = re.search(r"STACK:(\d+)", res)
    print(f"{short:8s} regs={reg.group(1) if reg else '?'} stack={spill.group(1) if spill else '?'} total={sum(ops.values())} "
          + " ".join(f"{k}={v}" for k, v in ops.most_common(12)))
    if a.dump:
        os.makedirs(a.dump, exist_ok=True)
        open(os.path.join(a.dump, short + ".cu"), "w").write(src)
        open(os.path.join(a.dump, short + ".sass"), "w").write(sass)
print("ALL", " ".join(f"{k}={v}" for k, v in tot.most_common(16)))
