"""Static shared-memory race check of the generated pass kernels -- TEST INFRASTRUCTURE.

compute-sanitizer (racecheck/synccheck) is not available on the GPU pool, so the barrier
discipline of every kernel codegen emits is verified statically instead. Every access to the
big shared buffers is a whole-tile permutation: each thread writes (or reads) its own 2^R
amplitudes of the tile, in a layout that differs from the previous one. So any two accesses of
one buffer by the block -- write/read, read/write, write/write -- touch other threads' data and
must be separated by a __syncthreads(). cp.async prefetches are writes that are in flight from
their issue until the issuing thread's cp_async_wait_all() and visible to the block only after
the barrier that follows it.

The kernel text is parsed into its brace tree; every path through the uniform branches
(`if (do_load)`, `if (nofwd)`/`else`, `if (t + 1 < t_end)`, ...) that contain buffer accesses or
barriers is simulated, with the tile loop unrolled twice (prologue -> tile t -> tile t + 1 ->
epilogue) so hazards across the loop back edge are seen. Buffers: `s_x` (exchange buffer) and
the prefetch stage's two vector regions (`s_stage`, `s_stage + 2^M`, also used as exchange
buffers by the rotating-buffer scheme).
"""

from __future__ import annotations

import itertools
import re


class Node:
    def __init__(self, header=None):
        self.header = header  # None for the root / plain statement lists
        self.items = []  # str statements or Node blocks


def parse_blocks(body: str) -> Node:
    """Brace tree of the kernel body (the generated code puts every '{' / '}' at a line end or
    as a whole '}' line, or a whole one-line block `{ ... }`)."""
    root = Node()
    stack = [root]
    alias = {}  # shared pointers off a buffer (codegen SWZ_IMM): name -> buffer expression
    for raw in body.splitlines():
        line = raw.strip()
        if not line:
            continue
        m = re.search(r"float2\* const (\w+) = (\(s_stage \+ \d+\)|s_x|s_stage) \+", line)
        if m:  # a (re)definition: no accesses on this line
            alias[m.group(1)] = m.group(2)
            continue
        for name, bexpr in alias.items():
            if name in line:
                line = re.sub(r"\b" + re.escape(name) + r"\b", bexpr, line)
        opens, closes = line.count("{"), line.count("}")
        if line.startswith("}") and "else" in line and line.endswith("{"):  # "} else {"
            if len(stack) > 1:
                stack.pop()
            nd = Node("else")
            stack[-1].items.append(nd)
            stack.append(nd)
            continue
        if opens == closes:  # one-line statement or one-line block
            stack[-1].items.append(line)
            continue
        if opens > closes:  # "header {" (possibly with statements before the brace)
            nd = Node(line[: line.rindex("{")].strip())
            stack[-1].items.append(nd)
            stack.append(nd)
            continue
        # closing line ("}", "} }", or statements followed by closing braces)
        pre = line[: line.index("}")].strip()
        if pre:
            stack[-1].items.append(pre)
        for _ in range(closes - opens):
            if len(stack) > 1:
                stack.pop()
    return root


_EV_PATTERNS = [
    (re.compile(r"__syncthreads\(\)"), "BAR"),
    (re.compile(r"cp_async_wait_all\(\)"), "WAIT"),
]


def _region(buf_expr: str, idx_expr: str, M: int):
    buf_expr = buf_expr.strip()
    if buf_expr == "s_x":
        return "x"
    base = 0
    m = re.match(r"\(s_stage \+ (\d+)\)", buf_expr)
    if m:
        base = int(m.group(1))
    elif buf_expr != "s_stage":
        return None
    m = re.match(r"\s*(\d+) \+", idx_expr)
    if m:
        base += int(m.group(1))
    return f"stage{base >> M}"


_SMALL = [
    # tables staged once (cross-thread writes, read by every thread afterwards)
    (re.compile(r"\bs_mat\[[^\]]*\]\s*=(?!=)"), "W", "mat"),
    (re.compile(r"\bs_mat \+"), "R", "mat"),
    (re.compile(r"\bs_acc\[i\]\s*=(?!=)"), "W", "acc"),
    (re.compile(r"\bs_z\[i\]\s*=(?!=)"), "W", "z"),
    (re.compile(r"\bs_zw\[i\]\s*=(?!=)"), "W", "zw"),
    # per-warp accumulation slots (each warp adds into its own: no hazard among themselves)
    (re.compile(r"\bwacc\b(?!\s*=)"), "A", "acc"),
    (re.compile(r"\bzw\["), "A", "zw"),
    # end-of-CTA flush: one thread per value reads every warp's slot
    (re.compile(r"\bs_acc\[ww \*"), "R", "acc"),
    (re.compile(r"\bs_zw\[ww \*"), "R", "zw"),
]


def events(stmt: str, M: int):
    """Buffer events of one statement, in order: ('BAR'|'WAIT', None), ('R'|'W'|'A'|'ASYNC',
    region). 'A' = per-warp accumulation into the warp's own slots."""
    out = []
    for pat, kind, reg in _SMALL:
        if pat.search(stmt) and not re.match(r"(float|double)\* (wacc|zw|s_acc|s_z|s_zw|s_mat|s_stage)\b", stmt) \
                and "(void)" not in stmt:
            out.append((kind, reg))
    for pat, kind in _EV_PATTERNS:
        if pat.search(stmt):
            out.append((kind, None))
    for m in re.finditer(r"cp_async16\(s_stage \+ (\d+)", stmt):
        out.append(("ASYNC", f"stage{int(m.group(1)) >> M}"))
    for m in re.finditer(r"\b(st_pair|ld_pair)\((\(s_stage \+ \d+\)|s_stage|s_x), ([^,]+),", stmt):
        reg = _region(m.group(2), m.group(3), M)
        out.append(("W" if m.group(1) == "st_pair" else "R", reg))
    buf = r"(\(s_stage \+ \d+\)|\bs_x|\bs_stage)"
    for m in re.finditer(buf + r"\[([^\]]*)\]\s*=(?!=)", stmt):
        out.append(("W", _region(m.group(1), m.group(2), M)))
    for m in re.finditer(r"=\s*" + buf + r"\[([^\]]*)\]", stmt):
        out.append(("R", _region(m.group(1), m.group(2), M)))
    return out


def _has_events(node, M) -> bool:
    for it in node.items:
        if isinstance(it, Node):
            if _has_events(it, M):
                return True
        elif events(it, M):
            return True
    return False


def _eval_atom(atom: str, env: dict):  # noqa: C901
    atom = atom.strip().strip("()").strip()
    if atom in ("do_load", "nofwd"):
        return env[atom]
    if atom.startswith("!") and atom[1:].strip() in ("do_load", "nofwd"):
        return not env[atom[1:].strip()]
    if atom == "t + 1 < t_end":
        return env["iter"] < env["trips"] - 1
    if atom == "t0 < t_end":
        return env["trips"] > 0
    if atom == "cp_on":
        return True  # thread-dependent: some threads copy
    return None


def eval_cond(header: str, env: dict):
    """True / False for conditions built from the kernel's uniform flags and the tile loop
    position; None when unknown (both branches explored)."""
    m = re.match(r"if \((.*)\)$", header)
    if not m:
        return None
    vals = [_eval_atom(a, env) for a in m.group(1).split("&&")]
    if any(v is False for v in vals):
        return False
    if all(v is True for v in vals):
        return True
    return None


def traces(node: Node, M: int, env: dict):
    """All event sequences through `node` under the uniform-flag assignment `env` (list of
    lists); the tile loop runs env['trips'] iterations."""
    seqs = [[]]
    items = node.items
    i = 0
    while i < len(items):
        it = items[i]
        if not isinstance(it, Node):
            ev = events(it, M)
            seqs = [s + ev for s in seqs]
            i += 1
            continue
        h = it.header or ""
        nxt = items[i + 1] if i + 1 < len(items) else None
        has_else = isinstance(nxt, Node) and nxt.header == "else"
        if h.startswith("for (int t = t0"):
            for k in range(env["trips"]):
                body = traces(it, M, dict(env, iter=k))
                seqs = [s + a for s in seqs for a in body]
        elif h.startswith("if") and (_has_events(it, M) or (has_else and _has_events(nxt, M))):
            c = eval_cond(h, env)
            taken = traces(it, M, env) if c is not False else []
            other = (traces(nxt, M, env) if has_else else [[]]) if c is not True else []
            seqs = [s + a for s in seqs for a in taken + other]
            if has_else:
                i += 1
        else:  # plain block, small loops, branches without buffer events: straight-line
            body = traces(it, M, env)
            seqs = [s + a for s in seqs for a in body]
        uniq = {tuple(s): s for s in seqs}  # identical traces are merged
        seqs = list(uniq.values())
        i += 1
    return seqs


def check_trace(trace):
    """First hazard of one event sequence, or None. Consecutive events of one kind on one buffer
    (the statements of one transpose put/get, the chunk copies of one prefetch) form one block
    access; two block accesses of one buffer that are not both reads need a barrier between
    them, and a buffer with cp.async writes in flight may not be touched until they are waited
    for and a barrier has made them visible."""
    last = {}  # region -> (kind, barrier epoch) of its last block access
    inflight = set()  # regions with cp.async writes not yet waited for
    waited = set()  # waited for, not yet made visible by a barrier
    epoch = 0
    prev_ev = None
    for pos, (kind, reg) in enumerate(trace):
        ev = (kind, reg)
        if kind == "BAR":
            epoch += 1
            for r in waited:
                last[r] = ("W", epoch - 1)
            waited = set()
            prev_ev = ev
            continue
        if kind == "WAIT":
            waited |= inflight
            inflight = set()
            prev_ev = ev
            continue
        if reg is None:
            return f"event {pos}: unknown buffer"
        continuing = prev_ev == ev
        prev_ev = ev
        if kind == "ASYNC":
            if reg in inflight:
                continue  # more chunk copies of the same prefetch
            if reg in waited:
                return f"event {pos}: prefetch into {reg} before the previous one is visible"
            p = last.get(reg)
            if p is not None and p[1] == epoch:
                return f"event {pos}: prefetch into {reg} after a {p[0]} with no barrier in between"
            inflight.add(reg)
            last.pop(reg, None)
            continue
        if reg in inflight or reg in waited:
            return f"event {pos}: {kind} on {reg} while a cp.async into it is not yet complete and visible"
        if continuing:
            continue
        p = last.get(reg)
        if p is not None and p[1] == epoch and not (p[0] == kind and kind in "RA"):
            return f"event {pos}: {kind} on {reg} after a {p[0]} with no barrier in between"
        last[reg] = (kind, epoch)
    if inflight:
        return "kernel ends with cp.async writes in flight"
    return None


def kernel_envs(body: str):
    """Uniform-flag assignments of one kernel: do_load / nofwd both ways unless the kernel
    declares them constant, and 1..3 tiles per CTA (the loop back edge twice)."""
    dl = [True] if "const bool do_load = true;" in body else [True, False]
    nf = [True, False] if "nofwd" in body else [False]
    return [dict(do_load=d, nofwd=f, trips=t, iter=0) for d in dl for f in nf for t in (1, 2, 3)]


def check_kernel_source(src: str, name: str, M: int):
    """Hazards over every path of one generated kernel (empty list = race-free); also returns
    the number of distinct paths checked."""
    body = src[src.index(name):]
    body = body[body.index("{") + 1:]
    root = parse_blocks(body)
    found, npaths = [], 0
    for env in kernel_envs(body):
        for tr in traces(root, M, env):
            npaths += 1
            h = check_trace(tr)
            if h:
                found.append(f"{h} (do_load={env['do_load']}, nofwd={env['nofwd']}, tiles={env['trips']})")
    return sorted(set(found)), npaths
