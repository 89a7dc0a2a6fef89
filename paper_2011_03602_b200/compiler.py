"""Per-app compiler: IR document -> host shared object + sm_100a cubin.

The paper recompiles the program for every candidate pattern (PGI OpenACC,
``PAPER.md:154``).  Here each program is compiled ONCE and every pattern of
the GA becomes a runtime configuration:

* every loop gets a CPU path (plain C, compiled with ``g++ -O3``, identical C
  semantics to the reference's ``c_openacc`` rendering, ``src/codegen.py``);
* every loop that can run on the GPU gets an sm_100a kernel plus a host launch
  stub; a loop becomes a GPU root when the pattern says so
  (``pattern.gpu_roots``, ``src/patterns.py:83-88``) and then takes its whole
  subtree along (``src/patterns.py:76-82``);
* every loop statement is a possible transfer site (a ``Placement`` always sits
  at its anchor loop's statement, ``src/transfers.py:160-163``), so the
  generated walk calls the runtime's hook before/after each loop whose site
  carries directives in the current plan.

Kernel shape (OpenACC ``kernels`` semantics): the maximal
perfectly nested chain of parallelisable loops under the root (the
reference's screen rules, ``src/screen.py:33-79``, restated in
:func:`parallelizable`) is collapsed into a 1-D grid with the innermost loop
fastest (coalesced along the contiguous index); the remaining loops run in
order inside each thread.  Scalars read by the nest travel by value in the
launch arguments; scalars written by the nest get lastprivate semantics (the
thread owning the sequentially-last iteration stores them in a device slab).
"""

from __future__ import annotations

import hashlib
import json
import os
import subprocess
import tempfile
import threading
from dataclasses import dataclass
from pathlib import Path

from . import appspec, reductions
from .ir import Program, expr_vars

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
CACHE = Path(os.environ.get("B2O_CACHE", PKG / "_cache"))
COMPILER_VERSION = "b2o-compiler-47"
ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
BLOCK_THREADS = 256
# plane-marching quad kernel: planes per thread and CTA size (NAS-MG resid
# 258^3: 67.6 -> 53.4 us; tools/kernel_sweep.py, profiles/r01/README.md)
MARCH_Z = 12  # planes per thread (NAS-MG resid 258^3, no prefetch: 8 -> 51.7 us, 16 -> 50.7 us; with the L2 prefetch 12 -> 41.9 us)
MARCH_BLOCK = 128
QUAD_NEXTPF = True     # quad kernels launched per host iteration prefetch the next launch's chunks (Himeno L 001001: 1.57 -> 1.28 s)
MARCH_SHFL = False     # plane-march: leading-plane +-1 chunks by warp shuffle (measured slower: 44.6 vs 39.0 us)
MARCH_CHAINS = True    # plane-march: carry plane-local subexpressions as scalars (NAS-MG resid: 96 -> 72 registers, 41.9 -> 38.7 us)
MARCH_FILL = True      # plane-march: carry chunks through unused middle planes (no reloads)
MARCH_L2PF = 2         # plane-march L2 prefetch distance in planes (0: off; NAS-MG 258: 50.6 -> 42.7 us)
MARCH_TMA_STAGES = 3   # shared-memory ring depth of the TMA-fed march (planes in flight: stages - 1)
MARCH_TMA_SPAN = 256   # largest chunk span of one CTA's quads staged (wider CTAs load directly)
MARCH_TMA_MIN_SPAN = 64  # below this (many streams), the register march kernel instead
STENCIL_TILE = (32, 8)      # (k, j) tile of the 2.5-D stencil kernels
BRICK_DEPTH = 4             # outer-loop points per thread in brick kernels

_lock = threading.Lock()


class CompileError(Exception):
    """The program (or one of its variants) cannot be built for B200."""


# ---------------------------------------------------------------------------
# typing helpers
# ---------------------------------------------------------------------------


def ctype(prog: Program, vid: int, precision: str) -> str:
    v = prog.vars[vid]
    if v.base_type == "int":
        return "int32_t"
    return "float" if precision == "fp32" else "double"


def etype(prog: Program, e, precision: str) -> str:
    """C type of an expression under the usual arithmetic conversions."""
    if e[0] == "num":
        return "double" if e[2] else "int32_t"
    if e[0] in ("var", "arr"):
        return ctype(prog, e[1], precision)
    a, b = etype(prog, e[2], precision), etype(prog, e[3], precision)
    for t in ("double", "float"):
        if t in (a, b):
            return t
    return "int32_t"


def render(e, name) -> str:
    """C text of an expression; ``name(vid, is_array)`` maps variables."""
    k = e[0]
    if k == "num":
        v = e[1]
        if e[2]:
            s = repr(float(v))
            return f"({s})" if float(v) < 0 else s
        return f"({int(v)})" if int(v) < 0 else str(int(v))
    if k == "var":
        return name(e[1], False)
    if k == "arr":
        return f"{name(e[1], True)}[{render(e[2], name)}]"
    return f"({render(e[2], name)} {e[1]} {render(e[3], name)})"


# ---------------------------------------------------------------------------
# nest analysis
# ---------------------------------------------------------------------------


def parallelizable(prog: Program, lid: int, extended: bool = False) -> bool:
    """The reference's screen (src/screen.py:33-79), restated on the IR
    document: no non-index scalar both read and set in the subtree, every array
    write indexed by this loop's index variable, no impure call.  With
    ``extended`` (the opt-in of reductions.py) carried scalars that are
    reductions or private temporaries are allowed."""
    loop = prog.loops[lid]
    if prog.doc["loops"][lid].get("directive_error", False):
        return False
    regions = set(prog.subtree_regions(lid))
    exempt = {prog.loops[x].index_var for x in prog.subtree_loops(lid)}
    if extended:
        cls = reductions.classify(prog, lid)
        if cls is None:
            return False
        exempt |= set(cls)
    reads, sets = set(), set()
    for o in prog.doc["occurrences"]:
        if o["region"] not in regions or prog.vars[o["var"]].is_array or o["var"] in exempt:
            continue
        if o["kind"] == "read":
            reads.add(o["var"])
        elif o["kind"] == "set":
            sets.add(o["var"])
    if reads & sets:
        return False
    for st in prog.walk(loop.body):
        if st.kind == "assign" and st.target[0] == "arr":
            if loop.index_var not in expr_vars(st.target[2]):
                return False
        if st.kind == "call" and not prog.calls[st.call].pure:
            return False
        if st.kind == "replaced":
            return False
    return True


@dataclass
class NestPlan:
    root: int
    kernel: str | None
    why_not: str | None
    chain: list[int]
    reads: list[int]        # vars whose value the nest needs (arrays: on device; scalars: by value)
    writes: list[int]       # vars the nest writes
    arrays: list[int]       # arrays referenced
    scalar_args: list[int]  # scalars passed by value
    swrites: list[int]      # scalars stored as lastprivate in the slab (incl. chain indices)
    locals_: list[int]      # scalars living in thread-local registers (non-chain)
    shape: str = "flat"     # flat | stencil
    ppt: int = 1            # points per thread (flat kernels, strided by the block)
    kb: int = 1             # consecutive innermost-index points per thread (flat kernels)
    staged: dict = None     # stencil kernels: var -> {ci, cj, dmin, planes}
    streams: dict = None    # stencil kernels: var -> {ci, base}: one affine read per point
    quad: dict = None       # quad kernels: quad_plan() result
    ktile: dict = None      # k-reduction tiled kernels: ktile_plan() result
    reds: dict = None       # reduction scalars of a chained nest: var -> "+" | "-" (reductions.py)
    exact: dict = None      # reductions summed exactly in loop order (b2o_xsum.cu): var -> slot


def affine(e, idx_vars):
    """(coefficients {var: c}, constant) when ``e`` is an integer affine form
    of ``idx_vars`` with literal coefficients, else None."""
    k = e[0]
    if k == "num":
        return None if e[2] else ({}, int(e[1]))
    if k == "var":
        return ({e[1]: 1}, 0) if e[1] in idx_vars else None
    if k != "bin":
        return None
    a, b = affine(e[2], idx_vars), affine(e[3], idx_vars)
    if a is None or b is None:
        return None
    op = e[1]
    if op in "+-":
        sg = 1 if op == "+" else -1
        co = dict(a[0])
        for v, c in b[0].items():
            co[v] = co.get(v, 0) + sg * c
        return ({v: c for v, c in co.items() if c}, a[1] + sg * b[1])
    if op == "*":
        if not a[0]:
            return ({v: c * a[1] for v, c in b[0].items() if c * a[1]}, a[1] * b[1])
        if not b[0]:
            return ({v: c * b[1] for v, c in a[0].items() if c * b[1]}, a[1] * b[1])
    return None


def stencil_offset(e, iv, ci, cj):
    """(di, dj, dk) of an index expression ``ci*i + cj*j + k + const`` with
    every component in [-1, 1], or None."""
    aff = affine(e, set(iv))
    if aff is None:
        return None
    co, const = aff
    if co != {iv[0]: ci, iv[1]: cj, iv[2]: 1}:
        return None
    hits = [(di, dj, dk) for di in (-1, 0, 1) for dj in (-1, 0, 1) for dk in (-1, 0, 1)
            if di * ci + dj * cj + dk == const]
    return hits[0] if len(hits) == 1 else None


def _array_refs(e, out):
    if e[0] == "arr":
        out.append(e)
        _array_refs(e[2], out)
    elif e[0] == "bin":
        _array_refs(e[2], out)
        _array_refs(e[3], out)


def _choose_shape(prog: Program, chain: list[int], writes: set[int], enable_stencil: bool = True):
    """Kernel shape for a chain: the 2.5-D stencil template when a read-only
    array is read at >= 4 distinct unit-radius offsets of a 3-deep affine
    nest; otherwise a flat kernel with 1-4 points per thread depending on the
    body's memory-reference count."""
    if not chain:
        return "flat", 1, None, None
    body = prog.regions[prog.loops[chain[-1]].body].statements
    if any(st.kind != "assign" for st in body):
        return "flat", 1, None, None
    refs: list = []
    for st in body:
        _array_refs(st.value, refs)
        if st.target[0] == "arr":
            refs.append(st.target)
            _array_refs(st.target[2], refs)
    staged = {}
    by_var: dict[int, list] = {}
    if len(chain) == 3:
        iv = [prog.loops[c].index_var for c in chain]
        for r in refs:
            by_var.setdefault(r[1], []).append(r)
        for v, rs in by_var.items():
            if v in writes:
                continue
            aff = affine(rs[0][2], set(iv))
            if aff is None:
                continue
            co = aff[0]
            ci, cj = co.get(iv[0], 0), co.get(iv[1], 0)
            if co.get(iv[2]) != 1 or cj < 3 or ci < 3 * cj:
                continue
            offs = [stencil_offset(r[2], iv, ci, cj) for r in rs]
            if any(o is None for o in offs) or len(set(offs)) < 4:
                continue
            dis = [o[0] for o in offs]
            staged[v] = {"ci": ci, "cj": cj, "dmin": min(dis), "planes": max(dis) - min(dis) + 1}
    if staged and enable_stencil == "brick":
        return "brick", 1, staged, None
    if staged and enable_stencil:
        streams = {}
        for v, rs in by_var.items():
            if v in writes or v in staged:
                continue
            idx = {json.dumps(r[2]) for r in rs}
            aff = affine(rs[0][2], set(iv))
            if len(idx) != 1 or aff is None or aff[0].get(iv[2]) != 1 or set(aff[0]) - set(iv):
                continue
            co, const = aff
            base = f"(int64_t){co.get(iv[1], 0)} * v{iv[1]} + v{iv[2]} + ({const})"
            streams[v] = {"ci": co.get(iv[0], 0), "base": base}
        return "stencil", 1, staged, streams
    # points per thread (strided by the block: coalescing kept) amortise the
    # per-thread prologue; keep refs x points within a ~96-value register
    # budget (measured: NAS-MG resid 23 refs best at 4, Himeno Jacobi 34 refs
    # at 2, tools/kernel_sweep.py)
    n = len({(r[1], json.dumps(r[2])) for r in refs})  # distinct memory references
    return "flat", max(1, min(4, 96 // max(n, 1))), None, None


QUAD = 4  # points per thread of the vectorised flat kernel (16-byte chunks of 4-byte elements)


def quad_plan(prog: Program, chain: list[int], precision: str) -> dict | None:
    """Vectorised ("quad") flat kernel eligibility (SURVEY.md §7 "Alignment":
    odd row pitches forbid aligned 3-D tiles, so process the flattened index
    space in aligned 16-byte chunks plus neighbour offsets).

    Eligible when the chain body is straight-line array assignments whose
    every array reference is ``sum_d c_d * i_d + k + const`` with literal
    coefficients, coefficient 1 on the innermost chain index ``k``, the same
    outer coefficients ``c_d`` for every reference (one row function
    ``F = sum c_d i_d``), 4-byte elements, and no array both read and written
    in the body (each written at a single offset).  A thread then owns one
    16-byte-aligned quad of a row (an array both read and written is allowed
    when every reference uses the write's offset): every reference ``const`` maps lane ``u``
    to element ``b + const + u`` of an aligned chunk known at compile time.
    Returns ``{"outer": (c_d...), "reads": {(v, const)}, "writes": {v: const}}``
    or None."""
    if not chain:
        return None
    body = prog.regions[prog.loops[chain[-1]].body].statements
    if not body or any(st.kind != "assign" or st.target[0] != "arr" for st in body):
        return None
    iv = [prog.loops[c].index_var for c in chain]
    # int scalars the body reads (by value, never written in a straight-line
    # array body) may appear in index expressions as well: they are part of
    # the row function, e.g. i and j of a k-rooted Himeno nest
    extra = set()
    for st in body:
        extra |= {v for v in expr_vars(st.value) + expr_vars(st.target[2])
                  if not prog.vars[v].is_array and prog.vars[v].base_type == "int" and v not in iv}
    ovars = iv[:-1] + sorted(extra)
    ivs = set(iv) | extra
    outer = None
    reads, writes = set(), {}

    def ref(r):
        nonlocal outer
        if ctype(prog, r[1], precision) not in ("float", "int32_t"):
            return None
        aff = affine(r[2], ivs)
        if aff is None or aff[0].get(iv[-1]) != 1:
            return None
        o = tuple(aff[0].get(v, 0) for v in ovars)
        if outer is None:
            outer = o
        elif o != outer:
            return None
        return aff[1]

    for st in body:
        refs: list = []
        _array_refs(st.value, refs)
        _array_refs(st.target[2], refs)
        for r in refs:
            c = ref(r)
            if c is None:
                return None
            reads.add((r[1], c))
        c = ref(st.target)
        if c is None or writes.get(st.target[1], c) != c:
            return None
        writes[st.target[1]] = c
    # an array both read and written must be touched at one offset only
    # (point-local read-modify-write); reads after the write in body order
    # then see the new lane value (quad_kernel_fn)
    if any(v in writes and c != writes[v] for v, c in reads):
        return None
    return {"outer": outer, "ovars": ovars, "ivs": sorted(ivs), "reads": reads, "writes": writes}


def march_plan(prog: Program, chain: list[int], qp: dict, Z: int) -> dict | None:
    """Plane-marching eligibility for a quad nest: at least two chain loops,
    the outermost chain index enters every reference with one coefficient
    ``C0`` that is a multiple of the quad (so a quad keeps its lanes from
    plane to plane), and every reference constant splits uniquely into
    ``d * C0 + rest`` with ``|rest| < C0 / 2 - QUAD``.  Returns
    ``{"Z", "C0", "keys": {(array, d, chunk)}, "split"}`` or None."""
    if len(chain) < 2 or Z < 2:
        return None
    iv0 = prog.loops[chain[0]].index_var
    if not qp["ovars"] or qp["ovars"][0] != iv0:
        return None
    C0 = qp["outer"][0]
    if C0 <= 0 or C0 % QUAD:
        return None

    def split(c):
        d = (c + C0 // 2) // C0
        return d, c - d * C0

    keys = set()
    for v, c in qp["reads"]:
        d, rest = split(c)
        if abs(rest) >= C0 // 2 - QUAD:
            return None
        if v in qp["writes"] and d != 0:
            return None
        for u in range(QUAD):
            keys.add((v, d, (rest + u) // QUAD))
    for v, c in qp["writes"].items():
        d, rest = split(c)
        if d != 0 or abs(rest) >= C0 // 2 - QUAD:
            return None
    if not any((v, d + 1, o) in keys and v not in qp["writes"] for v, d, o in keys):
        return None  # nothing to carry from plane to plane: the plain quad kernel wins
    return {"Z": Z, "C0": C0, "keys": keys, "split": split}


KT_TI = KT_TJ = 64   # k-reduction tiles: points per CTA along the two chain loops
KT_BK = 32           # k per shared-memory stage
KT_R = 4             # register micro-tile: KT_R x KT_R points per thread (256 threads)


def ktile_plan(prog: Program, chain: list[int], precision: str) -> dict | None:
    """Register-tiled k-reduction eligibility (the naive matmul nest and its
    relatives): two parallel chain loops (i, j) whose body is straight-line
    array assignments around exactly one sequential loop k, where

    * every array written in the body is indexed by one affine form of
      (i, j) only (a per-point accumulator, held in a register), and read
      only at that index;
    * inside the k loop every other array reference is affine in (i, k)
      only ("A" operands) or (k, j) only ("B" operands) and the array is not
      written by the nest: these are staged through shared memory tiles;
    * the k loop's bounds use literals and read-only scalars only.

    Each point still executes its statements in the original order (k
    ascending, same C expression per statement), so results are
    bit-identical to the sequential loop.  Returns the plan or None."""
    if len(chain) != 2 or precision != "fp32":
        return None
    iv, jv = (prog.loops[c].index_var for c in chain)
    body = prog.regions[prog.loops[chain[1]].body].statements
    if any(st.kind not in ("assign", "loop") for st in body):
        return None
    kls = [x for x, st in enumerate(body) if st.kind == "loop"]
    if len(kls) != 1:
        return None
    K = prog.loops[body[kls[0]].loop]
    kv = K.index_var
    kbody = prog.regions[K.body].statements
    if not kbody or any(st.kind != "assign" for st in kbody):
        return None
    for b in (K.lower, K.upper):
        if any(prog.vars[v].is_array or v in (iv, jv, kv) for v in expr_vars(b)):
            return None
    outer = body[:kls[0]] + body[kls[0] + 1:]
    accs: dict = {}
    for st in outer + kbody:
        t = st.target
        if t[0] != "arr" or ctype(prog, t[1], precision) != "float":
            return None
        aff = affine(t[2], {iv, jv})
        if aff is None:
            return None
        key = (tuple(sorted(aff[0].items())), aff[1])
        if accs.setdefault(t[1], key) != key:
            return None
    direct, tiles = set(), {}
    for inner, sts in ((False, outer), (True, kbody)):
        for st in sts:
            refs: list = []
            _array_refs(st.value, refs)
            _array_refs(st.target[2], refs)
            for r in refs:
                v = r[1]
                if v in accs:
                    aff = affine(r[2], {iv, jv})
                    if aff is None or (tuple(sorted(aff[0].items())), aff[1]) != accs[v]:
                        return None
                    continue
                if ctype(prog, v, precision) != "float":
                    return None
                if not inner:
                    if affine(r[2], {iv, jv}) is None:
                        return None
                    direct.add(v)
                    continue
                aff = affine(r[2], {iv, jv, kv})
                if aff is None:
                    return None
                co = aff[0]
                if co.get(jv, 0) == 0:
                    side = "A"
                elif co.get(iv, 0) == 0:
                    side = "B"
                else:
                    return None
                key = (v, tuple(sorted(co.items())), aff[1])
                tiles.setdefault(key, (side, len(tiles)))
    if not tiles:
        return None
    return {"iv": iv, "jv": jv, "kv": kv, "kloop": K.id, "kpos": kls[0], "accs": accs, "tiles": tiles,
            "direct": direct}


def _first_access_is_read(prog: Program, lid: int, vid: int) -> bool:
    """Walk the nest in execution order of one thread's first iteration; True
    when ``vid`` may be read before any write (conservative)."""
    def loop_first(l):
        lo = prog.loops[l]
        if vid in expr_vars(lo.lower):
            return True
        if lo.index_var == vid:
            return False
        if vid in expr_vars(lo.upper):
            return True
        return region_first(lo.body)

    def region_first(rid):
        for st in prog.regions[rid].statements:
            if st.kind == "loop":
                r = loop_first(st.loop)
            elif st.kind == "call":
                r = region_first(prog.calls[st.call].subtree) if not prog.is_opaque_call(st.call) else None
            else:
                reads, writes = prog.stmt_access(st)
                if vid in reads:
                    return True
                r = False if vid in writes else None
            if r is not None:
                return r
        return None

    return bool(loop_first(lid))


def plan_nest(prog: Program, lid: int, enable_stencil: bool = False, extended: bool = False) -> NestPlan:
    loop = prog.loops[lid]
    nest_loops = prog.subtree_loops(lid)
    reads, writes = prog.subtree_access(lid)
    why = None
    for st in prog.walk(loop.body):
        if st.kind == "replaced":
            why = "subtree holds a replaced function block"
        elif st.kind == "call" and prog.is_opaque_call(st.call):
            why = f"subtree calls opaque {prog.calls[st.call].name!r}"
    seen_idx = []
    for x in nest_loops:
        chain_up = [prog.loops[a].index_var for a in prog.ancestors(x) if a in nest_loops]
        if prog.loops[x].index_var in chain_up:
            why = why or "nested loops share an index variable"
        seen_idx.append(prog.loops[x].index_var)
    if why is not None:
        return NestPlan(lid, None, why, [], [], [], [], [], [], [])
    # assignments inside the nest (not loop headers)
    body_writes = set()
    for st in prog.walk(loop.body):
        if st.kind in ("assign", "decl"):
            body_writes |= prog.stmt_access(st)[1]
    chain: list[int] = []
    if parallelizable(prog, lid, extended) and not (set(expr_vars(loop.lower)) | set(expr_vars(loop.upper))) & writes \
            and loop.index_var not in body_writes:
        chain = [lid]
        while True:
            body = prog.regions[prog.loops[chain[-1]].body].statements
            if len(body) != 1 or body[0].kind != "loop":
                break
            c = body[0].loop
            cl = prog.loops[c]
            bound_vars = set(expr_vars(cl.lower)) | set(expr_vars(cl.upper))
            chain_idx = {prog.loops[x].index_var for x in chain}
            if (not parallelizable(prog, c, extended) or bound_vars & (writes | chain_idx)
                    or cl.index_var in chain_idx or cl.index_var in body_writes):
                break
            chain.append(c)
    # chain bounds are evaluated on the host at launch: no arrays there
    while chain and any(prog.vars[v].is_array for c in chain
                        for v in expr_vars(prog.loops[c].lower) + expr_vars(prog.loops[c].upper)):
        chain.pop()
    chain_idx = [prog.loops[x].index_var for x in chain]
    bound_scalars = {v for c in chain for v in expr_vars(prog.loops[c].lower) + expr_vars(prog.loops[c].upper)}
    scalars = sorted(v for v in (reads | writes) if not prog.vars[v].is_array)
    arrays = sorted(v for v in (reads | writes) if prog.vars[v].is_array)
    locals_ = [v for v in scalars if v not in chain_idx]
    scalar_args = [v for v in locals_ if v not in writes or _first_access_is_read(prog, lid, v)]
    # roots evaluate chain bounds on the host: those reads are host-side
    need = set(scalar_args) | {a for a in arrays if a in reads} | bound_scalars
    swrites = sorted(set(chain_idx) | {v for v in locals_ if v in writes})
    reds = {}
    if chain and extended:
        cls = reductions.classify(prog, chain[0]) or {}
        reds = {v: c.split(":")[1] for v, c in cls.items() if c.startswith("reduction")}
        if len(reds) > 8:  # B2O_RED_MAX_VARS
            chain, reds = [], {}
    shape, ppt, staged, streams = _choose_shape(prog, chain, writes, enable_stencil and not reds)
    return NestPlan(lid, f"b2o_k{lid}", None, chain, sorted(need), sorted(writes), arrays,
                    scalar_args, swrites, locals_, shape=shape, ppt=ppt, staged=staged, streams=streams,
                    reds=reds or None)


# ---------------------------------------------------------------------------
# code generation
# ---------------------------------------------------------------------------


class _Gen:
    def __init__(self, prog: Program, spec: dict):
        self.prog = prog
        self.spec = spec
        self.precision = spec.get("precision", "fp32")
        self.sets: list[tuple[tuple[int, ...], tuple[int, ...]]] = []
        self.set_ids: dict = {}
        self.blocks: list[dict] = []
        self.block_ids: dict[int, int] = {}
        self.calls: dict[int, dict] = {}
        self.nests = {l.id: plan_nest(prog, l.id, spec.get("stencil", False), bool(spec.get("reductions")))
                      for l in prog.loops}
        self.exact_slots = 0
        for nst in self.nests.values():
            ex = self.exact_reductions(nst)
            if ex:
                nst.exact = ex
                nst.ppt = 1
                self.exact_slots = max(self.exact_slots, len(ex))
        for nst in self.nests.values():
            if nst.shape == "flat" and nst.chain and nst.ppt == 1 and not nst.exact and all(
                    st.kind == "assign" for st in prog.regions[prog.loops[nst.chain[-1]].body].statements):
                nst.kb = int(spec.get("flat_kblock", 1))
        if spec.get("flat_ppt"):
            for nst in self.nests.values():
                if nst.shape == "flat" and nst.chain and not nst.exact and all(
                        st.kind == "assign" for st in prog.regions[prog.loops[nst.chain[-1]].body].statements):
                    nst.ppt = int(spec["flat_ppt"])
        if int(spec.get("flat_vec", QUAD)) == QUAD and not spec.get("flat_ppt") \
                and int(spec.get("flat_kblock", 1)) == 1:
            for nst in self.nests.values():
                if nst.shape == "flat" and nst.chain:
                    qp = quad_plan(prog, nst.chain, self.precision)
                    if qp is not None:
                        qp["groups"] = int(spec.get("quad_groups", 1))
                        if qp["groups"] == 1 and not spec.get("quad_shfl"):
                            qp["march"] = march_plan(prog, nst.chain, qp, int(spec.get("quad_march", MARCH_Z)))
                        nst.shape, nst.quad, nst.ppt = "quad", qp, 1
        if spec.get("ktile", True):
            for nst in self.nests.values():
                if nst.shape == "flat" and len(nst.chain) == 2 and not nst.reds:
                    kp = ktile_plan(prog, nst.chain, self.precision)
                    if kp is not None:
                        nst.shape, nst.ktile, nst.ppt = "ktile", kp, 1
        self.device_op = {}
        for l in prog.loops:
            self.device_op[l.id] = any(st.kind == "replaced" for st in prog.walk(l.body))
        for st in prog.stmts:
            if st.kind == "replaced":
                try:
                    b = appspec.block_binding(prog, spec, st)
                except ValueError as exc:
                    raise CompileError(str(exc)) from exc
                self.block_ids[st.uid] = len(self.blocks)
                self.blocks.append(b)
            elif st.kind == "call" and prog.is_opaque_call(st.call):
                c = prog.calls[st.call]
                try:
                    b = appspec.external_call_binding(prog, spec, c)
                except ValueError as exc:
                    raise CompileError(str(exc)) from exc
                for v in [b["out"]] + b["ins"]:
                    if not prog.vars[v].is_array:
                        raise CompileError(f"external {c.name!r} takes scalar argument {prog.vars[v].name!r}")
                self.calls[c.id] = b
        self.ext_writes = {cid: {b["out"]} for cid, b in self.calls.items()}

    def exact_reductions(self, n: NestPlan) -> dict:
        """Reductions of a chained nest that can be summed EXACTLY in loop
        order on the GPU (b2o_exact_sum_f32 / _f64, csrc/b2o_xsum.cu): an fp32
        or fp64 scalar whose every update in the nest is ``s = s + e`` /
        ``s = e + s`` / ``s = s - e`` with ``e`` of the scalar's own C type
        (one correctly rounded addition each), and
        which every point of the chain updates a compile-time constant
        number of times C (the loops run in-thread below the chain have
        literal bounds).  Point t's j-th update stores its term at
        ``t * C + j``: the buffer holds the terms in sequential loop order and
        the runtime reproduces the sequential sum bit for bit.  spec
        ``exact_reductions: false`` keeps the reassociating tree (faster,
        documented tolerance).  Returns ``{var: (slot, C)}``."""
        if not n.reds or not n.chain or self.spec.get("exact_reductions") is False:
            return {}
        prog = self.prog

        def count(rid, v):
            total = 0
            for st in prog.regions[rid].statements:
                if st.kind == "assign" and st.target[0] == "var" and st.target[1] == v:
                    red = reductions.reduction_stmt(st)
                    # one addition in the scalar's own format (an fp32 sum with
                    # a double term would round twice)
                    if red is None or etype(prog, red[2], self.precision) != self.T(v):
                        return None
                    total += 1
                elif st.kind == "loop":
                    lp = prog.loops[st.loop]
                    if lp.lower[0] != "num" or lp.upper[0] != "num" or lp.lower[2] or lp.upper[2]:
                        if any(x.kind == "assign" and x.target[0] == "var" and x.target[1] == v
                               for x in prog.walk(lp.body)):
                            return None
                        continue
                    c = count(lp.body, v)
                    if c is None:
                        return None
                    total += c * max(0, int(lp.upper[1]) - int(lp.lower[1]))
                elif st.kind == "call" and not prog.is_opaque_call(st.call):
                    c = count(prog.calls[st.call].subtree, v)  # inlined body (dev_region recurses too)
                    if c is None:
                        return None
                    total += c
            return total

        out = {}
        for v in sorted(n.reds):
            if self.T(v) not in ("float", "double"):
                continue
            c = count(prog.loops[n.chain[-1]].body, v)
            if not c:
                continue
            out[v] = (len(out), c)
        return out

    def exact_elems(self) -> int:
        """Largest iteration space of a nest with exact reductions when its
        chain bounds are literals (the runtime sizes the term buffers at
        replica setup, outside every timed run); 0: size on first use."""
        best = 0
        for n in self.nests.values():
            if not n.exact:
                continue
            tot = 1
            for c in n.chain:
                lo, hi = self.prog.loops[c].lower, self.prog.loops[c].upper
                if lo[0] != "num" or hi[0] != "num":
                    tot = 0
                    break
                tot *= max(0, int(hi[1]) - int(lo[1]))
            best = max(best, tot * max(c for _, c in n.exact.values()))
        return best

    # -- helpers -----------------------------------------------------------

    def T(self, vid: int) -> str:
        return ctype(self.prog, vid, self.precision)

    def access_set(self, need, writes) -> int:
        """Host footprint of a statement / fast loop / loop header: ``need``
        must be valid on the host before it runs, ``writes`` are host-dirty
        after it."""
        key = (tuple(sorted(need)), tuple(sorted(writes)))
        if key not in self.set_ids:
            self.set_ids[key] = len(self.sets)
            self.sets.append(key)
        return self.set_ids[key]

    def extra_writes(self, st):
        if st.kind == "call" and st.call in self.ext_writes:
            return self.ext_writes[st.call]
        return set()

    def subtree_access(self, lid):
        return self.prog.subtree_access(lid, self.extra_writes)

    def fast_footprint(self, lid):
        """(need, writes) of running loop ``lid`` on the CPU: every array it
        touches, scalars only when their first access may be a read."""
        reads, writes = self.subtree_access(lid)
        need = set()
        for v in reads | writes:
            if self.prog.vars[v].is_array or _first_access_is_read(self.prog, lid, v):
                need.add(v)
        return need, writes

    def progressive(self, lid: int) -> dict:
        """Arrays a CPU fast loop may start reading before their download has
        finished: read-only in the loop, every reference affine in the loop
        indices with one non-negative coefficient ``C`` on the outermost
        index ``x`` and literal bounds on every inner loop.  Iteration ``x``
        then touches elements below ``C * x + K + 1`` only, so the generated
        loop waits for that prefix of the (chunked, asynchronous) D2H copy
        before each outer iteration.  Returns ``{array: (C, K)}``."""
        if self.spec.get("progressive_d2h") is False:
            return {}
        prog = self.prog
        if any(st.kind in ("call", "replaced") for st in prog.walk(prog.loops[lid].body)):
            return {}
        reads, writes = self.subtree_access(lid)
        x = prog.loops[lid].index_var
        rng = {}
        for l in prog.subtree_loops(lid):
            if l == lid:
                continue
            lo, hi = prog.loops[l].lower, prog.loops[l].upper
            if lo[0] != "num" or hi[0] != "num" or lo[2] or hi[2]:
                return {}
            rng[prog.loops[l].index_var] = (int(lo[1]), int(hi[1]))
        lvars = set(rng) | {x}
        refs: dict = {}
        for st in prog.walk(prog.loops[lid].body):
            if st.kind == "assign":
                rs: list = []
                _array_refs(st.value, rs)
                _array_refs(st.target[2], rs) if st.target[0] == "arr" else None
                if st.target[0] == "arr":
                    rs.append(st.target)
                for r in rs:
                    refs.setdefault(r[1], []).append(r[2])
            elif st.kind == "decl" and st.init is not None:
                rs = []
                _array_refs(st.init, rs)
                for r in rs:
                    refs.setdefault(r[1], []).append(r[2])
        # the generated for-header evaluates the outer bounds before the first
        # host_wait (and the upper bound every iteration): an array read there
        # must be complete before the loop starts
        in_header: list = []
        _array_refs(prog.loops[lid].lower, in_header)
        _array_refs(prog.loops[lid].upper, in_header)
        header_arrays = {r[1] for r in in_header}
        out = {}
        for v, idxs in refs.items():
            if v in writes or not prog.vars[v].is_array or v in header_arrays:
                continue
            C, K = None, None
            for e in idxs:
                aff = affine(e, lvars)
                if aff is None:
                    break
                c = aff[0].get(x, 0)
                if c < 0 or (C is not None and c != C):
                    break
                C = c
                k = aff[1] + sum(max(cv * rng[u][0], cv * rng[u][1]) for u, cv in aff[0].items() if u != x)
                K = k if K is None else max(K, k)
            else:
                if C:  # C == 0: the first outer iteration needs the whole array anyway
                    out[v] = (C, K)
        return out

    @staticmethod
    def host_name(vid: int, is_array: bool) -> str:
        return f"A{vid}" if is_array else f"S{vid}"

    @staticmethod
    def local_name(vid: int, is_array: bool) -> str:
        return f"v{vid}"

    def bound(self, e, name) -> str:
        t = etype(self.prog, e, self.precision)
        txt = render(e, name)
        if t == "int32_t":
            return f"(int32_t)({txt})"
        return f"(int32_t)ceil((double)({txt}))"

    # -- CPU fast path -----------------------------------------------------------

    def fast_fn(self, lid: int) -> list[str]:
        prog = self.prog
        reads, writes = self.subtree_access(lid)
        used = sorted(reads | writes)
        out = [f"static void fast_L{lid}(b2o_exec *ex) {{"]
        for v in used:
            t = self.T(v)
            if prog.vars[v].is_array:
                out.append(f"  {t} *__restrict__ v{v} = ({t} *)ex->host[{v}];")
            else:
                out.append(f"  {t} v{v} = *({t} *)ex->host[{v}];")
        body: list[str] = []
        self.fast_loop(lid, 1, body, outer=True, waits=self.progressive(lid))
        out.extend(body)
        out.append(f" out_L{lid}:")
        for v in used:
            if not prog.vars[v].is_array and v in writes:
                out.append(f"  *({self.T(v)} *)ex->host[{v}] = v{v};")
        for v in used:
            if not prog.vars[v].is_array and v not in writes:
                out.append(f"  (void)v{v};")
        out.append("}")
        return out

    def fast_loop(self, lid: int, ind: int, out: list[str], outer: bool = False, label: int | None = None,
                  waits: dict | None = None) -> None:
        prog = self.prog
        loop = prog.loops[lid]
        label = lid if label is None else label
        iv = f"v{loop.index_var}"
        out.append("  " * ind + f"for ({iv} = {render(loop.lower, self.local_name)}; {iv} < "
                   f"{render(loop.upper, self.local_name)}; {iv}++) {{")
        if prog.children(lid):
            out.append("  " * (ind + 1) + f"if (__builtin_expect(ex->stop, 0)) goto out_L{label};")
        for v, (C, K) in sorted((waits or {}).items()):
            out.append("  " * (ind + 1) + f"ex->host_wait(ex, {v}, (int64_t){C} * {iv} + {K + 1});")
        self.fast_region(loop.body, ind + 1, out, label)
        out.append("  " * ind + "}")

    def fast_region(self, rid: int, ind: int, out: list[str], label: int) -> None:
        prog = self.prog
        for st in prog.regions[rid].statements:
            pad = "  " * ind
            if st.kind == "decl":
                if st.init is not None:
                    out.append(pad + f"v{st.var} = {render(st.init, self.local_name)};")
            elif st.kind == "assign":
                out.append(pad + f"{render(st.target, self.local_name)} = {render(st.value, self.local_name)};")
            elif st.kind == "loop":
                self.fast_loop(st.loop, ind, out, label=label)
            elif st.kind == "call":
                if prog.is_opaque_call(st.call):
                    out.append(pad + f"ex->external(ex, {st.call});")
                    out.append(pad + f"if (ex->stop) goto out_L{label};")
                else:
                    self.fast_region(prog.calls[st.call].subtree, ind, out, label)
            else:  # replaced blocks never reach the fast path
                raise AssertionError("replaced block in a CPU fast path")

    # -- instrumented walk ------------------------------------------------------

    def instr_region(self, rid: int, ind: int, out: list[str]) -> None:
        prog = self.prog
        for st in prog.regions[rid].statements:
            pad = "  " * ind
            if st.kind in ("decl", "assign"):
                reads, writes = prog.stmt_access(st)
                if st.kind == "decl" and st.init is None:
                    continue
                need = reads | {v for v in writes if prog.vars[v].is_array}
                sid = self.access_set(need, writes)
                out.append(pad + f"ex->host_access(ex, {sid}); if (ex->stop) return;")
                if st.kind == "decl":
                    out.append(pad + f"S{st.var} = {render(st.init, self.host_name)};")
                else:
                    out.append(pad + f"{render(st.target, self.host_name)} = {render(st.value, self.host_name)};")
            elif st.kind == "loop":
                self.instr_loop(st.loop, ind, out)
            elif st.kind == "call":
                if prog.is_opaque_call(st.call):
                    out.append(pad + f"ex->external(ex, {st.call}); if (ex->stop) return;")
                else:
                    self.instr_region(prog.calls[st.call].subtree, ind, out)
            else:
                out.append(pad + f"ex->block(ex, {self.block_ids[st.uid]}); if (ex->stop) return;")

    def instr_loop(self, lid: int, ind: int, out: list[str]) -> None:
        prog = self.prog
        loop = prog.loops[lid]
        pad = "  " * ind
        out.append(pad + f"if (ex->hook_mask[{lid}] & 1) {{ ex->hook(ex, {lid}, 0); if (ex->stop) return; }}")
        branches = []
        if self.nests[lid].kernel:
            branches.append((f"ex->is_root[{lid}]", [f"launch_L{lid}(ex); if (ex->stop) return;"]))
        if not self.device_op[lid]:
            sid = self.access_set(*self.fast_footprint(lid))
            prog_vars = self.progressive(lid)
            if prog_vars:
                # these arrays may still be arriving: fast_L waits per outer iteration
                psid = self.access_set(set(prog_vars), set())
                acc = f"ex->host_access_fast(ex, {sid}, {psid}); if (ex->stop) return;"
            else:
                acc = f"ex->host_access(ex, {sid}); if (ex->stop) return;"
            branches.append((f"!ex->dev_inside[{lid}]", [acc, f"fast_L{lid}(ex); if (ex->stop) return;"]))
        hneed = set(expr_vars(loop.lower)) | (set(expr_vars(loop.upper)) - {loop.index_var})
        hsid = self.access_set(hneed, {loop.index_var})
        iv = f"S{loop.index_var}"
        inner = [f"ex->host_access(ex, {hsid}); if (ex->stop) return;",
                 f"for ({iv} = {render(loop.lower, self.host_name)}; {iv} < {render(loop.upper, self.host_name)}; "
                 f"{iv}++) {{"]
        body: list[str] = []
        self.instr_region(loop.body, 1, body)
        inner.extend(body)
        inner.append("}")
        first = True
        for cond, lines in branches:
            out.append(pad + ("if (" if first else "} else if (") + cond + ") {")
            out.extend(pad + "  " + ln for ln in lines)
            first = False
        if branches:
            out.append(pad + "} else {")
            out.extend(pad + "  " + ln for ln in inner)
            out.append(pad + "}")
        else:
            out.extend(pad + ln for ln in inner)
        out.append(pad + f"if (ex->hook_mask[{lid}] & 2) {{ ex->hook(ex, {lid}, 1); if (ex->stop) return; }}")

    # -- kernels -------------------------------------------------------------------

    def next_pf(self, n: NestPlan):
        """(host loop, element stride) when a plain quad kernel is launched
        once per iteration of an enclosing host loop whose index enters its
        addresses (k-rooted Himeno: one launch per (i, j), stride = the row
        pitch): the kernel then prefetches into L2 what the NEXT launch will
        read -- its own chunks shifted by one host iteration -- so that launch
        finds its rows in L2 instead of paying DRAM latency (spec
        ``quad_nextpf``).  The launch stub passes whether that iteration
        exists, so every prefetched address is one the program reads."""
        if n.shape != "quad" or n.quad.get("march") or not self.spec.get("quad_nextpf", QUAD_NEXTPF):
            return None
        par = self.prog.loops[n.root].parent
        if par is None:
            return None
        pv = self.prog.loops[par].index_var
        qp = n.quad
        if pv not in qp["ovars"]:
            return None
        c = qp["outer"][qp["ovars"].index(pv)]
        return (par, c) if c else None

    def kernel_struct(self, n: NestPlan) -> list[str]:
        D = max(len(n.chain), 1)
        out = [f"typedef struct {{", "  uint32_t total, chunk;",
               f"  uint32_t n[{D}], tn[{D}], mul[{D}], shr[{D}];", f"  int32_t lo[{D}];", "  void *slab;",
               "  void *scratch;"]
        for v in n.arrays:
            const = "const " if v not in n.writes else ""
            out.append(f"  {const}{self.T(v)} *p{v};")
        for v in n.scalar_args:
            out.append(f"  {self.T(v)} s{v};")
        for v in (n.exact or {}):
            out.append(f"  {self.T(v)} *xb{v};  // per-point terms of reduction {self.prog.vars[v].name}, loop order")
        if self.next_pf(n):
            out.append("  int32_t pfn;  // the enclosing host loop has a next iteration")
        out.append(f"}} KA_L{n.root};")
        return out

    def launch_fn(self, n: NestPlan) -> list[str]:
        prog = self.prog
        lid = n.root
        out = [f"static void launch_L{lid}(b2o_exec *ex) {{", f"  ex->pre_launch(ex, {lid}); if (ex->stop) return;",
               f"  KA_L{lid} a; memset(&a, 0, sizeof a);", "  uint64_t total = 1;", "  uint32_t geom[6];"]
        for d, c in enumerate(n.chain):
            cl = prog.loops[c]
            out.append(f"  {{ int32_t lo = {self.bound(cl.lower, self.host_name)}; "
                       f"int32_t hi = {self.bound(cl.upper, self.host_name)};")
            out.append(f"    a.lo[{d}] = lo; a.n[{d}] = hi > lo ? (uint32_t)((int64_t)hi - lo) : 0u; "
                       f"total *= a.n[{d}]; }}")
        if n.chain:
            out.append("  if (total == 0) {")
            sid = self.access_set(*self.fast_footprint(lid))
            out.append(f"    ex->host_access(ex, {sid}); if (ex->stop) return;")
            out.append(f"    fast_L{lid}(ex); return;")
            out.append("  }")
            D = len(n.chain)
            out.append(f"  for (int d = 0; d < {D}; ++d) a.tn[d] = a.n[d];")
            if n.shape == "quad":
                # quads per row: the row's first element may sit anywhere in
                # its aligned chunk, so one extra (possibly empty) quad
                L = QUAD * n.quad["groups"]
                out.append(f"  a.tn[{D - 1}] = (a.n[{D - 1}] + {QUAD - 1 + L - 1}) / {L};")
                if n.quad.get("march"):
                    Z = n.quad["march"]["Z"]
                    out.append(f"  a.tn[0] = (a.n[0] + {Z - 1}) / {Z};")
                out.append("  total = 1;")
                out.append(f"  for (int d = 0; d < {D}; ++d) total *= a.tn[d];")
            if n.kb > 1:
                out.append(f"  a.tn[{D - 1}] = (a.n[{D - 1}] + {n.kb - 1}) / {n.kb};")
                out.append("  total = 1;")
                out.append(f"  for (int d = 0; d < {D}; ++d) total *= a.tn[d];")
            out.append("  if (total > 0xFFFFFFFFull) { ex->launch(ex, %d, 0, 0, 0); return; }" % lid)
            for d in range(1, len(n.chain)):
                out.append(f"  b2o_fastdiv_init(a.tn[{d}], &a.mul[{d}], &a.shr[{d}]);")
        out.append("  a.total = (uint32_t)total; a.slab = ex->slab; a.scratch = ex->scratch;")
        npf = self.next_pf(n)
        if npf:
            par = prog.loops[npf[0]]
            out.append(f"  a.pfn = ({self.host_name(par.index_var, False)} + 1 < "
                       f"{self.bound(par.upper, self.host_name)}) ? 1 : 0;")
        for v in n.arrays:
            const = "const " if v not in n.writes else ""
            out.append(f"  a.p{v} = ({const}{self.T(v)} *)ex->dev[{v}];")
        for v in n.scalar_args:
            out.append(f"  a.s{v} = S{v};")
        if n.shape == "ktile":
            T = int(self.spec.get("ktile_tile", KT_TI))
            R = int(self.spec.get("ktile_r", KT_R))
            RI = int(self.spec.get("ktile_ri", R))
            out.append(f"  geom[0] = (a.n[1] + {T - 1}) / {T}; geom[1] = (a.n[0] + {T - 1}) / {T}; "
                       f"geom[2] = 1; geom[3] = {T * T // (RI * R)}; geom[4] = geom[5] = 1;")
        elif n.shape == "brick":
            tk, tj = STENCIL_TILE
            out.append(f"  geom[0] = (a.n[2] + {tk - 1}) / {tk}; geom[1] = (a.n[1] + {tj - 1}) / {tj}; "
                       f"geom[2] = (a.n[0] + {BRICK_DEPTH - 1}) / {BRICK_DEPTH}; geom[3] = {tk}; geom[4] = {tj}; "
                       "geom[5] = 1;")
        elif n.shape == "stencil":
            tk, tj = STENCIL_TILE
            out.append(f"  {{ uint32_t tx = (a.n[2] + {tk - 1}) / {tk}, ty = (a.n[1] + {tj - 1}) / {tj};")
            out.append(f"    uint64_t want = (uint64_t)B2O_TARGET_CTAS; uint64_t tiles = (uint64_t)tx * ty;")
            out.append("    uint32_t chunks = (uint32_t)((want + tiles - 1) / tiles); if (chunks < 1) chunks = 1;")
            out.append("    if (chunks > a.n[0]) chunks = a.n[0];")
            out.append("    a.chunk = (a.n[0] + chunks - 1) / chunks;")
            out.append(f"    geom[0] = tx; geom[1] = ty; geom[2] = (a.n[0] + a.chunk - 1) / a.chunk; "
                       f"geom[3] = {tk}; geom[4] = {tj}; geom[5] = 1; }}")
        elif n.shape == "quad" and n.quad.get("march") and self.march_tma(n):
            # one CTA per (plane block, segment of bt quads of the row space)
            bt = int(self.spec.get("march_block", MARCH_BLOCK))
            D = len(n.chain)
            mid = " * ".join(f"(uint64_t)a.tn[{d}]" for d in range(1, D)) or "1"
            out.append(f"  {{ uint64_t nseg = ({mid} + {bt - 1}) / {bt}; uint64_t g = (uint64_t)a.tn[0] * nseg;")
            out.append("    if (g > 0x7FFFFFFFull) { ex->launch(ex, %d, 0, 0, 0); return; }" % lid)
            out.append(f"    geom[0] = (uint32_t)g; geom[1] = geom[2] = 1; geom[3] = {bt + 32}; "
                       "geom[4] = geom[5] = 1; }")
        else:
            bt = BLOCK_THREADS
            if n.shape == "quad" and n.quad.get("march"):
                bt = int(self.spec.get("march_block", MARCH_BLOCK))
            per = bt * n.ppt
            cap = int(self.spec.get("flat_grid_cap", 0)) or 0x7FFFFFFF
            if n.reds and set(n.reds) - set(n.exact or {}):
                cap = min(cap, 2048)  # B2O_RED_MAX_BLOCKS: one partial per CTA in the scratch
            out.append(f"  {{ uint64_t g = (total + {per - 1}) / {per}; geom[0] = (uint32_t)(g > {cap}u ? "
                       f"{cap}u : g); geom[1] = geom[2] = 1; geom[3] = {bt}; geom[4] = geom[5] = 1; }}")
        for v, (slot, cnt) in (n.exact or {}).items():
            out.append(f"  a.xb{v} = ({self.T(v)} *)ex->red_buf(ex, {slot}, (int64_t)total * {cnt}); if (ex->stop) return;")
        out.append(f"  ex->launch(ex, {lid}, &a, (uint32_t)sizeof a, geom);")
        for v, (slot, cnt) in (n.exact or {}).items():
            out.append(f"  if (!ex->stop) ex->red_exact(ex, {v}, {slot}, (int64_t)total * {cnt}, (double)a.s{v});")
        out.append("}")
        return out

    def _finals(self, n: NestPlan, ind: str) -> list[str]:
        prog = self.prog
        chain_idx = [prog.loops[c].index_var for c in n.chain]
        out = []
        for v in n.swrites:
            if n.reds and v in n.reds:
                continue  # written by the reduction epilogue
            if v in chain_idx:
                d = chain_idx.index(v)
                val = f"a.lo[{d}] + (int32_t)a.n[{d}]"
            else:
                val = f"v{v}"
            out.append(f"{ind}*({self.T(v)} *)((char *)a.slab + 8 * {v}) = {val};")
        return out

    def _locals(self, n: NestPlan, ind: str) -> list[str]:
        out = []
        for v in n.locals_:
            init = f"a.s{v}" if v in n.scalar_args else "0"
            cq = "const " if v not in n.writes else ""
            out.append(f"{ind}{cq}{self.T(v)} v{v} = {init};")
        return out

    def kernel_fn(self, n: NestPlan) -> list[str]:
        out = self._kernel_fn(n)
        assert out[0].rstrip().endswith("{"), out[0]
        # first statement of every kernel: programmatic-dependent-launch entry.
        # Memory-bound kernels let their dependents launch at once (the waiting
        # CTAs cost nothing there); the compute-bound k-tile kernel triggers
        # them only before its stores (b2o_pdl_trigger in ktile_kernel_fn), so
        # early dependents do not take issue slots from its FMA loop
        entry = "  b2o_pdl_wait();" if n.shape == "ktile" else "  b2o_pdl_enter();"
        return [out[0], entry] + out[1:]

    def _kernel_fn(self, n: NestPlan) -> list[str]:
        if n.shape == "stencil":
            return self.stencil_kernel_fn(n)
        if n.shape == "brick":
            return self.brick_kernel_fn(n)
        if n.shape == "ktile":
            return self.ktile_kernel_fn(n)
        if n.shape == "quad" and n.quad.get("march"):
            if self.march_tma(n):
                return self.quad_march_tma_kernel_fn(n)
            return self.quad_march_kernel_fn(n)
        if n.shape == "quad":
            return self.quad_kernel_fn(n)
        prog = self.prog
        lid = n.root
        U = n.ppt
        minb = self.spec.get("flat_min_blocks")
        lb = f"{BLOCK_THREADS}, {int(minb)}" if minb else f"{BLOCK_THREADS}"
        out = [f'extern "C" __global__ void __launch_bounds__({lb}) {n.kernel}(const KA_L{lid} a) {{']
        tree = {v: o for v, o in (n.reds or {}).items() if v not in (n.exact or {})}
        for v in tree:
            out.append(f"  {self.T(v)} rd{v} = ({self.T(v)})0;  // per-thread partial of reduction {prog.vars[v].name}")
        self._reds = n.reds or {}
        self._exact = n.exact or {}
        out.append("  auto point = [&](const uint32_t t) {")
        # the restrict pointers are declared inside the lambda: captured by
        # reference they lose __restrict__, and a store through one array
        # would then order every later load (an in-thread k loop turns into
        # one memory round trip per iteration)
        for v in n.arrays:
            const = "const " if v not in n.writes else ""
            out.append(f"    {const}{self.T(v)} *__restrict__ v{v} = a.p{v};")
        for v, (slot, cnt) in (n.exact or {}).items():
            if cnt > 1:
                out.append(f"    uint32_t xc{v} = 0;  // this point's terms of {prog.vars[v].name} so far")
        D = len(n.chain)
        for c in n.chain:
            out.append(f"    int32_t v{prog.loops[c].index_var}_;")
        KB = n.kb
        if D:
            out.append("    uint32_t r = t;")
            for d in range(D - 1, 0, -1):
                iv = prog.loops[n.chain[d]].index_var
                out.append(f"    {{ uint32_t q = b2o_fastdiv(r, a.mul[{d}], a.shr[{d}]); "
                           f"v{iv}_ = (int32_t)(r - q * a.tn[{d}]); r = q; }}")
            out.append(f"    v{prog.loops[n.chain[0]].index_var}_ = (int32_t)r;")
        for d, c in enumerate(n.chain):
            iv = prog.loops[c].index_var
            if d == D - 1 and KB > 1:
                continue
            out.append(f"    const int32_t v{iv} = a.lo[{d}] + v{iv}_;")
        out.extend(self._locals(n, "    "))
        if KB > 1:
            # KB consecutive points of the innermost loop per thread: one scope
            # per point with the same base pointers, so loads shared between
            # neighbouring points are common subexpressions
            kv = prog.loops[n.chain[-1]].index_var
            out.append(f"    const int32_t kb0 = v{kv}_ * {KB};")
            out.append("    const bool last_t = t == a.total - 1u;")
            for guarded in (False, True):
                out.append(f"    {'} else {' if guarded else f'if (kb0 + {KB} <= (int32_t)a.n[{D - 1}]) {{'}")
                for u in range(KB):
                    out.append(f"      {{ const int32_t v{kv} = a.lo[{D - 1}] + kb0 + {u};")
                    if guarded:
                        out.append(f"        if (kb0 + {u} < (int32_t)a.n[{D - 1}]) {{")
                    body: list[str] = []
                    self.dev_region(prog.loops[n.chain[-1]].body, 4, body)
                    out.extend(body)
                    out.append(f"        if (last_t && kb0 + {u} == (int32_t)a.n[{D - 1}] - 1) {{")
                    out.extend(self._finals(n, "          "))
                    out.append("        }")
                    if guarded:
                        out.append("        }")
                    out.append("      }")
            out.append("    }")
        else:
            body: list[str] = []
            if D:
                self.dev_region(prog.loops[n.chain[-1]].body, 2, body)
            else:
                self.dev_loop(lid, 2, body)
            out.extend(body)
            out.append("    if (t == a.total - 1u) {")
            out.extend(self._finals(n, "      "))
            out.append("    }")
        for v in n.locals_:
            if v not in n.swrites:
                out.append(f"    (void)v{v};")
        out.append("  };")
        out.append(f"  const uint32_t stride = gridDim.x * blockDim.x * {U}u;")
        out.append(f"  for (uint32_t t0 = blockIdx.x * blockDim.x * {U}u + threadIdx.x; t0 < a.total; t0 += stride) {{")
        if U > 1:
            # whole group in range: unrolled straight-line points (loads of
            # later points can issue before earlier stores: restrict pointers)
            out.append(f"    if (t0 + {U - 1}u * blockDim.x < a.total) {{")
            out.append("#pragma unroll")
            out.append(f"      for (uint32_t u = 0; u < {U}u; ++u) point(t0 + u * blockDim.x);")
            out.append("    } else {")
            out.append(f"      for (uint32_t u = 0; u < {U}u && t0 + u * blockDim.x < a.total; ++u) point(t0 + u * blockDim.x);")
            out.append("    }")
        else:
            out.append("    point(t0);")
        out.append("  }")
        self._reds = {}
        self._exact = {}
        if tree:
            out.extend(self._reduction_epilogue(n, tree))
        out.append("}")
        return out

    def _reduction_epilogue(self, n: NestPlan, reds: dict) -> list[str]:
        """Deterministic grid reduction: block totals (warp xor-butterfly +
        shared memory, b2o_block_sum) go to the scratch, one slot per CTA; the
        last CTA to finish (atomic ticket) sums the slots in CTA order, adds
        the value the scalar had at launch and stores it in the slab.  Fixed
        grid => bit-reproducible run to run."""
        out = ["  {", "    __shared__ double b2o_red_sm[32];", "    __shared__ int b2o_last;",
               "    char *scr_ = (char *)a.scratch;", "    unsigned *cnt_ = (unsigned *)scr_;"]
        for r, v in enumerate(reds):
            T = self.T(v)
            out.append(f"    {{ {T} bt = b2o_block_sum<{T}>(rd{v}, ({T} *)b2o_red_sm);")
            out.append(f"      if (threadIdx.x == 0) (({T} *)(scr_ + 256 + {r} * 8 * B2O_RED_MAX_BLOCKS))[blockIdx.x] = bt; }}")
        out.append("    if (threadIdx.x == 0) { __threadfence(); b2o_last = atomicAdd(cnt_, 1u) == gridDim.x - 1u; }")
        out.append("    __syncthreads();")
        out.append("    if (b2o_last) {")
        out.append("      __threadfence();")
        for r, v in enumerate(reds):
            T = self.T(v)
            out.append(f"      {{ const {T} *part = (const {T} *)(scr_ + 256 + {r} * 8 * B2O_RED_MAX_BLOCKS);")
            out.append(f"        {T} s = ({T})0;")
            out.append("        for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) s = s + __ldcg(part + b);")
            out.append(f"        s = b2o_block_sum<{T}>(s, ({T} *)b2o_red_sm);")
            out.append(f"        if (threadIdx.x == 0) *({T} *)((char *)a.slab + 8 * {v}) = ({T})(a.s{v} + s); }}")
        out.append("      if (threadIdx.x == 0) *cnt_ = 0u;")
        out.append("    }")
        out.append("  }")
        return out

    def quad_kernel_fn(self, n: NestPlan) -> list[str]:
        """Vectorised flat kernel (see :func:`quad_plan`): one thread per
        16-byte-aligned quad of a row of the innermost loop.  Every array
        reference becomes a lane of an aligned ``float4``/``int4`` chunk
        loaded once per thread (the 19 ``p`` reads of the Himeno Jacobi body
        share 18 chunks; the 12 coefficient arrays one chunk each), so the
        LSU issues ~8x fewer load instructions than the scalar flat kernel.
        Lanes outside the loop's range are masked at the store; aligned
        writes of fully valid quads are single 16-byte stores.  Each lane
        evaluates the same C expression tree as the CPU path (bit-exact)."""
        prog = self.prog
        lid = n.root
        qp = n.quad
        D = len(n.chain)
        iv = [prog.loops[c].index_var for c in n.chain]
        kv = iv[-1]
        minb = self.spec.get("flat_min_blocks")
        lb = f"{BLOCK_THREADS}, {int(minb)}" if minb else f"{BLOCK_THREADS}"
        out = [f'extern "C" __global__ void __launch_bounds__({lb}) {n.kernel}(const KA_L{lid} a) {{']
        for v in n.arrays:
            const = "const " if v not in n.writes else ""
            out.append(f"  {const}{self.T(v)} *__restrict__ v{v} = a.p{v};")
        out.extend(self._locals(n, "  "))
        G = qp["groups"]
        # warp-shuffle neighbour exchange (one quad per thread only): adjacent
        # lanes own adjacent aligned chunks of a row, so of a run of chunks
        # {o-1, o, o+1} a thread loads o and takes the lanes it needs of o-1 /
        # o+1 from lanes -1 / +1; lanes whose neighbour sits in another row,
        # another warp or is idle load those elements directly
        shfl = G == 1 and bool(self.spec.get("quad_shfl", False))  # measured slower
        out.append("  const uint32_t stride = gridDim.x * blockDim.x;")
        if shfl:
            out.append("  const uint32_t lane_ = threadIdx.x & 31u;")
            out.append("  for (uint32_t tw_ = blockIdx.x * blockDim.x + threadIdx.x - lane_; tw_ < a.total; "
                       "tw_ += stride) {")
            out.append("    const uint32_t t = tw_ + lane_;")
            out.append("    const bool act_ = t < a.total;")
            out.append("    if (t == a.total - 1u) {")
            out.extend(self._finals(n, "      "))
            out.append("    }")
            out.append("    uint32_t r = act_ ? t : a.total - 1u;")
        else:
            out.append("  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < a.total; t += stride) {")
            out.append("    if (t == a.total - 1u) {")
            out.extend(self._finals(n, "      "))
            out.append("    }")
            out.append("    uint32_t r = t;")
        for d in range(D - 1, 0, -1):
            nm = "q_" if d == D - 1 else f"v{iv[d]}_"
            out.append(f"    uint32_t {nm};")
            out.append(f"    {{ uint32_t q = b2o_fastdiv(r, a.mul[{d}], a.shr[{d}]); {nm} = r - q * a.tn[{d}]; r = q; }}")
        if D == 1:
            out.append("    const uint32_t q_ = r;")
        else:
            out.append(f"    const uint32_t v{iv[0]}_ = r;")
        for d in range(D - 1):
            out.append(f"    const int32_t v{iv[d]} = a.lo[{d}] + (int32_t)v{iv[d]}_;")
        row = [f"(int64_t){c} * v{v}" for v, c in zip(qp["ovars"], qp["outer"]) if c]
        out.append(f"    const int64_t F_ = {' + '.join(row) if row else '0'};")
        L = QUAD * G  # lanes (points) per thread: G aligned quads of one row
        out.append(f"    const int64_t b_ = ((F_ + a.lo[{D - 1}]) & ~(int64_t){QUAD - 1}) + (int64_t){L} * q_;")
        out.append(f"    const int32_t k0_ = (int32_t)(b_ - F_);")
        out.append(f"    const int32_t kr_ = k0_ - a.lo[{D - 1}];")
        out.append(f"    const int32_t kn_ = (int32_t)a.n[{D - 1}];")
        if not shfl:
            out.append(f"    if (kr_ + {L - 1} < 0 || kr_ >= kn_) continue;")
        else:
            out.append(f"    const bool ok_ = act_ && !(kr_ + {L - 1} < 0 || kr_ >= kn_);")
        # aligned chunks every read needs, and the lanes used of each
        comps: dict = {}
        for v, c in qp["reads"]:
            for u in range(L):
                comps.setdefault((v, (c + u) // QUAD), set()).add((c + u) % QUAD)
        chunks = sorted(comps)

        def cname(v, o):
            return f"c{v}_{'m' if o < 0 else ''}{abs(o)}"

        def ldexpr(v, o):
            vt = "float4" if self.T(v) == "float" else "int4"
            if v in qp["writes"]:  # read-only path only for arrays the nest never writes
                return f"(reinterpret_cast<const {vt} *>(v{v} + b_)[{o}])"
            return f"__ldg(reinterpret_cast<const {vt} *>(v{v} + b_) + ({o}))"

        npf = self.next_pf(n)
        if npf and not shfl:
            # the next launch's chunks (one host iteration further): L2 prefetch
            ro = sorted({(v, o) for v, o in chunks if v not in qp["writes"]})
            out.append("    if (a.pfn) {")
            for v, o in ro:
                out.append(f"      {{ const char *pf_ = reinterpret_cast<const char *>(v{v} + b_ + {npf[1]} + "
                           f"{QUAD * o}); asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(pf_)); }}")
            out.append("    }")
        shuffled: set = set()  # chunks held as per-lane scalars taken from neighbours
        if not shfl:
            for v, o in chunks:
                vt = "float4" if self.T(v) == "float" else "int4"
                out.append(f"    const {vt} {cname(v, o)} = {ldexpr(v, o)};")
        else:
            out.append("    const unsigned vm_ = __ballot_sync(0xffffffffu, ok_);")
            out.append("    const uint32_t bl_ = (uint32_t)b_;")
            # runs of consecutive chunks per array: load the middle one
            runs: list = []
            for v, o in chunks:
                if runs and runs[-1][0] == v and runs[-1][-1] == o - 1:
                    runs[-1].append(o)
                else:
                    runs.append([v, o])
            # the centre is the chunk with the most lanes used (ties: the
            # middle one); a neighbour chunk of which more than quad_shfl_max
            # lanes are needed is loaded rather than shuffled
            smax = int(self.spec.get("quad_shfl_max", 2))
            deltas = set()
            centres = {}
            loaded: list = []
            for run in runs:
                v, os_ = run[0], run[1:]
                mid = os_[len(os_) // 2]
                oc = max(os_, key=lambda o: (len(comps[(v, o)]), -abs(o - mid)))
                loaded.append((v, oc))
                for o in os_:
                    if o == oc:
                        continue
                    if len(comps[(v, o)]) > smax or abs(o - oc) > 1:
                        loaded.append((v, o))
                    else:
                        centres[(v, o)] = oc
                        deltas.add(o - oc)
            for dl in sorted(deltas):
                nm = f"nb{'m' if dl < 0 else ''}{abs(dl)}_"
                # the shuffle runs on every lane (never behind a short-circuit)
                out.append(f"    const uint32_t {nm}b = __shfl_sync(0xffffffffu, bl_, (lane_ + ({dl})) & 31u);")
                out.append(f"    const bool {nm} = (lane_ + ({dl})) < 32u && ((vm_ >> ((lane_ + ({dl})) & 31u)) & 1u) "
                           f"&& {nm}b == bl_ + {QUAD * dl}u;")
            for v, o in sorted(loaded):
                vt = "float4" if self.T(v) == "float" else "int4"
                zero = "make_float4(0.f, 0.f, 0.f, 0.f)" if vt == "float4" else "make_int4(0, 0, 0, 0)"
                out.append(f"    {vt} {cname(v, o)} = {zero};")
                out.append(f"    if (ok_) {cname(v, o)} = {ldexpr(v, o)};")
            for (v, o), oc in sorted(centres.items()):
                T = self.T(v)
                dl = o - oc
                nm = f"nb{'m' if dl < 0 else ''}{abs(dl)}_"
                shuffled.add((v, o))
                for j in sorted(comps[(v, o)]):
                    x = f"{cname(v, o)}_{j}"
                    out.append(f"    {T} {x} = __shfl_sync(0xffffffffu, {cname(v, oc)}.{'xyzw'[j]}, "
                               f"(lane_ + ({dl})) & 31u);")
                    ptr = f"v{v} + b_ + ({QUAD * o + j})"
                    src = f"__ldg({ptr})" if v not in qp["writes"] else f"*({ptr})"
                    out.append(f"    if (!{nm} && ok_) {x} = {src};")
            out.append("    if (!ok_) continue;")
        ivs = set(qp["ivs"])

        latest: dict[int, int] = {}  # array -> statement whose lane values it now holds

        def lane_expr(e, u):
            k = e[0]
            if k == "arr" and e[1] in latest:
                return f"r{latest[e[1]]}_{u}"
            if k == "arr":
                c = affine(e[2], ivs)[1]
                el = c + u
                if (e[1], el // QUAD) in shuffled:
                    return f"{cname(e[1], el // QUAD)}_{el % QUAD}"
                return f"{cname(e[1], el // QUAD)}.{'xyzw'[el % QUAD]}"
            if k == "var" and e[1] == kv:
                return f"(k0_ + {u})"
            if k in ("num", "var"):
                return render(e, self.local_name)
            return f"({lane_expr(e[2], u)} {e[1]} {lane_expr(e[3], u)})"

        body = prog.regions[prog.loops[n.chain[-1]].body].statements
        for si, st in enumerate(body):
            v = st.target[1]
            T = self.T(v)
            for u in range(L):
                out.append(f"    const {T} r{si}_{u} = ({T})({lane_expr(st.value, u)});")
            latest[v] = si
        for si, st in enumerate(body):
            v = st.target[1]
            c = qp["writes"][v]
            for g in range(G):
                us = range(QUAD * g, QUAD * g + QUAD)
                lanes = [f"r{si}_{u}" for u in us]
                masked = [f"      if ((uint32_t)(kr_ + {u}) < (uint32_t)kn_) v{v}[b_ + ({c + u})] = r{si}_{u};"
                          for u in us]
                if c % QUAD == 0:
                    vt = "float4" if self.T(v) == "float" else "int4"
                    mk = "make_float4" if vt == "float4" else "make_int4"
                    out.append(f"    if (kr_ + {QUAD * g} >= 0 && kr_ + {QUAD * g + QUAD} <= kn_) {{")
                    out.append(f"      reinterpret_cast<{vt} *>(v{v} + b_)[{c // QUAD + g}] = {mk}({', '.join(lanes)});")
                    out.append("    } else {")
                    out.extend(masked)
                    out.append("    }")
                else:
                    out.append("    {")
                    out.extend(masked)
                    out.append("    }")
        for v in n.locals_:
            out.append(f"    (void)v{v};")
        out.append("  }")
        out.append("}")
        return out

    def march_streams(self, n: NestPlan) -> list[tuple[int, int, int, int]]:
        """TMA streams of a plane-march nest: one per (read-only array, plane
        offset) among the chunks loaded fresh each step, with the chunk-offset
        range they cover: ``[(v, d, lo, hi)]``."""
        qp = n.quad
        mp = qp["march"]
        keys = mp["keys"]
        carried = {k for k in keys if (k[0], k[1] + 1, k[2]) in keys and k[0] not in qp["writes"]}
        rng: dict = {}
        for v, d, o in keys - carried:
            if v in qp["writes"] or self.T(v) not in ("float", "int32_t"):
                continue
            lo, hi = rng.get((v, d), (o, o))
            rng[(v, d)] = (min(lo, o), max(hi, o))
        return [(v, d, lo, hi) for (v, d), (lo, hi) in sorted(rng.items())]

    def march_tma(self, n: NestPlan) -> bool:
        """The TMA-fed variant (spec ``march_tma``, default OFF: measured
        slower than the register kernel on NAS-MG resid 258^3 -- 58.8 us at
        Z=32/4 stages vs 50.7 us, profiles/r02/README.md) applies when the
        march loads anything fresh per step from read-only arrays."""
        if not self.spec.get("march_tma", False) or self.spec.get("march_async") or \
                self.spec.get("march_prefetch"):
            return False
        return self.march_tma_span(n) >= MARCH_TMA_MIN_SPAN

    def march_tma_span(self, n: NestPlan) -> int:
        """Largest per-CTA chunk span the ring can stage within the 48 KB of
        static shared memory (0: no stream)."""
        streams = self.march_streams(n)
        if not streams:
            return 0
        P = int(self.spec.get("march_tma_stages", MARCH_TMA_STAGES))
        budget = (48 * 1024 - 64) // (16 * P)  # chunks per stage
        fixed = sum(1 + hi - lo for _, _, lo, hi in streams)
        fit = (budget - fixed) // len(streams) - 1
        return min(int(self.spec.get("march_tma_span", MARCH_TMA_SPAN)), fit)

    def quad_march_tma_kernel_fn(self, n: NestPlan) -> list[str]:
        """TMA-fed plane-marching quad kernel.  A CTA owns ``bt`` consecutive
        quads of the (rows x quads) index space of one block of ``Z`` planes
        -- consecutive quads are consecutive 16-byte chunks of the flattened
        arrays, so the chunks every stream of the CTA needs from one plane form
        ONE contiguous range [bmin + lo, bmax + hi].  An extra producer warp
        streams those ranges plane by plane with bulk asynchronous copies
        (``cp.async.bulk``, completion on a "full" mbarrier) into a
        ``P``-stage shared-memory ring, refilling a stage once every consumer
        warp has released it ("empty" mbarrier) -- no CTA-wide barrier per
        step.  Consumer threads read their leading chunks from the ring and
        carry the rest in registers exactly as the register kernel does
        (:meth:`quad_march_kernel_fn`).  A CTA whose quads span more than
        ``MAXSPAN`` chunks (very short rows) loads directly.  Lanes evaluate
        the same C expression tree (bit-exact)."""
        prog = self.prog
        lid = n.root
        qp = n.quad
        mp = qp["march"]
        Z = mp["Z"]
        C0 = mp["C0"]
        D = len(n.chain)
        iv = [prog.loops[c].index_var for c in n.chain]
        bt = int(self.spec.get("march_block", MARCH_BLOCK))
        P = int(self.spec.get("march_tma_stages", MARCH_TMA_STAGES))
        SPAN = self.march_tma_span(n)
        streams = self.march_streams(n)
        offs, tot = [], 0
        for v, d, lo, hi in streams:
            offs.append(tot)
            tot += SPAN + 1 + hi - lo
        NW = bt // 32  # consumer warps
        out = [f'extern "C" __global__ void __launch_bounds__({bt + 32}) {n.kernel}(const KA_L{lid} a) {{']
        for v in n.arrays:
            const = "const " if v not in n.writes else ""
            out.append(f"  {const}{self.T(v)} *__restrict__ v{v} = a.p{v};")
        out.extend(self._locals(n, "  "))
        out.append(f"  __shared__ __align__(128) int4 ring_[{P}][{tot}];")
        out.append(f"  __shared__ __align__(8) unsigned long long full_[{P}], empty_[{P}];")
        out.append("  __shared__ long long bmin_, bmax_;")
        out.append("  if (threadIdx.x == 0) {")
        out.append(f"    for (int p_ = 0; p_ < {P}; ++p_) {{ b2o_mbar_init(&full_[p_], 1u); "
                   f"b2o_mbar_init(&empty_[p_], {NW}u); }}")
        out.append("    b2o_mbar_fence_init();")
        out.append("    bmin_ = 0x7fffffffffffffffll; bmax_ = -0x7fffffffffffffffll;")
        out.append("  }")
        out.append("  __syncthreads();")
        mid = " * ".join(f"a.tn[{d}]" for d in range(1, D)) or "1u"
        out.append(f"  const uint32_t nmid_ = {mid};")
        out.append(f"  const uint32_t nseg_ = (nmid_ + {bt - 1}u) / {bt}u;")
        out.append("  const uint32_t zb_ = blockIdx.x / nseg_, seg_ = blockIdx.x - zb_ * nseg_;")
        out.append(f"  const bool prod_ = threadIdx.x >= {bt}u;  // the producer warp")
        out.append(f"  const uint32_t tin_ = seg_ * {bt}u + threadIdx.x;")
        out.append("  bool act_ = !prod_ && tin_ < nmid_ && zb_ < a.tn[0];")
        out.append("  const uint32_t t = zb_ * nmid_ + tin_;")
        out.append("  if (act_ && t == a.total - 1u) {")
        out.extend(self._finals(n, "    "))
        out.append("  }")
        out.append("  uint32_t r = act_ ? tin_ : 0u;")
        for d in range(D - 1, 0, -1):
            nm = "q_" if d == D - 1 else f"v{iv[d]}_"
            out.append(f"  uint32_t {nm};")
            out.append(f"  {{ uint32_t q = b2o_fastdiv(r, a.mul[{d}], a.shr[{d}]); {nm} = r - q * a.tn[{d}]; r = q; }}")
        out.append(f"  const uint32_t z0_ = zb_ * {Z}u;")
        out.append(f"  const uint32_t zn_ = zb_ < a.tn[0] ? min({Z}u, a.n[0] - z0_) : 0u;")
        for d in range(1, D - 1):
            out.append(f"  const int32_t v{iv[d]} = a.lo[{d}] + (int32_t)v{iv[d]}_;")
        out.append(f"  int32_t v{iv[0]} = a.lo[0] + (int32_t)z0_;")
        row = [f"(int64_t){c} * v{v}" for v, c in zip(qp["ovars"], qp["outer"]) if c]
        out.append(f"  const int64_t F0_ = {' + '.join(row) if row else '0'};")
        out.append(f"  int64_t b_ = ((F0_ + a.lo[{D - 1}]) & ~(int64_t){QUAD - 1}) + (int64_t){QUAD} * q_;")
        out.append(f"  const int32_t k0_ = (int32_t)(b_ - F0_);")
        out.append(f"  const int32_t kr_ = k0_ - a.lo[{D - 1}];")
        out.append(f"  const int32_t kn_ = (int32_t)a.n[{D - 1}];")
        out.append(f"  act_ = act_ && !(kr_ + {QUAD - 1} < 0 || kr_ >= kn_);")
        out.append(f"  const long long bc_ = b_ / {QUAD};")
        out.append("  if (act_) { atomicMin(&bmin_, bc_); atomicMax(&bmax_, bc_); }")
        out.append("  __syncthreads();")
        out.append("  const long long bmin = bmin_, bmax = bmax_;")
        out.append(f"  const bool tma_ = bmax >= bmin && bmax - bmin <= {SPAN};")
        out.append("  if (prod_) {")
        out.append("    // producer: step s (>= 1) of the march into stage (s - 1) % P, after")
        out.append("    // the consumers released that stage's previous use")
        out.append("    if (!tma_ || threadIdx.x != " + str(bt) + "u) return;")
        out.append("    const unsigned ext_ = (unsigned)(bmax - bmin);")
        nbytes = " + ".join(f"(ext_ + {1 + hi - lo}u)" for _, _, lo, hi in streams)
        out.append("    for (uint32_t s = 1; s < zn_; ++s) {")
        out.append(f"      const uint32_t st = (s - 1u) % {P}u, use = (s - 1u) / {P}u;")
        out.append("      if (use > 0) b2o_mbar_wait(&empty_[st], (use - 1u) & 1u);")
        out.append(f"      b2o_mbar_expect_tx(&full_[st], 16u * ({nbytes}));")
        for (v, d, lo, hi), off in zip(streams, offs):
            out.append(f"      b2o_bulk_g2s(&ring_[st][{off}], reinterpret_cast<const int4 *>(v{v}) + "
                       f"(bmin + (long long)({d} + (int)s) * {C0 // QUAD} + ({lo})), 16u * (ext_ + {1 + hi - lo}u), "
                       f"&full_[st]);")
        out.append("    }")
        out.append("    return;")
        out.append("  }")
        keys = mp["keys"]

        def cname(v, d, o):
            return f"h{v}_{'m' if d < 0 else ''}{abs(d)}_{'m' if o < 0 else ''}{abs(o)}"

        def ldexpr(v, d, o):
            vt = "float4" if self.T(v) == "float" else "int4"
            off = d * C0 // QUAD + o
            if v in qp["writes"]:
                return f"(reinterpret_cast<const {vt} *>(v{v} + b_)[{off}])"
            return f"__ldg(reinterpret_cast<const {vt} *>(v{v} + b_) + ({off}))"

        for v, d, o in sorted(keys):
            vt = "float4" if self.T(v) == "float" else "int4"
            zero = "make_float4(0.f, 0.f, 0.f, 0.f)" if vt == "float4" else "make_int4(0, 0, 0, 0)"
            out.append(f"  {vt} {cname(v, d, o)} = act_ ? {ldexpr(v, d, o)} : {zero};")
        carried = {k for k in keys if (k[0], k[1] + 1, k[2]) in keys and k[0] not in qp["writes"]}
        sidx = {}
        for (v, d, lo, hi), off in zip(streams, offs):
            for o in range(lo, hi + 1):
                sidx[(v, d, o)] = off - lo + o
        out.append("  for (uint32_t s_ = 0; s_ < zn_; ++s_) {")
        out.append("    if (s_ > 0) {")
        out.append(f"      b_ += (int64_t){C0}; ++v{iv[0]};")
        out.append(f"      const uint32_t st_ = (s_ - 1u) % {P}u;")
        out.append(f"      if (tma_) b2o_mbar_wait(&full_[st_], ((s_ - 1u) / {P}u) & 1u);")
        out.append("      if (act_) {")
        for v, d, o in sorted(keys, key=lambda k: (k[1], k[0], k[2])):
            if (v, d, o) in carried:
                out.append(f"        {cname(v, d, o)} = {cname(v, d + 1, o)};")
            elif (v, d, o) in sidx:
                vt = "float4" if self.T(v) == "float" else "int4"
                out.append(f"        {cname(v, d, o)} = tma_ ? *reinterpret_cast<const {vt} *>("
                           f"&ring_[st_][(unsigned)(bc_ - bmin) + {sidx[(v, d, o)]}]) : "
                           f"{ldexpr(v, d, o)};")
            else:
                out.append(f"        {cname(v, d, o)} = {ldexpr(v, d, o)};")
        out.append("      }")
        out.append("      if (tma_) {  // this warp is done with the stage")
        out.append("        __syncwarp();")
        out.append("        if ((threadIdx.x & 31u) == 0u) b2o_mbar_arrive(&empty_[st_]);")
        out.append("      }")
        out.append("    }")
        out.append("    if (!act_) continue;")
        out.extend(self._march_compute(n, cname, "    "))
        out.append("  }")
        for v in n.locals_:
            out.append(f"  (void)v{v};")
        out.append("}")
        return out

    def _march_compute(self, n: NestPlan, cname, ind: str) -> list[str]:
        """Lanes and stores of one plane step of a march kernel."""
        prog = self.prog
        qp = n.quad
        mp = qp["march"]
        kv = prog.loops[n.chain[-1]].index_var
        ivs = set(qp["ivs"])
        latest: dict[int, int] = {}
        out = []

        def lane_expr(e, u):
            k = e[0]
            if k == "arr" and e[1] in latest:
                return f"r{latest[e[1]]}_{u}"
            if k == "arr":
                c = affine(e[2], ivs)[1]
                d, rest = mp["split"](c)
                el = rest + u
                return f"{cname(e[1], d, el // QUAD)}.{'xyzw'[el % QUAD]}"
            if k == "var" and e[1] == kv:
                return f"(k0_ + {u})"
            if k in ("num", "var"):
                return render(e, self.local_name)
            return f"({lane_expr(e[2], u)} {e[1]} {lane_expr(e[3], u)})"

        body = prog.regions[prog.loops[n.chain[-1]].body].statements
        for si, st in enumerate(body):
            v = st.target[1]
            T = self.T(v)
            for u in range(QUAD):
                out.append(f"{ind}const {T} r{si}_{u} = ({T})({lane_expr(st.value, u)});")
            latest[v] = si
        for si, st in enumerate(body):
            v = st.target[1]
            c = qp["writes"][v]
            lanes = [f"r{si}_{u}" for u in range(QUAD)]
            masked = [f"{ind}  if ((uint32_t)(kr_ + {u}) < (uint32_t)kn_) v{v}[b_ + ({c + u})] = r{si}_{u};"
                      for u in range(QUAD)]
            if c % QUAD == 0:
                vt = "float4" if self.T(v) == "float" else "int4"
                mk = "make_float4" if vt == "float4" else "make_int4"
                out.append(f"{ind}if (kr_ >= 0 && kr_ + {QUAD} <= kn_) {{")
                out.append(f"{ind}  reinterpret_cast<{vt} *>(v{v} + b_)[{c // QUAD}] = {mk}({', '.join(lanes)});")
                out.append(f"{ind}}} else {{")
                out.extend(masked)
                out.append(f"{ind}}}")
            else:
                out.append(f"{ind}{{")
                out.extend(masked)
                out.append(f"{ind}}}")
        return out

    def quad_march_kernel_fn(self, n: NestPlan) -> list[str]:
        """Plane-marching quad kernel (see :func:`march_plan`): a thread owns
        one aligned quad of a row and walks ``Z`` consecutive values of the
        outermost chain index.  Because the plane stride is a multiple of the
        quad, the chunks a reference at plane offset ``d`` needs at step
        ``s + 1`` are the ones the reference at ``d + 1`` loaded at step
        ``s``: they move between registers and only the leading plane is
        loaded (NAS-MG resid: 9 of 25 chunks per step).  No shared memory, no
        barrier; coalescing is the quad kernel's (adjacent lanes, adjacent
        quads).  Lanes evaluate the same C expression tree (bit-exact)."""
        prog = self.prog
        lid = n.root
        qp = n.quad
        mp = qp["march"]
        Z = mp["Z"]
        D = len(n.chain)
        iv = [prog.loops[c].index_var for c in n.chain]
        kv = iv[-1]
        minb = self.spec.get("flat_min_blocks")
        bt = int(self.spec.get("march_block", MARCH_BLOCK))
        lb = f"{bt}, {int(minb)}" if minb else f"{bt}"
        out = [f'extern "C" __global__ void __launch_bounds__({lb}) {n.kernel}(const KA_L{lid} a) {{']
        for v in n.arrays:
            const = "const " if v not in n.writes else ""
            out.append(f"  {const}{self.T(v)} *__restrict__ v{v} = a.p{v};")
        out.extend(self._locals(n, "  "))
        # warp-shuffle neighbour chunks (spec ``march_shfl``): the leading
        # plane's chunks at quad offsets +-1 of a loaded chunk come from the
        # neighbouring lane (same row: the lane's base address says so),
        # halving the L1 wavefronts per step; every lane of the warp walks
        # the same number of steps (predicated), so the shuffles converge
        sh = bool(self.spec.get("march_shfl", MARCH_SHFL)) and not self.spec.get("march_async") and \
            not self.spec.get("march_prefetch")
        out.append("  const uint32_t stride = gridDim.x * blockDim.x;")
        if sh:
            out.append("  const uint32_t lane_ = threadIdx.x & 31u;")
            out.append("  for (uint32_t tw_ = blockIdx.x * blockDim.x + threadIdx.x - lane_; tw_ < a.total; "
                       "tw_ += stride) {")
            out.append("    const uint32_t t = tw_ + lane_;")
            out.append("    const bool act_ = t < a.total;")
        else:
            out.append("  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < a.total; t += stride) {")
        out.append("    if (t == a.total - 1u) {")
        out.extend(self._finals(n, "      "))
        out.append("    }")
        out.append("    uint32_t r = t;")
        for d in range(D - 1, 0, -1):
            nm = "q_" if d == D - 1 else f"v{iv[d]}_"
            out.append(f"    uint32_t {nm};")
            out.append(f"    {{ uint32_t q = b2o_fastdiv(r, a.mul[{d}], a.shr[{d}]); {nm} = r - q * a.tn[{d}]; r = q; }}")
        out.append(f"    const uint32_t z0_ = r * {Z}u;")
        out.append(f"    const uint32_t zn_ = min({Z}u, a.n[0] - z0_);")
        for d in range(1, D - 1):
            out.append(f"    const int32_t v{iv[d]} = a.lo[{d}] + (int32_t)v{iv[d]}_;")
        out.append(f"    int32_t v{iv[0]} = a.lo[0] + (int32_t)z0_;")
        row = [f"(int64_t){c} * v{v}" for v, c in zip(qp["ovars"], qp["outer"]) if c]
        out.append(f"    const int64_t F0_ = {' + '.join(row) if row else '0'};")
        out.append(f"    int64_t b_ = ((F0_ + a.lo[{D - 1}]) & ~(int64_t){QUAD - 1}) + (int64_t){QUAD} * q_;")
        out.append(f"    const int32_t k0_ = (int32_t)(b_ - F0_);")
        out.append(f"    const int32_t kr_ = k0_ - a.lo[{D - 1}];")
        out.append(f"    const int32_t kn_ = (int32_t)a.n[{D - 1}];")
        if sh:
            out.append(f"    const bool ok_ = act_ && !(kr_ + {QUAD - 1} < 0 || kr_ >= kn_);")
            out.append("    const uint32_t zw_ = __reduce_max_sync(0xffffffffu, ok_ ? zn_ : 0u);")
            out.append("    const uint32_t bl_ = (uint32_t)b_;")
            out.append("    const unsigned vm0_ = __ballot_sync(0xffffffffu, ok_);")
            # neighbour lanes on the same row (their chunk is this chunk +-1)
            for dl in (-1, 1):
                nm = f"nb{'m' if dl < 0 else ''}{abs(dl)}_"
                out.append(f"    const uint32_t {nm}b = __shfl_sync(0xffffffffu, bl_, (lane_ + ({dl})) & 31u);")
                out.append(f"    const bool {nm} = (lane_ + ({dl})) < 32u && ((vm0_ >> ((lane_ + ({dl})) & 31u)) & 1u) "
                           f"&& {nm}b == bl_ + {QUAD * dl}u;")
        else:
            out.append(f"    if (kr_ + {QUAD - 1} < 0 || kr_ >= kn_) continue;")
        C0 = mp["C0"]
        keys = set(mp["keys"])  # {(v, d, o)} chunks relative to the current plane
        ivs = set(qp["ivs"])
        body = prog.regions[prog.loops[n.chain[-1]].body].statements
        # plane-local subexpression chains (spec ``march_chains``): a maximal
        # subexpression whose array leaves are all read-only and on one plane
        # (e.g. NAS-MG's u(z-1, j-1, k) + u(z-1, j+1, k)) is evaluated once,
        # when its plane is the leading plane, and carried to the later steps
        # as one scalar register instead of its operand chunks -- the same
        # operations on the same operands in the same order, so the value is
        # bit-identical; subexpressions equal up to the plane share one chain
        # (and across lanes and statements).  Frees registers for occupancy.
        MIX, INV = "mix", "inv"
        targets = {st.target[1] for st in body}
        inv_vars = (set(n.scalar_args) - set(n.writes) - targets) | {kv}
        use_chains = bool(self.spec.get("march_chains", MARCH_CHAINS)) and \
            not self.spec.get("march_async") and not self.spec.get("march_prefetch")

        def plane_of(e):
            k = e[0]
            if k == "num":
                return INV
            if k == "var":
                return INV if e[1] in inv_vars else MIX
            if k == "arr":
                if e[1] in targets or e[1] in qp["writes"]:
                    return MIX
                return mp["split"](affine(e[2], ivs)[1])[0]
            a_, b_p = plane_of(e[2]), plane_of(e[3])
            if MIX in (a_, b_p):
                return MIX
            if a_ == INV:
                return b_p
            if b_p == INV:
                return a_
            return a_ if a_ == b_p else MIX

        def canon(e, u):
            k = e[0]
            if k == "arr":
                el = mp["split"](affine(e[2], ivs)[1])[1] + u
                return f"a{e[1]}[{el // QUAD}].{'xyzw'[el % QUAD]}"
            if k == "var" and e[1] == kv:
                return f"(k0_ + {u})"
            if k in ("num", "var"):
                return render(e, self.local_name)
            return f"({canon(e[2], u)} {e[1]} {canon(e[3], u)})"

        def leaf_chunks(e, u, acc):
            if e[0] == "arr":
                el = mp["split"](affine(e[2], ivs)[1])[1] + u
                acc.add((e[1], el // QUAD))
            elif e[0] == "bin":
                leaf_chunks(e[2], u, acc)
                leaf_chunks(e[3], u, acc)
            return acc

        chains: dict[str, dict] = {}
        if use_chains:
            plain: set = set()

            def collect(e, u):
                if e[0] == "bin":
                    pl = plane_of(e)
                    if pl not in (MIX, INV):
                        ch = chains.setdefault(canon(e, u), {"e": e, "u": u, "ds": set(),
                                                             "T": etype(prog, e, self.precision),
                                                             "leaves": leaf_chunks(e, u, set())})
                        ch["ds"].add(pl)
                        return
                    collect(e[2], u)
                    collect(e[3], u)
                elif e[0] == "arr":
                    d, rest = mp["split"](affine(e[2], ivs)[1])
                    plain.add((e[1], d, (rest + u) // QUAD))

            for st in body:
                for u in range(QUAD):
                    collect(st.value, u)
            if chains:
                dmax_v: dict[int, int] = {}
                for v, d, o in keys:
                    if v not in qp["writes"]:
                        dmax_v[v] = max(dmax_v.get(v, d), d)
                keys = set(plain)
                for i, (ck, ch) in enumerate(sorted(chains.items())):
                    ch["name"] = f"p{i}_"
                    ch["h"] = min(dmax_v[v] for v, _ in ch["leaves"])
                    ch["dmin"] = min(ch["ds"])
                    keys |= {(v, ch["h"], o) for v, o in ch["leaves"]}
            else:
                use_chains = False
        if self.spec.get("march_fill", MARCH_FILL):
            # carry a chunk through the planes between its first and last use
            # (a register move per step) instead of reloading it: NAS-MG's
            # (j, k-1) and (j, k+4) chunks are read at planes -1 and +1 only
            for v, o in {(v, o) for v, _, o in keys if v not in qp["writes"]}:
                ds = [d for w, d, p in keys if w == v and p == o]
                keys.update((v, d, o) for d in range(min(ds), max(ds) + 1))

        def cname(v, d, o):
            return f"h{v}_{'m' if d < 0 else ''}{abs(d)}_{'m' if o < 0 else ''}{abs(o)}"

        def ldexpr(v, d, o, ahead=0):
            vt = "float4" if self.T(v) == "float" else "int4"
            off = (d + ahead) * C0 // QUAD + o
            if v in qp["writes"]:
                return f"(reinterpret_cast<const {vt} *>(v{v} + b_)[{off}])"
            return f"__ldg(reinterpret_cast<const {vt} *>(v{v} + b_) + ({off}))"

        for v, d, o in sorted(keys):
            vt = "float4" if self.T(v) == "float" else "int4"
            if sh:
                zero = "make_float4(0.f, 0.f, 0.f, 0.f)" if vt == "float4" else "make_int4(0, 0, 0, 0)"
                out.append(f"    {vt} {cname(v, d, o)} = ok_ ? {ldexpr(v, d, o)} : {zero};")
            else:
                out.append(f"    {vt} {cname(v, d, o)} = {ldexpr(v, d, o)};")

        def dnm(d):
            return f"{'m' if d < 0 else ''}{abs(d)}"

        def chain_expr(e, u, d, prologue):
            """the chain's subexpression on plane offset d (chunk registers, or
            direct loads for prologue planes no chunk register holds)"""
            k = e[0]
            if k == "arr":
                el = mp["split"](affine(e[2], ivs)[1])[1] + u
                key = (e[1], d, el // QUAD)
                if key in keys or not prologue:
                    return f"{cname(*key)}.{'xyzw'[el % QUAD]}"
                return f"{ldexpr(*key)}.{'xyzw'[el % QUAD]}"
            if k == "var" and e[1] == kv:
                return f"(k0_ + {u})"
            if k in ("num", "var"):
                return render(e, self.local_name)
            return f"({chain_expr(e[2], u, d, prologue)} {e[1]} {chain_expr(e[3], u, d, prologue)})"

        for ch in (chains.values() if use_chains else ()):
            for d in range(ch["dmin"], ch["h"] + 1):
                val = f"({ch['T']}){chain_expr(ch['e'], ch['u'], d, True)}"
                out.append(f"    {ch['T']} {ch['name']}{dnm(d)} = " + (f"ok_ ? {val} : ({ch['T']})0;" if sh else f"{val};"))
        carried = {k for k in keys if (k[0], k[1] + 1, k[2]) in keys and k[0] not in qp["writes"]}
        lead = sorted(keys - carried)
        # shuffle sources: runs of consecutive leading chunks of one array and
        # plane; the centre (most components used) is loaded, its +-1
        # neighbours are shuffled from the adjacent lanes
        sh_from: dict = {}
        if sh:
            used: dict = {}
            for st in body:
                for u in range(QUAD):
                    stack = [st.value]
                    while stack:
                        e = stack.pop()
                        if e[0] == "arr" and e[1] not in qp["writes"] and e[1] not in targets:
                            d_, rest = mp["split"](affine(e[2], ivs)[1])
                            used.setdefault((e[1], d_, (rest + u) // QUAD), set()).add((rest + u) % QUAD)
                        elif e[0] == "bin":
                            stack += [e[2], e[3]]
            runs: list = []
            for v, d, o in lead:
                if v in qp["writes"]:
                    continue
                if runs and runs[-1][0] == (v, d) and runs[-1][-1] == o - 1:
                    runs[-1].append(o)
                else:
                    runs.append([(v, d), o])
            for run in runs:
                (v, d), os_ = run[0], run[1:]
                if len(os_) < 2:
                    continue
                mid = os_[len(os_) // 2]
                oc = max(os_, key=lambda o: (len(used.get((v, d, o), ())), -abs(o - mid)))
                for o in os_:
                    if o != oc and abs(o - oc) == 1:
                        sh_from[(v, d, o)] = oc
        # staged leading plane: each thread copies its own next-plane chunks
        # into private shared-memory slots (cp.async, P-stage ring) and reads
        # them back one step later -- no barrier (a thread reads only what it
        # copied), the copies in flight hold no registers
        P = int(self.spec.get("march_async", 0) or 0)
        staged = [k for k in lead if k[0] not in qp["writes"]] if P >= 2 else []
        if staged:
            vts = {self.T(v) for v, _, _ in staged}
            if vts - {"float", "int32_t"}:
                staged = []
        if staged:
            NS = len(staged)
            out.append(f"    __shared__ __align__(16) int4 st_[{P}][{NS}][{bt}];")
            sidx = {k: i for i, k in enumerate(staged)}

            def issue(plane_off, slot, ind):
                for i, (v, d, o) in enumerate(staged):
                    off = (d + plane_off) * C0 // QUAD + o
                    out.append(f"{ind}b2o_cp16(&st_[{slot}][{i}][threadIdx.x], "
                               f"reinterpret_cast<const int4 *>(v{v} + b_) + ({off}));")
        # software pipelining: the chunks the next plane loads are issued
        # before this plane's arithmetic (prefetch registers n*)
        pipe = bool(self.spec.get("march_prefetch", False))  # measured slower
        if pipe:
            for v, d, o in lead:
                vt = "float4" if self.T(v) == "float" else "int4"
                out.append(f"    {vt} n{cname(v, d, o)};")
        if staged:
            # prologue: planes 1 .. P-1 into slots 1 .. P-1 (one group each)
            for q in range(1, P):
                out.append(f"    if ({q}u < zn_) {{")
                issue(q, q, "      ")
                out.append("    }")
                out.append("    b2o_cp_commit();")
        # L2 prefetch of the leading plane PF steps ahead (spec ``march_l2pf``):
        # one prefetch per read-only array at the thread's own chunk of that
        # plane -- every chunk of a plane is some thread's own, so the whole
        # plane is requested from DRAM PF steps early without holding
        # registers; the neighbour-row loads then hit L2.  Guarded to planes
        # the nest itself reads.
        PF = int(self.spec.get("march_l2pf", MARCH_L2PF) or 0)
        pf_lines = []
        if PF > 0 and not staged:
            dmax: dict[int, int] = {}
            for v, d, o in keys:
                if v not in qp["writes"]:
                    dmax[v] = max(dmax.get(v, d), d)
            for v in sorted(dmax):
                off = (dmax[v] + PF) * C0
                pf_lines.append(f"{{ const char *pf_ = reinterpret_cast<const char *>(v{v} + b_ + {off}); "
                                f"asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(pf_)); }}")
            pf_guard = (f"if ({'live_ && ' if sh else ''}v{iv[0]} + {PF} < a.lo[0] + (int32_t)a.n[0])")
            for q in range(1, PF):  # prologue: the first steps' leading planes
                out.append(f"    if ({'ok_ && ' if sh else ''}v{iv[0]} + {q} < a.lo[0] + (int32_t)a.n[0] && {q}u < zn_) {{")
                for v in sorted(dmax):
                    out.append(f"      {{ const char *pf_ = reinterpret_cast<const char *>(v{v} + b_ + "
                               f"{(dmax[v] + q) * C0}); asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(pf_)); }}")
                out.append("    }")
        if sh:
            out.append("    for (uint32_t s_ = 0; s_ < zw_; ++s_) {")
            out.append("      const bool live_ = ok_ && s_ < zn_;")
        else:
            out.append("    for (uint32_t s_ = 0; s_ < zn_; ++s_) {")
        out.append("      if (s_ > 0) {")
        out.append(f"        b_ += (int64_t){C0}; ++v{iv[0]};")
        for ch in (chains.values() if use_chains else ()):
            for d in range(ch["dmin"], ch["h"]):
                out.append(f"        {ch['name']}{dnm(d)} = {ch['name']}{dnm(d + 1)};")
        if staged:
            # plane s_+P-1 goes out, plane s_ must be in: P-1 younger groups
            # may stay pending
            out.append(f"        if (s_ + {P - 1}u < zn_) {{")
            issue(P - 1, f"(s_ + {P - 1}u) % {P}u", "          ")
            out.append("        }")
            out.append("        b2o_cp_commit();")
            out.append(f"        b2o_cp_wait<{P - 1}>();")
        # ascending plane offset: the old value of (d+1) is read before it
        # is replaced
        for v, d, o in sorted(keys, key=lambda k: (k[1], k[0], (k in sh_from), k[2])):
            if (v, d, o) in carried:
                out.append(f"        {cname(v, d, o)} = {cname(v, d + 1, o)};")
            elif staged and (v, d, o) in sidx:
                vt = "float4" if self.T(v) == "float" else "int4"
                out.append(f"        {cname(v, d, o)} = *reinterpret_cast<const {vt} *>("
                           f"&st_[s_ % {P}u][{sidx[(v, d, o)]}][threadIdx.x]);")
            elif pipe:
                out.append(f"        {cname(v, d, o)} = n{cname(v, d, o)};")
            elif sh and (v, d, o) in sh_from:
                oc = sh_from[(v, d, o)]
                dl = o - oc
                nm = f"nb{'m' if dl < 0 else ''}{abs(dl)}_"
                vt = "float4" if self.T(v) == "float" else "int4"
                T = self.T(v)
                comps4 = []
                for j in range(QUAD):
                    x = f"{cname(v, d, o)}_{j}"
                    out.append(f"        {T} {x} = __shfl_sync(0xffffffffu, {cname(v, d, oc)}.{'xyzw'[j]}, "
                               f"(lane_ + ({dl})) & 31u);")
                    comps4.append(x)
                mk = "make_float4" if vt == "float4" else "make_int4"
                out.append(f"        {cname(v, d, o)} = {mk}({', '.join(comps4)});")
                out.append(f"        if (!{nm} && live_) {cname(v, d, o)} = {ldexpr(v, d, o)};")
            elif sh:
                out.append(f"        if (live_) {cname(v, d, o)} = {ldexpr(v, d, o)};")
            else:
                out.append(f"        {cname(v, d, o)} = {ldexpr(v, d, o)};")
        for ch in (chains.values() if use_chains else ()):
            h = ch["h"]
            out.append(f"        {ch['name']}{dnm(h)} = ({ch['T']}){chain_expr(ch['e'], ch['u'], h, False)};")
        out.append("      }")
        if pf_lines:  # b_ is the current plane here
            out.append(f"      {pf_guard} {{")
            out.extend("        " + x for x in pf_lines)
            out.append("      }")
        if pipe:
            out.append("      if (s_ + 1 < zn_) {")
            for v, d, o in lead:
                out.append(f"        n{cname(v, d, o)} = {ldexpr(v, d, o, 1)};")
            out.append("      }")
        latest: dict[int, int] = {}

        def lane_expr(e, u):
            k = e[0]
            if use_chains and k == "bin":
                pl = plane_of(e)
                if pl not in (MIX, INV):
                    return f"{chains[canon(e, u)]['name']}{dnm(pl)}"
            if k == "arr" and e[1] in latest:
                return f"r{latest[e[1]]}_{u}"
            if k == "arr":
                c = affine(e[2], ivs)[1]
                d, rest = mp["split"](c)
                el = rest + u
                return f"{cname(e[1], d, el // QUAD)}.{'xyzw'[el % QUAD]}"
            if k == "var" and e[1] == kv:
                return f"(k0_ + {u})"
            if k in ("num", "var"):
                return render(e, self.local_name)
            return f"({lane_expr(e[2], u)} {e[1]} {lane_expr(e[3], u)})"

        body = prog.regions[prog.loops[n.chain[-1]].body].statements
        for si, st in enumerate(body):
            v = st.target[1]
            T = self.T(v)
            for u in range(QUAD):
                out.append(f"      const {T} r{si}_{u} = ({T})({lane_expr(st.value, u)});")
            latest[v] = si
        for si, st in enumerate(body):
            v = st.target[1]
            c = qp["writes"][v]
            lanes = [f"r{si}_{u}" for u in range(QUAD)]
            live = "live_ && " if sh else ""
            masked = [f"        if ({live}(uint32_t)(kr_ + {u}) < (uint32_t)kn_) v{v}[b_ + ({c + u})] = r{si}_{u};"
                      for u in range(QUAD)]
            if c % QUAD == 0:
                vt = "float4" if self.T(v) == "float" else "int4"
                mk = "make_float4" if vt == "float4" else "make_int4"
                out.append(f"      if ({'live_ && ' if sh else ''}kr_ >= 0 && kr_ + {QUAD} <= kn_) {{")
                out.append(f"        reinterpret_cast<{vt} *>(v{v} + b_)[{c // QUAD}] = {mk}({', '.join(lanes)});")
                out.append("      } else {")
                out.extend(masked)
                out.append("      }")
            else:
                out.append("      {")
                out.extend(masked)
                out.append("      }")
        out.append("    }")
        for v in n.locals_:
            out.append(f"    (void)v{v};")
        out.append("  }")
        out.append("}")
        return out

    def ktile_kernel_fn(self, n: NestPlan) -> list[str]:
        """Register-tiled k-reduction kernel (see :func:`ktile_plan`): a CTA
        of 256 threads owns a 64 x 64 block of (i, j) points, each thread a
        4 x 4 micro-tile whose accumulators live in registers.  The k loop
        runs in stages of 32: the A operands (i, k) and B operands (k, j) of
        the stage are staged in shared memory (coalesced along whichever index
        has unit stride), then every point applies the k-loop statements for
        k ascending, each statement the same C expression as the CPU path, so
        the per-point operation sequence (and every rounding) is the
        sequential loop's."""
        prog = self.prog
        lid = n.root
        kp = n.ktile
        iv, jv, kv = kp["iv"], kp["jv"], kp["kv"]
        T = int(self.spec.get("ktile_tile", KT_TI))
        R, TI, TJ, BK = int(self.spec.get("ktile_r", KT_R)), T, T, KT_BK
        RI = int(self.spec.get("ktile_ri", R))  # micro-tile rows (i); R columns (j)
        nthr = TI * TJ // (RI * R)
        if TI % RI or TJ % R or (BK * TI) % nthr or (BK * TJ) % nthr or nthr % 32 or nthr > 1024:
            # the staging loops move BK * T / nthr elements per thread: a tile
            # that does not divide evenly would leave operands unstaged
            raise CompileError(f"k-tile shape {TI} x {TJ} with {RI} x {R} micro-tiles is unsupported: "
                               f"{nthr} threads must be a multiple of 32 dividing {BK} x the tile edge")
        TX = TJ // R  # threads along j
        K = prog.loops[kp["kloop"]]
        body = prog.regions[prog.loops[n.chain[1]].body].statements
        kbody = prog.regions[K.body].statements
        pre, post = body[:kp["kpos"]], body[kp["kpos"] + 1:]
        out = [f'extern "C" __global__ void __launch_bounds__({nthr}) {n.kernel}(const KA_L{lid} a) {{']
        for v in n.arrays:
            const = "const " if v not in n.writes else ""
            out.append(f"  {const}{self.T(v)} *__restrict__ v{v} = a.p{v};")
        out.extend(self._locals(n, "  "))
        tiles = sorted(kp["tiles"].items(), key=lambda x: x[1][1])
        for (v, co, c0), (side, t) in tiles:
            ext = TI if side == "A" else TJ
            out.append(f"  __shared__ __align__(16) float s{t}_[{BK}][{ext + 4}];")
        out.append(f"  const int tx_ = threadIdx.x % {TX}, ty_ = threadIdx.x / {TX};")
        out.append(f"  const int32_t i0_ = a.lo[0] + (int32_t)(blockIdx.y * {TI}u), "
                   f"j0_ = a.lo[1] + (int32_t)(blockIdx.x * {TJ}u);")
        out.append(f"  const int32_t ie_ = a.lo[0] + (int32_t)a.n[0], je_ = a.lo[1] + (int32_t)a.n[1];")
        for p_ in range(RI):
            out.append(f"  const int32_t vI{p_} = i0_ + ty_ * {RI} + {p_};")
        for q_ in range(R):
            out.append(f"  const int32_t vJ{q_} = j0_ + tx_ * {R} + {q_};")
        out.append(f"  const int32_t klo_ = {self.bound(K.lower, self.local_name)}, "
                   f"khi_ = {self.bound(K.upper, self.local_name)};")
        out.append(f"  const bool full_ = i0_ + {TI} <= ie_ && j0_ + {TJ} <= je_;")
        out.append("  (void)full_;")

        def sub(e, p_, q_, inner):
            """C text of ``e`` for point (p_, q_) of the micro-tile."""
            k = e[0]
            if k == "num":
                return render(e, self.local_name)
            if k == "var":
                if e[1] == iv:
                    return f"vI{p_}"
                if e[1] == jv:
                    return f"vJ{q_}"
                if e[1] == kv:
                    return "vK_"
                return self.local_name(e[1], False)
            if k == "arr":
                v = e[1]
                if v in kp["accs"]:
                    return f"acc{v}_{p_}{q_}"
                if inner:
                    aff = affine(e[2], {iv, jv, kv})
                    key = (v, tuple(sorted(aff[0].items())), aff[1])
                    side, t = kp["tiles"][key]
                    return f"a{t}_{p_}" if side == "A" else f"b{t}_{q_}"
                return f"v{v}[{sub(e[2], p_, q_, inner)}]"
            return f"({sub(e[2], p_, q_, inner)} {e[1]} {sub(e[3], p_, q_, inner)})"

        first_read = {}
        for st in pre + kbody + post:
            refs: list = []
            _array_refs(st.value, refs)
            for r in refs:
                if r[1] in kp["accs"]:
                    first_read.setdefault(r[1], True)
            first_read.setdefault(st.target[1], False)
        for v in sorted(kp["accs"]):
            for p_ in range(RI):
                for q_ in range(R):
                    if first_read.get(v):
                        # the accumulator starts from the array's current value
                        idx = sub(self._acc_index(kp, v), p_, q_, False)
                        out.append(f"  float acc{v}_{p_}{q_} = (vI{p_} < ie_ && vJ{q_} < je_) ? v{v}[{idx}] : 0.f;")
                    else:
                        out.append(f"  float acc{v}_{p_}{q_} = 0.f;")

        def emit(sts, inner, ind):
            for st in sts:
                v = st.target[1]
                for p_ in range(RI):
                    for q_ in range(R):
                        val = sub(st.value, p_, q_, inner)
                        line = f"acc{v}_{p_}{q_} = (float)({val});"
                        if inner:
                            out.append(f"{ind}{line}")
                        else:
                            out.append(f"{ind}if (vI{p_} < ie_ && vJ{q_} < je_) {line}")

        emit(pre, False, "  ")
        # operand staging: each thread moves ELT elements of every tile per
        # stage; the next stage's elements are loaded into registers while
        # the current stage is consumed from shared memory
        ELT = BK * max(TI, TJ) // nthr

        swz = bool(self.spec.get("ktile_swz", True))

        def slot(cod, ov, ext, r_):
            """(k, other) tile coordinates of staging element r_ of this
            thread.  When k has unit stride, lanes walk k; with ``swz`` a warp
            covers 8 consecutive k of 4 rows (32-byte segments, still whole
            sectors) so the transposed shared-memory stores hit 32 distinct
            banks (row pitch ext+4 = 4 mod 32)."""
            e = f"(threadIdx.x + {r_ * nthr})"
            kfast = abs(cod.get(kv, 0)) == 1 and abs(cod.get(ov, 0)) != 1
            if not kfast:
                return f"({e} / {ext})", f"({e} % {ext})"
            if swz and BK % 8 == 0 and ext % 4 == 0:
                return f"(({e} & 7) + 8 * ({e} / {8 * ext}))", f"(({e} >> 3) % {ext})"
            return f"({e} % {BK})", f"({e} / {BK})"

        def tile_load(side, t, v, co, c0, kb, dst, ind, guard=True):
            cod = dict(co)
            ext = TI if side == "A" else TJ
            ov = iv if side == "A" else jv
            o0, oe = ("i0_", "ie_") if side == "A" else ("j0_", "je_")
            for r_ in range(BK * ext // nthr):
                kk, oo = slot(cod, ov, ext, r_)
                terms = [f"(int64_t){cod.get(kv, 0)} * ({kb} + {kk})", f"(int64_t){cod.get(ov, 0)} * ({o0} + {oo})"]
                for x, c in cod.items():
                    if x not in (kv, ov):
                        terms.append(f"(int64_t){c} * {self.local_name(x, False)}")
                addr = " + ".join(terms + [f"(int64_t){c0}"])
                if guard:
                    out.append(f"{ind}{dst(r_, kk, oo)} = ({kb} + {kk} < khi_ && {o0} + {oo} < {oe}) "
                               f"? __ldg(v{v} + ({addr})) : 0.f;")
                else:
                    out.append(f"{ind}{dst(r_, kk, oo)} = __ldg(v{v} + ({addr}));")

        def tile_store(side, t, v, co, c0, ind):
            cod = dict(co)
            ext = TI if side == "A" else TJ
            ov = iv if side == "A" else jv
            for r_ in range(BK * ext // nthr):
                kk, oo = slot(cod, ov, ext, r_)
                out.append(f"{ind}s{t}_[{kk}][{oo}] = p{t}_{r_};")

        for (v, co, c0), (side, t) in tiles:
            ext = TI if side == "A" else TJ
            for r_ in range(BK * ext // nthr):
                out.append(f"  float p{t}_{r_};")
        for (v, co, c0), (side, t) in tiles:
            tile_load(side, t, v, co, c0, "klo_", lambda r_, kk, oo, t=t: f"p{t}_{r_}", "  ")
        for (v, co, c0), (side, t) in tiles:
            tile_store(side, t, v, co, c0, "  ")
        out.append("  __syncthreads();")
        out.append(f"  for (int32_t kb_ = klo_; kb_ < khi_; kb_ += {BK}) {{")
        out.append(f"    const int32_t kn_ = min({BK}, khi_ - kb_);")
        # fast paths (bit-identical: the per-point operation sequence is
        # unchanged): unguarded staging loads when the whole next stage lies
        # inside the nest's ranges, and a fully unrolled k stage with the next
        # k's shared-memory operands loaded one step ahead
        fast = bool(self.spec.get("ktile_fast", True))
        out.append(f"    if (kb_ + {BK} < khi_) {{")
        if fast:
            out.append(f"      if (full_ && kb_ + {2 * BK} <= khi_) {{")
            for (v, co, c0), (side, t) in tiles:
                tile_load(side, t, v, co, c0, f"(kb_ + {BK})", lambda r_, kk, oo, t=t: f"p{t}_{r_}", "        ",
                          guard=False)
            out.append("      } else {")
            for (v, co, c0), (side, t) in tiles:
                tile_load(side, t, v, co, c0, f"(kb_ + {BK})", lambda r_, kk, oo, t=t: f"p{t}_{r_}", "        ")
            out.append("      }")
        else:
            for (v, co, c0), (side, t) in tiles:
                tile_load(side, t, v, co, c0, f"(kb_ + {BK})", lambda r_, kk, oo, t=t: f"p{t}_{r_}", "      ")
        out.append("    }")

        def operands(kk, src, ind):
            for (v, co, c0), (side, t) in tiles:
                nm, off = (f"a{t}", "ty_") if side == "A" else (f"b{t}", "tx_")
                RS = RI if side == "A" else R
                for h_ in range(RS // 4):
                    rhs = (f"*reinterpret_cast<const float4 *>(&s{t}_[{kk}][{off} * {RS} + {4 * h_}])"
                           if src is None else f"{nm}n{h_}_")
                    out.append(f"{ind}const float4 {nm}q{h_}_ = {rhs};")
                for p_ in range(RS):
                    out.append(f"{ind}const float {nm}_{p_} = {nm}q{p_ // 4}_.{'xyzw'[p_ % 4]};")

        def prefetch(kk, decl, ind):
            for (v, co, c0), (side, t) in tiles:
                nm, off = (f"a{t}", "ty_") if side == "A" else (f"b{t}", "tx_")
                RS = RI if side == "A" else R
                for h_ in range(RS // 4):
                    out.append(f"{ind}{'float4 ' if decl else ''}{nm}n{h_}_ = "
                               f"*reinterpret_cast<const float4 *>(&s{t}_[{kk}][{off} * {RS} + {4 * h_}]);")

        if fast:
            pf = bool(self.spec.get("ktile_prefetch", True))
            out.append(f"    if (kn_ == {BK}) {{")
            if pf:
                prefetch("0", True, "      ")
            out.append("#pragma unroll")
            out.append(f"      for (int kk_ = 0; kk_ < {BK}; ++kk_) {{")
            out.append("        const int32_t vK_ = kb_ + kk_;")
            operands("kk_", "n" if pf else None, "        ")
            if pf:
                out.append(f"        if (kk_ + 1 < {BK}) {{")
                prefetch("kk_ + 1", False, "          ")
                out.append("        }")
            emit(kbody, True, "        ")
            out.append("        (void)vK_;")
            out.append("      }")
            out.append("    } else {")
        out.append("#pragma unroll 4")
        out.append("    for (int kk_ = 0; kk_ < kn_; ++kk_) {")
        out.append("      const int32_t vK_ = kb_ + kk_;")
        operands("kk_", None, "      ")
        emit(kbody, True, "      ")
        out.append("      (void)vK_;")
        out.append("    }")
        if fast:
            out.append("    }")
        out.append(f"    if (kb_ + {BK} < khi_) {{")
        out.append("      __syncthreads();")
        for (v, co, c0), (side, t) in tiles:
            tile_store(side, t, v, co, c0, "      ")
        out.append("      __syncthreads();")
        out.append("    }")
        out.append("  }")
        emit(post, False, "  ")
        out.append("  b2o_pdl_trigger();")
        for v in sorted(kp["accs"]):
            for p_ in range(RI):
                for q_ in range(R):
                    idx = sub(self._acc_index(kp, v), p_, q_, False)
                    out.append(f"  if (vI{p_} < ie_ && vJ{q_} < je_) v{v}[{idx}] = acc{v}_{p_}{q_};")
        out.append("  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {")
        if kv in n.swrites:
            out.append(f"    v{kv} = khi_ > klo_ ? khi_ : klo_;")
        out.extend(self._finals(n, "    "))
        out.append("  }")
        for v in n.locals_:
            out.append(f"  (void)v{v};")
        out.append("}")
        return out

    def _acc_index(self, kp: dict, v: int):
        """The index expression an accumulator array is written at."""
        for st in self.prog.walk(self.prog.loops[self.prog.loops[kp["kloop"]].parent].body):
            if st.kind == "assign" and st.target[1] == v:
                return st.target[2]
        raise CompileError(f"accumulator {v} has no assignment")

    def brick_kernel_fn(self, n: NestPlan) -> list[str]:
        """3-D brick tiling: the CTA stages a (BI+2) x (TJ+2) x (TK+2) box of
        each staged array (tile + one-point halo) in shared memory with ONE
        barrier, then every thread computes BI points along the outer chain
        loop, unrolled, so the stream loads of all BI points are independent
        and in flight together.  Staged neighbours come from SMEM."""
        prog = self.prog
        lid = n.root
        tk, tj = STENCIL_TILE
        BI = BRICK_DEPTH
        hk, hj, hi = tk + 2, tj + 2, BI + 2
        nthr = tk * tj
        iv = [prog.loops[c].index_var for c in n.chain]
        out = [f'extern "C" __global__ void __launch_bounds__({nthr}) {n.kernel}(const KA_L{lid} a) {{']
        for v in n.arrays:
            const = "const " if v not in n.writes else ""
            out.append(f"  {const}{self.T(v)} *__restrict__ v{v} = a.p{v};")
        for v in n.staged:
            out.append(f"  __shared__ {self.T(v)} s{v}[{hi}][{hj}][{hk}];")
        out.append("  const int tk = threadIdx.x, tj = threadIdx.y;")
        out.append(f"  const uint32_t ok_ = blockIdx.x * {tk}u + tk, oj_ = blockIdx.y * {tj}u + tj;")
        out.append("  const bool inside = ok_ < a.n[2] && oj_ < a.n[1];")
        out.append(f"  const int32_t v{iv[2]} = a.lo[2] + (int32_t)ok_;")
        out.append(f"  const int32_t v{iv[1]} = a.lo[1] + (int32_t)oj_;")
        out.append(f"  const int32_t i0 = a.lo[0] + (int32_t)(blockIdx.z * {BI}u);")
        out.append(f"  const int32_t i_end = a.lo[0] + (int32_t)a.n[0];")
        out.append(f"  const int32_t j0 = a.lo[1] + (int32_t)(blockIdx.y * {tj}u) - 1;")
        out.append(f"  const int32_t k0 = a.lo[2] + (int32_t)(blockIdx.x * {tk}u) - 1;")
        out.append(f"  const int lin = tj * {tk} + tk;")
        for v, st in n.staged.items():
            T = self.T(v)
            L = prog.vars[v].length
            out.append(f"  for (int e = lin; e < {hi * hj * hk}; e += {nthr}) {{")
            out.append(f"    const int ii = e / {hj * hk}, rem = e - ii * {hj * hk}, jj = rem / {hk}, kk = rem - jj * {hk};")
            out.append(f"    const int64_t g = (int64_t){st['ci']} * (i0 - 1 + ii) + (int64_t){st['cj']} * (j0 + jj) + (k0 + kk);")
            out.append(f"    s{v}[ii][jj][kk] = (g >= 0 && g < {L}) ? v{v}[g] : ({T})0;")
            out.append("  }")
        out.append("  __syncthreads();")
        out.append("  if (!inside) return;")
        out.append("#pragma unroll")
        out.append(f"  for (int q = 0; q < {BI}; ++q) {{")
        out.append(f"    const int32_t v{iv[0]} = i0 + q;")
        out.append(f"    if (v{iv[0]} >= i_end) break;")
        out.extend(self._locals(n, "    "))
        body: list[str] = []
        self._staged = {v: dict(st, brick=True) for v, st in n.staged.items()}
        self._streams = None
        self._stencil_iv = iv
        self.dev_region(prog.loops[n.chain[-1]].body, 2, body)
        self._staged = None
        out.extend(body)
        out.append(f"    if (v{iv[0]} == i_end - 1 && ok_ == a.n[2] - 1u && oj_ == a.n[1] - 1u) {{")
        out.extend(self._finals(n, "      "))
        out.append("    }")
        for v in n.locals_:
            if v not in n.swrites:
                out.append(f"    (void)v{v};")
        out.append("  }")
        out.append("}")
        return out

    def stencil_kernel_fn(self, n: NestPlan) -> list[str]:
        """2.5-D plane marching (SURVEY.md §2.2 K1 technique notes).

        The CTA owns a TK x TJ tile of the two inner chain loops and walks a
        chunk of the outer loop.  Staged arrays (read-only, >= 4 unit-radius
        affine offsets) keep a rolling window of planes (tile + halo) in
        shared memory: each element is read from HBM once, neighbours come
        from SMEM.  Stream arrays (read-only, one affine index) are read
        straight into registers.  Both are double-buffered in registers: the
        next plane's halo values and stream values are requested before the
        barrier of the current plane, so every thread keeps ~one plane of
        loads in flight across the barriers."""
        prog = self.prog
        lid = n.root
        tk, tj = STENCIL_TILE
        hk, hj = tk + 2, tj + 2
        nthr = tk * tj
        halo = hk * hj
        per = (halo + nthr - 1) // nthr  # halo elements per thread
        iv = [prog.loops[c].index_var for c in n.chain]
        minb = self.spec.get("stencil_min_blocks")
        lb = f"{nthr}, {int(minb)}" if minb else f"{nthr}"
        out = [f'extern "C" __global__ void __launch_bounds__({lb}) {n.kernel}(const KA_L{lid} a) {{']
        for v in n.arrays:
            const = "const " if v not in n.writes else ""
            out.append(f"  {const}{self.T(v)} *__restrict__ v{v} = a.p{v};")
        for v, st in n.staged.items():
            out.append(f"  __shared__ {self.T(v)} s{v}[{st['planes']}][{hj}][{hk}];")
        out.append("  const int tk = threadIdx.x, tj = threadIdx.y;")
        out.append(f"  const uint32_t ok_ = blockIdx.x * {tk}u + tk, oj_ = blockIdx.y * {tj}u + tj;")
        out.append("  const bool inside = ok_ < a.n[2] && oj_ < a.n[1];")
        out.append(f"  const int32_t v{iv[2]} = a.lo[2] + (int32_t)ok_;")
        out.append(f"  const int32_t v{iv[1]} = a.lo[1] + (int32_t)oj_;")
        out.append("  const int32_t i_begin = a.lo[0] + (int32_t)(blockIdx.z * a.chunk);")
        out.append("  int32_t i_end = i_begin + (int32_t)a.chunk;")
        out.append("  if (i_end > a.lo[0] + (int32_t)a.n[0]) i_end = a.lo[0] + (int32_t)a.n[0];")
        out.append(f"  const int32_t j0 = a.lo[1] + (int32_t)(blockIdx.y * {tj}u) - 1;")
        out.append(f"  const int32_t k0 = a.lo[2] + (int32_t)(blockIdx.x * {tk}u) - 1;")
        out.append(f"  const int lin = tj * {tk} + tk;")
        # halo slots owned by this thread
        for q in range(per):
            out.append(f"  const int hj{q} = (lin + {q * nthr}) / {hk}, hk{q} = (lin + {q * nthr}) - hj{q} * {hk};")
            out.append(f"  const bool hv{q} = lin + {q * nthr} < {halo};")
        for v, st in n.staged.items():
            T = self.T(v)
            L = prog.vars[v].length
            ci, cj = st["ci"], st["cj"]
            P, dmin = st["planes"], st["dmin"]
            dmax = dmin + P - 1
            out.append(f"  auto fetch{v} = [&](int32_t ii, int q_j, int q_k) -> {T} {{")
            out.append(f"    const int64_t g = (int64_t){ci} * ii + (int64_t){cj} * (j0 + q_j) + (k0 + q_k);")
            out.append(f"    return (g >= 0 && g < {L}) ? v{v}[g] : ({T})0;")
            out.append("  };")
            # plane i_begin + dmin lives in buffer 0, the next in 1, ...; the
            # window rotates by one buffer per plane (no modulo in the loop)
            out.append(f"  for (int32_t d = {dmin}; d < {dmax}; ++d) {{")
            for q in range(per):
                out.append(f"    if (hv{q}) s{v}[d - ({dmin})][hj{q}][hk{q}] = fetch{v}(i_begin + d, hj{q}, hk{q});")
            out.append("  }")
            out.append(f"  int b{v}_base = {-dmin};          // buffer of plane i (offset 0)")
            out.append(f"  int b{v}_new = {P - 1};           // buffer receiving plane i + dmax")
            for q in range(per):
                out.append(f"  {T} h{v}_{q} = hv{q} ? fetch{v}(i_begin + {dmax}, hj{q}, hk{q}) : ({T})0;")
        for v, st in n.streams.items():
            T = self.T(v)
            co, c0 = st["ci"], st["base"]
            out.append(f"  const int64_t sb{v} = {c0};")
            out.append(f"  {T} pf{v} = (inside && i_begin < i_end) ? v{v}[sb{v} + (int64_t){co} * i_begin] : ({T})0;")
        out.append(f"  for (int32_t v{iv[0]} = i_begin; v{iv[0]} < i_end; ++v{iv[0]}) {{")
        out.append(f"    const bool more = v{iv[0]} + 1 < i_end;")
        for v, st in n.staged.items():
            T = self.T(v)
            dmax = st["dmin"] + st["planes"] - 1
            for q in range(per):
                out.append(f"    if (hv{q}) s{v}[b{v}_new][hj{q}][hk{q}] = h{v}_{q};")
            out.append("    if (more) {")
            for q in range(per):
                out.append(f"      if (hv{q}) h{v}_{q} = fetch{v}(v{iv[0]} + {dmax + 1}, hj{q}, hk{q});")
            out.append("    }")
        for v, st in n.streams.items():
            T = self.T(v)
            out.append(f"    const {T} c{v} = pf{v};")
            out.append(f"    if (inside && more) pf{v} = v{v}[sb{v} + (int64_t){st['ci']} * (v{iv[0]} + 1)];")
        out.append("    __syncthreads();")
        out.append("    if (inside) {")
        out.extend(self._locals(n, "      "))
        body: list[str] = []
        self._staged = n.staged
        self._streams = n.streams
        self._stencil_iv = iv
        self.dev_region(prog.loops[n.chain[-1]].body, 3, body)
        self._staged = None
        self._streams = None
        out.extend(body)
        out.append(f"      if (v{iv[0]} == a.lo[0] + (int32_t)a.n[0] - 1 && ok_ == a.n[2] - 1u && oj_ == a.n[1] - 1u) {{")
        out.extend(self._finals(n, "        "))
        out.append("      }")
        for v in n.locals_:
            if v not in n.swrites:
                out.append(f"      (void)v{v};")
        out.append("    }")
        out.append("    __syncthreads();")
        for v, st in n.staged.items():
            P = st["planes"]
            out.append(f"    b{v}_base = b{v}_base + 1 == {P} ? 0 : b{v}_base + 1;")
            out.append(f"    b{v}_new = b{v}_new + 1 == {P} ? 0 : b{v}_new + 1;")
        out.append("  }")
        out.append("}")
        return out

    def dev_name(self, vid: int, is_array: bool) -> str:
        return f"v{vid}"

    def dev_expr(self, e) -> str:
        """Device rendering; staged stencil reads become shared-memory reads."""
        staged = getattr(self, "_staged", None)
        if not staged:
            return render(e, self.local_name)

        def rec(x):
            k = x[0]
            if k == "arr" and x[1] in staged:
                st = staged[x[1]]
                di, dj, dk = stencil_offset(x[2], self._stencil_iv, st["ci"], st["cj"])
                if st.get("brick"):
                    return f"s{x[1]}[q + {1 + di}][tj + {1 + dj}][tk + {1 + dk}]"
                P = st["planes"]
                buf = f"((b{x[1]}_base + {di % P}) % {P})" if di else f"b{x[1]}_base"
                return f"s{x[1]}[{buf}][tj + {1 + dj}][tk + {1 + dk}]"
            if k == "arr" and self._streams and x[1] in self._streams:
                return f"c{x[1]}"
            if k == "num" or k == "var":
                return render(x, self.local_name)
            if k == "arr":
                return f"v{x[1]}[{rec(x[2])}]"
            return f"({rec(x[2])} {x[1]} {rec(x[3])})"

        return rec(e)

    def dev_loop(self, lid: int, ind: int, out: list[str]) -> None:
        loop = self.prog.loops[lid]
        iv = f"v{loop.index_var}"
        out.append("  " * ind + f"for ({iv} = {render(loop.lower, self.local_name)}; {iv} < "
                   f"{render(loop.upper, self.local_name)}; {iv}++) {{")
        self.dev_region(loop.body, ind + 1, out)
        out.append("  " * ind + "}")

    def dev_region(self, rid: int, ind: int, out: list[str]) -> None:
        prog = self.prog
        for st in prog.regions[rid].statements:
            pad = "  " * ind
            if st.kind == "decl":
                if st.init is not None:
                    out.append(pad + f"v{st.var} = {render(st.init, self.local_name)};")
            elif st.kind == "assign":
                red = reductions.reduction_stmt(st) if getattr(self, "_reds", None) else None
                if red is not None and red[0] in getattr(self, "_exact", {}):
                    # the term of this point, in loop order (t); s - e == s + (-e) exactly
                    v, op, e = red
                    sign = "-" if op == "-" else ""
                    cnt = self._exact[v][1]
                    T = self.T(v)
                    if cnt == 1:
                        out.append(pad + f"a.xb{v}[t] = {sign}({T})({self.dev_expr(e)});")
                    else:
                        out.append(pad + f"a.xb{v}[(size_t)t * {cnt}u + xc{v}++] = {sign}({T})({self.dev_expr(e)});")
                elif red is not None and red[0] in self._reds:
                    v, op, e = red
                    out.append(pad + f"rd{v} = rd{v} {op} ({self.dev_expr(e)});")
                else:
                    out.append(pad + f"{self.dev_expr(st.target)} = {self.dev_expr(st.value)};")
            elif st.kind == "loop":
                self.dev_loop(st.loop, ind, out)
            elif st.kind == "call":
                self.dev_region(prog.calls[st.call].subtree, ind, out)
            else:
                raise AssertionError("replaced block inside a kernel")

    # -- module ------------------------------------------------------------------------

    def generate(self) -> tuple[str, str, str]:
        prog = self.prog
        digest = prog.digest()
        hdr = ["#pragma once", '#include "b2o_module.h"', "#include <stdint.h>"]
        for n in self.nests.values():
            if n.kernel:
                hdr.extend(self.kernel_struct(n))
        # device source
        dev = ['#include "app.h"', ""]
        for n in self.nests.values():
            if n.kernel:
                dev.extend(self.kernel_fn(n))
                dev.append("")
        # host source
        host = ["#include <math.h>", "#include <string.h>", '#include "app.h"', ""]
        for v in prog.vars:
            t = self.T(v.id)
            if v.is_array:
                host.append(f"#define A{v.id} (({t} *)ex->host[{v.id}])  /* {v.name} */")
            else:
                host.append(f"#define S{v.id} (*({t} *)ex->host[{v.id}])  /* {v.name} */")
        host.append("")
        for l in prog.loops:
            if not self.device_op[l.id]:
                host.extend(self.fast_fn(l.id))
        for n in self.nests.values():
            if n.kernel:
                host.extend(self.launch_fn(n))
        run = ['extern "C" void b2o_mod_run(b2o_exec *ex) {']
        self.instr_region(prog.root, 1, run)
        run.append("}")
        host.extend(run)
        host.extend(self.info_tables(digest))
        return "\n".join(hdr) + "\n", "\n".join(dev) + "\n", "\n".join(host) + "\n"

    def info_tables(self, digest: str) -> list[str]:
        prog = self.prog
        elem = {"int32_t": 0, "float": 1, "double": 2}
        written = set()
        for st in prog.stmts:
            written |= prog.stmt_access(st)[1]
            if st.kind == "loop":
                written.add(prog.loops[st.loop].index_var)
        for b in list(self.blocks) + list(self.calls.values()):
            written.add(b["out"])
        out = []

        def arr(name, ctype_, items):
            body = ", ".join(str(x) for x in items) if items else "0"
            n = max(len(items), 1)
            out.append(f"static const {ctype_} {name}[{n}] = {{{body}}};")

        def vs(prefix, vals):
            arr(prefix, "int32_t", list(vals))
            return f"{{{len(vals)}, {prefix}}}"

        out.append("static const b2o_var_info VARS[] = {")
        for v in prog.vars:
            out.append(f'  {{"{v.name}", {int(v.is_array)}, {elem[self.T(v.id)]}, {v.length if v.is_array else 1}, '
                       f"{int(v.id in written)}, 0}},")
        out.append("};")
        loop_rows = []
        for l in prog.loops:
            n = self.nests[l.id]
            r = vs(f"LR{l.id}", n.reads)
            w = vs(f"LW{l.id}", n.writes)
            s = vs(f"LS{l.id}", n.swrites)
            kern = f'"{n.kernel}"' if n.kernel else "0"
            why = json.dumps(n.why_not) if n.why_not else "0"
            parent = -1 if l.parent is None else l.parent
            loop_rows.append(f"  {{{kern}, {parent}, {l.index_var}, {len(n.chain)}, {int(self.device_op[l.id])}, "
                             f"{r}, {w}, {s}, {why}}},")
        set_rows, wrow = [], []
        for i, (allv, wv) in enumerate(self.sets):
            set_rows.append("  " + vs(f"SA{i}", allv) + ",")
            wrow.append("  " + vs(f"SW{i}", wv) + ",")
        out.append("static const b2o_loop_info LOOPS[] = {")
        out.extend(loop_rows or ["  {0}"])
        out.append("};")
        out.append("static const b2o_varset SETS[] = {")
        out.extend(set_rows or ["  {0, 0}"])
        out.append("};")
        out.append("static const b2o_varset SETW[] = {")
        out.extend(wrow or ["  {0, 0}"])
        out.append("};")
        outputs = appspec.outputs_of(prog, self.spec)
        out.append("static const b2o_output_info OUTS[] = {")
        for vid, rel, mode in outputs:
            out.append(f"  {{{vid}, {1 if mode == 'normwise' else 0}, {rel!r}}},")
        if not outputs:
            out.append("  {0, 0, 0.0}")
        out.append("};")

        def op_row(b):
            if b is None:
                return "  {-1, 0, 0, 0, 0, 0, 0},"
            op = {"gemm": 0, "fft2d": 1, "histogram": 2}[b["kind"]]
            ins = b["ins"] + [-1, -1]
            return (f"  {{{op}, {b['out']}, {ins[0]}, {ins[1]}, {b.get('m', b.get('n', 0))}, "
                    f"{b.get('n', 0)}, {b.get('k', 0)}}},")

        out.append("static const b2o_op_info BLOCKS[] = {")
        out.extend([op_row(b) for b in self.blocks] or ["  {-1, 0, 0, 0, 0, 0, 0}"])
        out.append("};")
        out.append("static const b2o_op_info CALLS[] = {")
        out.extend([op_row(self.calls.get(c.id)) for c in prog.calls] or ["  {-1, 0, 0, 0, 0, 0, 0}"])
        out.append("};")
        prec = 1 if self.precision == "fp32" else 2
        out.append("static const b2o_module_info INFO = {")
        out.append(f"  B2O_MODULE_ABI, {len(prog.vars)}, {len(prog.loops)}, {len(self.sets)}, {len(outputs)}, "
                   f"{len(self.blocks)}, {len(prog.calls)}, {prec},")
        out.append(f'  VARS, LOOPS, SETS, SETW, OUTS, BLOCKS, CALLS, "{digest}",')
        out.append(f"  {self.exact_slots}, {self.exact_elems()}")
        out.append("};")
        out.append('extern "C" const b2o_module_info *b2o_mod_info(void) { return &INFO; }')
        return out


# ---------------------------------------------------------------------------
# build + cache
# ---------------------------------------------------------------------------


@dataclass
class CompiledApp:
    key: str
    host_so: Path
    cubin: Path
    source_dir: Path
    nests: dict
    n_loops: int


def _spec_key(spec: dict) -> dict:
    """Every spec field that can change the generated program: all of them
    but the input values (initial state, set at load) and the display name.
    (A whitelist silently dropped new kernel-shape options.)"""
    return {k: v for k, v in spec.items() if k not in ("inputs", "name")}


def _host_flags() -> list[str]:
    """ISA level of the generated host C: the widest x86-64 micro-architecture
    level this machine implements (part of the module key, so a module built
    for AVX-512 is never loaded on a host without it), and a higher alias-check
    budget so the long stencil statements of CPU-resident nests vectorise
    (gcc gives up on them at its default of 10 runtime checks).  Element-wise
    vector arithmetic is the scalar arithmetic lane by lane (no contraction,
    no reassociation: -ffp-contract=off, no -ffast-math), so results stay
    bit-identical to the reference's emission."""
    if os.environ.get("B2O_HOST_MARCH"):
        level = os.environ["B2O_HOST_MARCH"]
    else:
        try:
            flags = set()
            for line in Path("/proc/cpuinfo").read_text().splitlines():
                if line.startswith("flags"):
                    flags = set(line.split(":", 1)[1].split())
                    break
        except OSError:
            flags = set()
        if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= flags:
            level = "x86-64-v4"
        elif {"avx2", "fma", "bmi2", "movbe"} <= flags:
            level = "x86-64-v3"
        else:
            level = "x86-64"
    return [f"-march={level}", "--param", "vect-max-version-for-alias-checks=200"]


HOST_FLAGS = _host_flags()


def build_key(doc: dict, spec: dict) -> str:
    blob = json.dumps({"doc": doc, "spec": _spec_key(spec), "v": COMPILER_VERSION, "host": HOST_FLAGS},
                      sort_keys=True)
    return hashlib.sha256(blob.encode()).hexdigest()[:24]


def _run(cmd: list[str], cwd: Path) -> None:
    p = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if p.returncode != 0:
        raise CompileError(f"{cmd[0]} failed ({p.returncode}): {(p.stdout + p.stderr)[-1500:]}")


def compile_program(doc: dict, spec: dict, cache_dir: Path | None = None) -> CompiledApp:
    """Generate and build (or fetch from the cache) one program's module."""
    prog = Program(doc)
    gen = _Gen(prog, spec)
    key = build_key(doc, spec)
    cache = Path(cache_dir or CACHE)
    out_dir = cache / key
    host_so = out_dir / "app_host.so"
    cubin = out_dir / "app.cubin"
    nests = gen.nests
    if host_so.exists() and cubin.exists():
        return CompiledApp(key, host_so, cubin, out_dir, nests, len(prog.loops))
    hdr, dev, host = gen.generate()
    with _lock:
        if host_so.exists() and cubin.exists():
            return CompiledApp(key, host_so, cubin, out_dir, nests, len(prog.loops))
        cache.mkdir(parents=True, exist_ok=True)
        tmp = Path(tempfile.mkdtemp(prefix=f"{key}.", dir=cache))
        (tmp / "app.h").write_text(hdr)
        (tmp / "app_dev.cu").write_text(dev)
        (tmp / "app_host.cpp").write_text(host)
        inc = ["-I", str(CSRC), "-I", str(tmp)]
        fmad = "true" if spec.get("fmad", False) else "false"
        nvcc = os.environ.get("NVCC", "nvcc")
        jobs = [
            ["g++", "-O3", "-std=c++17", "-shared", "-fPIC", "-ffp-contract=off", "-fno-fast-math", *HOST_FLAGS,
             *inc, "app_host.cpp", "-o", "app_host.so"],
            [nvcc, "-cubin", *ARCH_FLAGS, "-O3", "-lineinfo", f"-fmad={fmad}", "-std=c++17", *inc,
             "app_dev.cu", "-o", "app.cubin"],
        ]
        procs = [subprocess.Popen(c, cwd=tmp, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
                 for c in jobs]
        for c, p in zip(jobs, procs):
            text, _ = p.communicate()
            if p.returncode != 0:
                raise CompileError(f"{c[0]} failed ({p.returncode}): {text[-2000:]}")
        try:
            os.replace(tmp, out_dir)
        except OSError:
            # another process won the race; keep theirs
            pass
    return CompiledApp(key, host_so, cubin, out_dir, nests, len(prog.loops))


def generate_sources(doc: dict, spec: dict) -> tuple[str, str, str]:
    """(app.h, app_dev.cu, app_host.cpp) without building; for inspection/tests."""
    return _Gen(Program(doc), spec).generate()
