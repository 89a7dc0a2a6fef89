"""ORACLE — test infrastructure only (tests/, __graft_entry__.build()/smoke()
and bench.py's cpu_baseline leg and ``--impl reference`` arm; never imported by
the product package).

``oracle/_ref``: the reference's OWN C text for a program, compiled with gcc
and executed.  The reference renders every program it analyses as C
(``gpuoffload.codegen.pretty_print``, src/gpuoffload/codegen.py:230-232; an
annotated ``c_openacc`` emission for a pattern, ``emit_annotated``,
codegen.py:235-247; expression rendering and precedence codegen.py:57-68; loop
headers codegen.py:182-200).  This module asks the reference for that text,
writes it verbatim into ``oracle/_ref/ref_<key>.c`` behind a forced-include
prelude (``oracle/ref_prelude.h``: ``func`` -> ``void``, ``main`` renamed, opaque
calls routed to a callback), compiles it with ``gcc -O2 -ffp-contract=off``
into ``oracle/_ref/ref_<key>.so`` and runs it through ctypes, injecting the
app's inputs into the file-scope globals the reference declares
(codegen.py:141-160) and reading every variable back by name.

This is what pins the C restatement (``oracle/cgen.py``) and, through it, the
GPU path to the reference: ``tests/test_refc.py`` checks the two bit for bit
on every golden app, the committed fuzz programs and Himeno M.

Semantics the reference's text leaves to the C compiler, fixed identically in
both oracles: ``float`` is C ``float`` (fp32 apps) or ``double``
(``precision: fp64``, ``-Dfloat=double``); ``int`` is C ``int``; declaration
initialisers are C static initialisers (the value at program start, which is
what ``oracle/cgen.py`` assigns first); everything else starts at the app
spec's input or zero (C file scope).  Opaque calls / replaced blocks get the
app spec's CPU semantics (``oracle/externals.py``), exactly as in cgen.

Two flavours:

* ``RefProgram.build(doc, precision)``: ``pretty_print`` of the program
  (sequential; the parity oracle);
* ``RefProgram.build(doc, precision, pattern=record, openmp=True)``: the
  reference's ``emit_annotated(..., "c_openacc")`` text for one pattern, with
  ``#pragma omp parallel for`` inserted under each ``#pragma acc kernels`` /
  ``#pragma acc parallel loop`` line (the loops the reference offloads; every
  index variable and written scalar of the nest ``lastprivate``, the
  reference's lastprivate-free C being sequential) -- the reference's own
  program run on every host core (bench.py's reference arm).  Acc data
  pragmas stay in the text; gcc ignores them.

Build needs the reference importable (``/root/reference`` here, or the
installed copy in ``baseline/_ref``); running a built ``.so`` needs only its
``.json`` sidecar, so ``oracle/_ref`` built here also works on the GPU box.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
OUT = HERE / "_ref"
PRELUDE = HERE / "ref_prelude.h"
EXT_FN = ctypes.CFUNCTYPE(None, ctypes.c_int)
CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fno-builtin", "-w", "-shared", "-fPIC",
          "-mcmodel=medium"]


def _baseline_flags() -> list[str]:
    """The CPU-baseline build (``openmp=True``, the bench's reference arm):
    as strong as the product's own host build (paper_2011_03602_b200/compiler.py
    ``_host_flags``) -- -O3 at the widest x86-64 level this machine implements,
    with the alias-check budget that lets the long stencil statements
    vectorise -- so the GPU is not compared with a handicapped CPU.  The
    parity builds keep plain -O2 (results are identical either way: no
    contraction, no reassociation)."""
    flags = set()
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("flags"):
                flags = set(line.split(":", 1)[1].split())
                break
    except OSError:
        pass
    if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= flags:
        level = "x86-64-v4"
    elif {"avx2", "fma", "bmi2", "movbe"} <= flags:
        level = "x86-64-v3"
    else:
        level = "x86-64"
    return ["-O3", f"-march={level}", "--param", "vect-max-version-for-alias-checks=200"]


BASELINE_FLAGS = _baseline_flags()


class RefUnavailable(RuntimeError):
    """The reference package is not importable (needed only to emit text)."""


def _reference():
    try:
        from gpuoffload import codegen, irdoc, patterns, transfers  # noqa: F401
    except ImportError:
        for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
            if p.exists() and str(p) not in sys.path:
                sys.path.append(str(p))
        try:
            from gpuoffload import codegen, irdoc, patterns, transfers  # noqa: F401
        except ImportError as exc:
            raise RefUnavailable(f"reference package not importable: {exc}") from exc
    from gpuoffload import codegen, irdoc, patterns, transfers

    return codegen, irdoc, patterns, transfers


# ---------------------------------------------------------------------------
# emission (needs the reference)
# ---------------------------------------------------------------------------


def _sites(doc: dict) -> list[dict]:
    """Opaque call / replaced-block statements in the order the reference's
    emitter visits them (codegen.py:137-180: root region, loop bodies,
    inlined call subtrees), i.e. the order their ``name(args);`` lines
    appear in the text and hence their ``__COUNTER__`` ordinals."""
    regions = {r["id"]: r for r in doc["regions"]}
    loops = {l["id"]: l for l in doc["loops"]}
    calls = {c["id"]: c for c in doc["calls"]}
    out: list[dict] = []

    def walk(rid: int) -> None:
        for idx, s in enumerate(regions[rid]["statements"]):
            if "loop" in s:
                walk(loops[s["loop"]]["body"])
            elif "call" in s:
                c = calls[s["call"]]
                if regions[c["subtree"]]["statements"]:
                    walk(c["subtree"])
                else:
                    out.append({"kind": "call", "call": c["id"], "name": c["name"], "arg_vars": list(c["arg_vars"])})
            elif "replaced" in s:
                out.append({"kind": "replaced", "name": s["replaced"], "args": list(s["args"]), "rid": rid,
                            "index": idx})

    walk(doc.get("root_region", 0))
    return out


def _walk_loops(doc: dict) -> list[int]:
    """Loop ids in emission order."""
    regions = {r["id"]: r for r in doc["regions"]}
    loops = {l["id"]: l for l in doc["loops"]}
    calls = {c["id"]: c for c in doc["calls"]}
    out: list[int] = []

    def walk(rid: int) -> None:
        for s in regions[rid]["statements"]:
            if "loop" in s:
                out.append(s["loop"])
                walk(loops[s["loop"]]["body"])
            elif "call" in s:
                walk(calls[s["call"]]["subtree"])

    walk(doc.get("root_region", 0))
    return out


def _nest_lastprivate(doc: dict, root: int) -> list[str] | None:
    """Names of the index variables and assigned scalars of a nest, or None
    when OpenMP cannot take the loop (non-int bounds)."""
    regions = {r["id"]: r for r in doc["regions"]}
    loops = {l["id"]: l for l in doc["loops"]}
    calls = {c["id"]: c for c in doc["calls"]}
    vars_ = {v["id"]: v for v in doc["variables"]}

    def int_expr(e) -> bool:
        if "num" in e:
            return not e.get("float", False)
        if "var" in e or "array" in e:
            return vars_[e.get("var", e.get("array"))]["type"] == "int"
        return int_expr(e["left"]) and int_expr(e["right"])

    names: set[int] = set()
    stack = [root]
    while stack:
        lid = stack.pop()
        l = loops[lid]
        if not (int_expr(l["lower"]) and int_expr(l["upper"])):
            return None
        names.add(l["index_var"])
        rs = [l["body"]]
        while rs:
            rid = rs.pop()
            for s in regions[rid]["statements"]:
                if "loop" in s:
                    stack.append(s["loop"])
                elif "assign" in s and "var" in s["assign"]:
                    names.add(s["assign"]["var"])
                elif "call" in s:
                    rs.append(calls[s["call"]]["subtree"])
    return sorted(vars_[v]["name"] for v in names)


def emit(doc: dict, pattern: dict | None = None, genome_loops=None) -> str:
    """The reference's C text: ``pretty_print(model)`` or, for a pattern
    record (tests/golden ``patterns[genome]``), ``emit_annotated(model,
    pattern, plan_transfers(model, pattern), "c_openacc")``."""
    codegen, irdoc, patterns, transfers = _reference()
    model = irdoc.load_ir_document(json.dumps(doc))
    if pattern is None:
        return codegen.pretty_print(model)
    bits = tuple(int(c) for c in pattern["genome"])
    placements = {int(k): v for k, v in pattern["placements"].items()}
    pat = patterns.OffloadPattern(bits, tuple(genome_loops or ()), placements, tuple(pattern["gpu_roots"]))
    plan = transfers.plan_transfers(model, pat)
    return codegen.emit_annotated(model, pat, plan, codegen.C_OPENACC)


def _omp(doc: dict, text: str, gpu_roots) -> str:
    roots = [l for l in _walk_loops(doc) if l in set(gpu_roots)]
    out, k = [], 0
    for ln in text.splitlines():
        out.append(ln)
        s = ln.strip()
        if s in ("#pragma acc kernels", "#pragma acc parallel loop"):
            priv = _nest_lastprivate(doc, roots[k])
            k += 1
            if priv is not None:
                ind = ln[: len(ln) - len(ln.lstrip())]
                out.append(f"{ind}#pragma omp parallel for schedule(static) lastprivate({', '.join(priv)})")
    if k != len(roots):
        raise RuntimeError(f"{k} acc compute pragmas for {len(roots)} GPU roots")
    return "\n".join(out) + "\n"


def source(doc: dict, precision: str = "fp32", pattern: dict | None = None, openmp: bool = False,
           genome_loops=None) -> tuple[str, dict]:
    """(C file text, sidecar meta) for one program."""
    text = emit(doc, pattern, genome_loops)
    if openmp:
        if pattern is None:
            raise ValueError("the OpenMP flavour maps a pattern's acc pragmas")
        text = _omp(doc, text, pattern["gpu_roots"])
    sites = _sites(doc)
    macros = []
    for name in sorted({s["name"] for s in sites}):
        macros.append(f"#define {name}(...) (b2o_ref_ext(__COUNTER__))")
    head = ["/* ORACLE (test infrastructure): the reference's own emission follows verbatim",
            " * (gpuoffload.codegen." + ("emit_annotated c_openacc" if pattern else "pretty_print") + ")"
            + (", #pragma omp lines added under its acc compute pragmas" if openmp else "") + ". */"]
    c = "\n".join(head + macros + ['#line 1 "reference-emission"', text])
    meta = {
        "precision": precision,
        "openmp": openmp,
        "variables": [{"id": v["id"], "name": v["name"], "type": v["type"], "array": v["array"],
                       "length": v["length"]} for v in doc["variables"]],
        "static_init": sorted(s["decl"] for s in
                              next(r for r in doc["regions"] if r["id"] == doc.get("root_region", 0))["statements"]
                              if "decl" in s and "init" in s),
        "sites": sites,
    }
    return c, meta


def key_of(c: str, precision: str, openmp: bool) -> str:
    return hashlib.sha256((c + precision + str(openmp) + " ".join(CFLAGS)
                           + (" ".join(BASELINE_FLAGS) if openmp else "")
                           + PRELUDE.read_text()).encode()).hexdigest()[:20]


def build(doc: dict, precision: str = "fp32", pattern: dict | None = None, openmp: bool = False,
          genome_loops=None) -> Path:
    """Emit (reference), write ``oracle/_ref/ref_<key>.{c,json}``, compile the
    ``.so``; returns the ``.so`` path.  Cached by content."""
    c, meta = source(doc, precision, pattern, openmp, genome_loops)
    key = key_of(c, precision, openmp)
    OUT.mkdir(parents=True, exist_ok=True)
    so = OUT / f"ref_{key}.so"
    if not so.exists():
        (OUT / f"ref_{key}.c").write_text(c)
        (OUT / f"ref_{key}.json").write_text(json.dumps(meta))
        with tempfile.TemporaryDirectory() as td:
            tmp = Path(td) / "ref.so"
            cmd = ["gcc", *CFLAGS, "-include", str(PRELUDE), "-Dmain=b2o_ref_main"]
            if precision == "fp64":
                cmd.append("-Dfloat=double")
            if openmp:
                cmd += ["-fopenmp", *BASELINE_FLAGS]
            cmd += [str(OUT / f"ref_{key}.c"), "-o", str(tmp)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"gcc rejected the reference emission ({OUT / f'ref_{key}.c'}):\n{r.stderr[-2000:]}")
            os.replace(tmp, so)
    # a program's index: doc hash -> .so, so a box without the reference can
    # find the prebuilt object for a golden document
    idx = OUT / "index.json"
    table = json.loads(idx.read_text()) if idx.exists() else {}
    dk = doc_key(doc, precision, pattern, openmp)
    if table.get(dk) != so.name:
        table[dk] = so.name
        tmpi = idx.with_suffix(f".{os.getpid()}.tmp")
        tmpi.write_text(json.dumps(table, sort_keys=True))
        os.replace(tmpi, idx)
    return so


def doc_key(doc: dict, precision: str, pattern: dict | None, openmp: bool) -> str:
    g = pattern["genome"] if pattern else ""
    return hashlib.sha256((json.dumps(doc, sort_keys=True) + precision + g + str(openmp)).encode()).hexdigest()[:24]


def prebuilt(doc: dict, precision: str = "fp32", pattern: dict | None = None, openmp: bool = False) -> Path | None:
    idx = OUT / "index.json"
    if not idx.exists():
        return None
    name = json.loads(idx.read_text()).get(doc_key(doc, precision, pattern, openmp))
    return OUT / name if name and (OUT / name).exists() else None


# ---------------------------------------------------------------------------
# execution (needs only the built .so and its sidecar)
# ---------------------------------------------------------------------------


def _np_type(t: str, precision: str):
    if t == "int":
        return np.int32
    return np.float32 if precision == "fp32" else np.float64


_LOADED: dict[str, list] = {}


class RefProgram:
    """A compiled reference emission.  ``run(state)`` injects the state into
    the program's globals, calls the entry and returns every variable."""

    def __init__(self, so: Path | str):
        so = Path(so)
        self.meta = json.loads(so.with_suffix(".json").read_text())
        # dlopen hands every RefProgram of one path the same globals: the
        # start values of initialised declarations are snapshotted at the
        # first load in this process, before anything ran
        first = str(so) not in _LOADED
        if first:
            _LOADED[str(so)] = [ctypes.CDLL(str(so), mode=ctypes.RTLD_LOCAL), None]
        self.lib = _LOADED[str(so)][0]
        self.entry = self.lib.b2o_ref_main
        self.entry.argtypes = []
        self.entry.restype = None
        prec = self.meta["precision"]
        self.views: dict[int, np.ndarray] = {}
        for v in self.meta["variables"]:
            dt = _np_type(v["type"], prec)
            n = v["length"] if v["array"] else 1
            ct = {np.int32: ctypes.c_int32, np.float32: ctypes.c_float, np.float64: ctypes.c_double}[dt]
            buf = (ct * n).in_dll(self.lib, v["name"])
            self.views[v["id"]] = np.ctypeslib.as_array(buf)
        # value of initialised declarations at program start (C static init)
        if first:
            _LOADED[str(so)][1] = {vid: self.views[vid].copy() for vid in self.meta["static_init"]}
        self.static = _LOADED[str(so)][1]
        self._cb = None
        self._errors: list[BaseException] = []

    @classmethod
    def build(cls, doc: dict, precision: str = "fp32", pattern: dict | None = None, openmp: bool = False,
              genome_loops=None) -> "RefProgram":
        so = prebuilt(doc, precision, pattern, openmp)
        if so is None:
            so = build(doc, precision, pattern, openmp, genome_loops)
        return cls(so)

    def load(self, state: dict[int, np.ndarray], binder=None) -> None:
        """Untimed: write the program's start state into its globals."""
        for vid, view in self.views.items():
            src = self.static.get(vid)
            if src is None:
                src = np.asarray(state[vid]).reshape(-1)
            view[:] = src.astype(view.dtype, copy=False)
        sites = self.meta["sites"]
        if sites:
            if binder is None:
                raise RuntimeError("program calls an external without a binder")
            views = self.views

            def ext(site: int) -> None:
                try:
                    _ext(site)
                except BaseException as exc:  # noqa: BLE001 -- ctypes would swallow it
                    self._errors.append(exc)

            def _ext(site: int) -> None:
                s = sites[site]
                if s["kind"] == "call":
                    binder("call", {"id": s["call"], "name": s["name"], "arg_vars": s["arg_vars"]}, views)
                else:
                    binder("replaced", {"name": s["name"], "args": s["args"], "rid": s["rid"], "index": s["index"]},
                           views)

            self._cb = EXT_FN(ext)
            ctypes.c_void_p.in_dll(self.lib, "b2o_ref_ext").value = ctypes.cast(self._cb, ctypes.c_void_p).value

    def execute(self) -> None:
        """Timed part: the program itself."""
        self._errors.clear()
        self.entry()
        if self._errors:
            raise RuntimeError(f"external call failed inside the reference program: {self._errors[0]!r}") \
                from self._errors[0]

    def result(self) -> dict[int, np.ndarray]:
        return {vid: v.copy() for vid, v in self.views.items()}

    def run(self, state: dict[int, np.ndarray], binder=None) -> dict[int, np.ndarray]:
        self.load(state, binder)
        self.execute()
        return self.result()


# ---------------------------------------------------------------------------
# prebuild (build container): every golden program the GPU suites check
# ---------------------------------------------------------------------------


def golden_programs(golden_dir: Path) -> list[tuple[dict, str]]:
    """(doc, precision) of every committed golden program (apps, block
    variants, fuzz programs, the fp64 builds)."""
    items: list[tuple[dict, str]] = []
    for f in sorted(golden_dir.glob("*.json")):
        g = json.loads(f.read_text())
        if f.name in ("fuzz.json", "fuzz_shapes.json"):
            items += [(r["doc"], r["spec"].get("precision", "fp32")) for r in g.values()]
        elif "doc" in g:
            items.append((g["doc"], g["spec"].get("precision", "fp32")))
        else:
            items += [(v["doc"], g["spec"].get("precision", "fp32")) for v in g["variants"]]
    fuzz = json.loads((golden_dir / "fuzz.json").read_text())
    items += [(fuzz[k]["doc"], "fp64") for k in sorted(fuzz, key=int)[:16]]
    for a in ("four_loops", "nest2d", "stencil", "triple_nest", "himeno_xs_inline", "himeno_17x9x33", "matmul_48",
              "nasmg_18", "himeno_M"):
        items.append((json.loads((golden_dir / f"{a}.json").read_text())["doc"], "fp64"))
    return items


BENCH_PATTERNS = [("himeno_M", "100100"), ("matmul_1024", "10"), ("nasmg_258", "100100"), ("himeno_17x9x33", "100100")]


def _build_item(item) -> str:
    doc, prec = item
    return build(doc, prec).name


def prebuild(golden_dir: Path, workers: int = 8) -> int:
    """Compile the reference emission of every golden program into
    oracle/_ref (needs the reference importable; the objects travel to the
    GPU box, where tests load them by document hash)."""
    from concurrent.futures import ProcessPoolExecutor

    _reference()
    items = golden_programs(golden_dir)
    with ProcessPoolExecutor(max(1, workers)) as pool:
        names = list(pool.map(_build_item, items, chunksize=4))
    # the index is rewritten by each worker; rebuild it in one place
    table = {doc_key(doc, prec, None, False): name for (doc, prec), name in zip(items, names)}
    # bench.py's CPU arms: the annotated emission of the benchmarked pattern,
    # acc nests as OpenMP
    for app, genome in BENCH_PATTERNS:
        g = json.loads((golden_dir / f"{app}.json").read_text())
        pat = g["patterns"][genome]
        so = build(g["doc"], "fp32", pattern=pat, openmp=True, genome_loops=g["genome_loops"])
        table[doc_key(g["doc"], "fp32", pat, True)] = so.name
    idx = OUT / "index.json"
    old = json.loads(idx.read_text()) if idx.exists() else {}
    old.update(table)
    idx.write_text(json.dumps(old, sort_keys=True))
    return len(items)


def reference_state(doc: dict, spec: dict, state: dict, binder=None) -> tuple[dict, str]:
    """Final state of the program by the reference's own emission when it is
    prebuilt (or buildable here), else by the C restatement (pinned to it
    bit for bit by tests/test_refc.py).  Returns (state, which)."""
    prec = spec.get("precision", "fp32")
    so = prebuilt(doc, prec)
    if so is None:
        try:
            so = build(doc, prec)
        except RefUnavailable:
            so = None
    if so is not None:
        return RefProgram(so).run(state, binder), "reference emission (oracle/_ref)"
    from oracle.cgen import CProgram

    return CProgram(doc, prec).run(state, binder), "C restatement (oracle/cgen.py)"
