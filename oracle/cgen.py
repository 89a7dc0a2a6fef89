"""ORACLE — test infrastructure only (tests/, __graft_entry__.smoke(),
bench.py's cpu_baseline leg and ``--impl reference`` arm).

CPU restatement of a whole program in plain C, compiled with gcc, run through
ctypes on numpy buffers.  This is the reference CPU implementation of every
offloaded app: the all-CPU pattern (genome 0...0) executed sequentially with
the C semantics the reference implies (see ``oracle/interp.py`` for the
ledger; the C text mirrors the ``c_openacc`` rendering, ``src/codegen.py:57-68``
and ``:189-200``).  It is pinned against ``oracle/interp.py`` on the small
fixtures and against closed forms (numpy matmul, a direct Himeno formula).
No reference test executes a program, so numeric app outputs are "parity
unpinned" by the reference; what the reference does pin
(placements, plans, screen verdicts) comes from the reference itself.

``openmp=True`` adds ``#pragma omp parallel for`` to the outermost loops that
pass the reference's parallelizability screen (restated from
``src/screen.py:33-79``), for the multi-core CPU baseline.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
import tempfile
from pathlib import Path

import numpy as np

CACHE = Path(__file__).resolve().parent / "_build"

EXT_FN = ctypes.CFUNCTYPE(None, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p))


def _ctype(base: str, precision: str) -> str:
    if base == "int":
        return "int"
    return "float" if precision == "fp32" else "double"


class _Gen:
    def __init__(self, doc: dict, precision: str, openmp: bool):
        self.doc = doc
        self.precision = precision
        self.openmp = openmp
        self.vars = {v["id"]: v for v in doc["variables"]}
        self.regions = {r["id"]: r for r in doc["regions"]}
        self.loops = {l["id"]: l for l in doc["loops"]}
        self.calls = {c["id"]: c for c in doc["calls"]}
        self.lines: list[str] = []
        self.ext_sites: list[tuple] = []

    # -- expressions ----------------------------------------------------------

    def name(self, vid: int) -> str:
        return f"v{vid}"

    def expr(self, e) -> str:
        if "num" in e:
            v = e["num"]
            if e.get("float", False):
                s = repr(float(v))
                return f"({s})" if float(v) < 0 else s
            return f"({int(v)})" if int(v) < 0 else str(int(v))
        if "var" in e:
            return self.name(e["var"])
        if "array" in e:
            return f"{self.name(e['array'])}[{self.expr(e['index'])}]"
        return f"({self.expr(e['left'])} {e['op']} {self.expr(e['right'])})"

    def etype(self, e) -> str:
        if "num" in e:
            return "double" if e.get("float", False) else "int"
        if "var" in e or "array" in e:
            vid = e.get("var", e.get("array"))
            return _ctype(self.vars[vid]["type"], self.precision)
        a, b = self.etype(e["left"]), self.etype(e["right"])
        for t in ("double", "float"):
            if t in (a, b):
                return t
        return "int"

    # -- screen restatement (src/screen.py:33-79) ------------------------------

    def _subtree(self, lid: int):
        out = [self.loops[lid]["body"]]
        stack = [self.loops[lid]["body"]]
        loops = [lid]
        while stack:
            rid = stack.pop()
            for s in self.regions[rid]["statements"]:
                if "loop" in s:
                    loops.append(s["loop"])
                    out.append(self.loops[s["loop"]]["body"])
                    stack.append(self.loops[s["loop"]]["body"])
                elif "call" in s:
                    out.append(self.calls[s["call"]]["subtree"])
                    stack.append(self.calls[s["call"]]["subtree"])
        return out, loops

    def parallelizable(self, lid: int) -> bool:
        regions, loops = self._subtree(lid)
        rs = set(regions)
        exempt = {self.loops[x]["index_var"] for x in loops}
        reads, sets = set(), set()
        for o in self.doc["occurrences"]:
            if o["region"] not in rs or self.vars[o["var"]]["array"] or o["var"] in exempt:
                continue
            (reads if o["kind"] == "read" else sets if o["kind"] == "set" else set()).add(o["var"])
        if reads & sets:
            return False
        iv = self.loops[lid]["index_var"]
        for rid in regions:
            for s in self.regions[rid]["statements"]:
                if "assign" in s and "array" in s["assign"]:
                    if iv not in _expr_vars(s["assign"]["index"]):
                        return False
                if "call" in s and not self.calls[s["call"]]["pure"]:
                    return False
                if "replaced" in s:
                    return False
        for x in loops:  # bounds must be loop-invariant ints for OpenMP
            l = self.loops[x]
            if self.etype(l["lower"]) != "int" or self.etype(l["upper"]) != "int":
                return False
        return True

    def _written_scalars(self, lid: int) -> list[int]:
        regions, loops = self._subtree(lid)
        out = {self.loops[x]["index_var"] for x in loops}
        for rid in regions:
            for s in self.regions[rid]["statements"]:
                if "assign" in s and "var" in s["assign"]:
                    out.add(s["assign"]["var"])
        return sorted(out)

    # -- statements ---------------------------------------------------------------

    def emit(self, ind: int, text: str) -> None:
        self.lines.append("  " * ind + text)

    def region(self, rid: int, ind: int, in_parallel: bool) -> None:
        for idx, s in enumerate(self.regions[rid]["statements"]):
            if "decl" in s:
                if "init" in s:
                    self.emit(ind, f"{self.name(s['decl'])} = {self.expr(s['init'])};")
            elif "assign" in s:
                self.emit(ind, f"{self.expr(s['assign'])} = {self.expr(s['value'])};")
            elif "loop" in s:
                self.loop(s["loop"], ind, in_parallel)
            elif "call" in s:
                c = self.calls[s["call"]]
                if self.regions[c["subtree"]]["statements"]:
                    self.region(c["subtree"], ind, in_parallel)
                else:
                    self.external(ind, 0, c["id"])
            else:
                self.ext_sites.append((rid, idx))
                self.external(ind, 1, len(self.ext_sites) - 1)

    def external(self, ind: int, kind: int, ident: int) -> None:
        self.emit(ind, "SAVE_SCALARS();")
        self.emit(ind, f"ext({kind}, {ident}, slots);")
        self.emit(ind, "LOAD_SCALARS();")

    def loop(self, lid: int, ind: int, in_parallel: bool) -> None:
        l = self.loops[lid]
        iv = self.name(l["index_var"])
        par = self.openmp and not in_parallel and self.parallelizable(lid)
        if par:
            priv = ", ".join(self.name(v) for v in self._written_scalars(lid))
            self.emit(ind, f"#pragma omp parallel for schedule(static) lastprivate({priv})")
        self.emit(ind, f"for ({iv} = {self.expr(l['lower'])}; {iv} < {self.expr(l['upper'])}; {iv}++) {{")
        self.region(l["body"], ind + 1, in_parallel or par)
        self.emit(ind, "}")

    def generate(self) -> str:
        arrays = [v for v in self.vars.values() if v["array"]]
        scalars = [v for v in self.vars.values() if not v["array"]]
        out = ["#include <stdint.h>", "typedef void (*ext_fn)(int, int, void **);"]
        body_lines = self.lines
        self.region(self.doc.get("root_region", 0), 1, False)
        save = " ".join(f"*({_ctype(v['type'], self.precision)} *)slots[{v['id']}] = {self.name(v['id'])};"
                        for v in scalars)
        load = " ".join(f"{self.name(v['id'])} = *({_ctype(v['type'], self.precision)} *)slots[{v['id']}];"
                        for v in scalars)
        out.append(f"#define SAVE_SCALARS() do {{ {save} }} while (0)")
        out.append(f"#define LOAD_SCALARS() do {{ {load} }} while (0)")
        out.append("void oracle_run(void **slots, ext_fn ext) {")
        for v in arrays:
            t = _ctype(v["type"], self.precision)
            out.append(f"  {t} *restrict {self.name(v['id'])} = ({t} *)slots[{v['id']}];  /* {v['name']} */")
        for v in scalars:
            out.append(f"  {_ctype(v['type'], self.precision)} {self.name(v['id'])};  /* {v['name']} */")
        out.append("  (void)ext;")
        out.append("  LOAD_SCALARS();")
        out.extend(body_lines)
        out.append("  SAVE_SCALARS();")
        out.append("}")
        return "\n".join(out) + "\n"


def _expr_vars(e) -> list[int]:
    if "var" in e:
        return [e["var"]]
    if "array" in e:
        return [e["array"]] + _expr_vars(e["index"])
    if "op" in e:
        return _expr_vars(e["left"]) + _expr_vars(e["right"])
    return []


def generate_c(doc: dict, precision: str = "fp32", openmp: bool = False) -> tuple[str, list]:
    g = _Gen(doc, precision, openmp)
    return g.generate(), g.ext_sites


class CProgram:
    """A compiled C restatement of one program."""

    def __init__(self, doc: dict, precision: str = "fp32", openmp: bool = False, opt: str = "-O2"):
        self.doc = doc
        self.precision = precision
        src, self.ext_sites = generate_c(doc, precision, openmp)
        key = hashlib.sha256((src + opt + str(openmp)).encode()).hexdigest()[:20]
        CACHE.mkdir(parents=True, exist_ok=True)
        so = CACHE / f"oracle_{key}.so"
        if not so.exists():
            with tempfile.TemporaryDirectory() as td:
                c = Path(td) / "prog.c"
                c.write_text(src)
                tmp = Path(td) / "prog.so"
                cmd = ["gcc", opt, "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
                       str(c), "-o", str(tmp)]
                if openmp:
                    cmd.insert(1, "-fopenmp")
                subprocess.run(cmd, check=True, capture_output=True, text=True)
                os.replace(tmp, so)
        self.lib = ctypes.CDLL(str(so))
        self.fn = self.lib.oracle_run
        self.fn.argtypes = [ctypes.POINTER(ctypes.c_void_p), EXT_FN]
        self.fn.restype = None

    def run(self, state: dict[int, np.ndarray], binder=None, copy: bool = True) -> dict[int, np.ndarray]:
        st = {k: (v.copy() if copy else v) for k, v in state.items()}
        n = len(self.doc["variables"])
        slots = (ctypes.c_void_p * n)(*[st[i].ctypes.data for i in range(n)])
        calls = {c["id"]: c for c in self.doc["calls"]}
        stmts = {r["id"]: r["statements"] for r in self.doc["regions"]}

        def ext(kind, ident, _slots):
            if binder is None:
                raise RuntimeError("program calls an external without a binder")
            if kind == 0:
                binder("call", calls[ident], st)
            else:
                rid, idx = self.ext_sites[ident]
                s = stmts[rid][idx]
                binder("replaced", {"name": s["replaced"], "args": s["args"], "rid": rid, "index": idx}, st)

        errors: list[BaseException] = []

        def guarded(kind, ident, _slots):
            try:
                ext(kind, ident, _slots)
            except BaseException as exc:  # noqa: BLE001 -- ctypes would swallow it
                errors.append(exc)

        cb = EXT_FN(guarded)
        self.fn(slots, cb)
        if errors:
            raise RuntimeError(f"external call failed inside the oracle program: {errors[0]!r}") from errors[0]
        return st
