"""ORACLE — test infrastructure only (imported by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg; never by the product package).

Pure-Python interpreter of a program in the reference IR document format,
with C semantics.  It is the oracle-of-the-oracle: slow, obviously-correct,
used on small fixtures to pin the C restatement in ``oracle/cgen.py``.

Parity status: the reference never executes programs, so no
reference test pins numeric app outputs ("parity unpinned" for app values).
What *is* pinned against the reference: the program structure, the gene
encoding, placements and transfer plans (tests/golden/*.json are produced by
the reference itself, tests/golden/make_golden.py).  The semantics restated
here are the ones the reference implies:

* statements / expressions: ``src/model.py:45-211``; loop headers
  ``for (i = lower; i < upper; i++)`` re-evaluate ``upper`` every iteration,
  as the C rendering ``src/codegen.py:189-200`` does;
* C usual arithmetic conversions (the ``c_openacc`` rendering is C,
  ``src/codegen.py:57-68``): ``int op int`` is 32-bit int with truncating
  division, a float literal (``Num.is_float``) is a C ``double``, model
  ``float`` is C ``float`` in fp32 mode and ``double`` in fp64 mode;
* declarations are file-scope: zero-initialised, initialisers run in order
  (``src/build.py:83-87``);
* opaque calls / replaced blocks follow the app-spec binding (Appendix A.5).
"""

from __future__ import annotations

import numpy as np

INT, FLT, DBL = "int", "float", "double"


def _wrap32(x: int) -> int:
    return ((x + 0x80000000) & 0xFFFFFFFF) - 0x80000000


class Interpreter:
    def __init__(self, doc: dict, state: dict[int, np.ndarray], precision: str = "fp32",
                 externals=None, max_steps: int = 50_000_000):
        self.doc = doc
        self.vars = {v["id"]: v for v in doc["variables"]}
        self.regions = {r["id"]: r for r in doc["regions"]}
        self.loops = {l["id"]: l for l in doc["loops"]}
        self.calls = {c["id"]: c for c in doc["calls"]}
        self.state = state
        self.ftype = np.float32 if precision == "fp32" else np.float64
        self.float_ctype = FLT if precision == "fp32" else DBL
        self.externals = externals  # callable(kind_desc, stmt_or_call, state)
        self.steps = 0
        self.max_steps = max_steps

    # -- values -------------------------------------------------------------

    def _vtype(self, vid: int) -> str:
        return INT if self.vars[vid]["type"] == "int" else self.float_ctype

    def _conv(self, value, src: str, dst: str):
        if dst == INT:
            if src == INT:
                return value
            return _wrap32(int(value))  # C truncation toward zero
        if dst == FLT:
            return np.float32(value)
        return float(value)

    def eval(self, e) -> tuple[object, str]:
        if "num" in e:
            if e.get("float", False):
                return float(e["num"]), DBL
            return int(e["num"]), INT
        if "var" in e:
            vid = e["var"]
            return self.state[vid][0].item() if self._vtype(vid) != FLT else self.state[vid][0], self._vtype(vid)
        if "array" in e:
            idx, it = self.eval(e["index"])
            if it != INT:
                raise TypeError("array index must be an int expression")
            arr = self.state[e["array"]]
            if not 0 <= idx < arr.shape[0]:
                raise IndexError(f"index {idx} out of bounds for {self.vars[e['array']]['name']}")
            t = self._vtype(e["array"])
            v = arr[idx]
            return (v if t == FLT else v.item()), t
        a, ta = self.eval(e["left"])
        b, tb = self.eval(e["right"])
        op = e["op"]
        if DBL in (ta, tb):
            t = DBL
        elif FLT in (ta, tb):
            t = FLT
        else:
            t = INT
        a = self._conv(a, ta, t)
        b = self._conv(b, tb, t)
        if t == INT:
            if op == "+":
                r = a + b
            elif op == "-":
                r = a - b
            elif op == "*":
                r = a * b
            else:
                if b == 0:
                    raise ZeroDivisionError("integer division by zero")
                q = abs(a) // abs(b)
                r = q if (a >= 0) == (b >= 0) else -q
            return _wrap32(r), INT
        if op == "+":
            r = a + b
        elif op == "-":
            r = a - b
        elif op == "*":
            r = a * b
        else:
            r = a / b
        return (np.float32(r) if t == FLT else float(r)), t

    def _store(self, target, value, vtype):
        vid = target["var"] if "var" in target else target["array"]
        t = self._vtype(vid)
        v = self._conv(value, vtype, t)
        if "var" in target:
            self.state[vid][0] = v
        else:
            idx, it = self.eval(target["index"])
            arr = self.state[vid]
            if it != INT or not 0 <= idx < arr.shape[0]:
                raise IndexError(f"bad store index {idx} for {self.vars[vid]['name']}")
            arr[idx] = v

    # -- statements -----------------------------------------------------------

    def run(self) -> dict[int, np.ndarray]:
        self.region(self.doc.get("root_region", 0))
        return self.state

    def region(self, rid: int) -> None:
        for idx, s in enumerate(self.regions[rid]["statements"]):
            self.steps += 1
            if self.steps > self.max_steps:
                raise RuntimeError("interpreter step budget exceeded")
            if "decl" in s:
                if "init" in s:
                    v, t = self.eval(s["init"])
                    self._store({"var": s["decl"]}, v, t)
            elif "assign" in s:
                v, t = self.eval(s["value"])
                self._store(s["assign"], v, t)
            elif "loop" in s:
                self.loop(s["loop"])
            elif "call" in s:
                c = self.calls[s["call"]]
                if self.regions[c["subtree"]]["statements"]:
                    self.region(c["subtree"])
                else:
                    if self.externals is None:
                        raise RuntimeError(f"opaque call {c['name']!r} without a binding")
                    self.externals("call", c, self.state)
            else:
                if self.externals is None:
                    raise RuntimeError(f"replaced block {s['replaced']!r} without a binding")
                self.externals("replaced", {"name": s["replaced"], "args": s["args"], "rid": rid,
                                            "index": idx}, self.state)

    def loop(self, lid: int) -> None:
        l = self.loops[lid]
        iv = l["index_var"]
        v, t = self.eval(l["lower"])
        self._store({"var": iv}, v, t)
        while True:
            cur, ct = self.eval({"var": iv})
            hi, ht = self.eval(l["upper"])
            tt = DBL if DBL in (ct, ht) else (FLT if FLT in (ct, ht) else INT)
            if not (self._conv(cur, ct, tt) < self._conv(hi, ht, tt)):
                break
            self.region(l["body"])
            cur, ct = self.eval({"var": iv})
            r, rt = self.eval({"op": "+", "left": {"var": iv}, "right": {"num": 1, "float": False}})
            self._store({"var": iv}, r, rt)


def run_program(doc: dict, state: dict[int, np.ndarray], precision: str = "fp32", externals=None):
    """Execute ``doc`` on a copy of ``state``; returns the final state."""
    st = {k: v.copy() for k, v in state.items()}
    return Interpreter(doc, st, precision, externals).run()
