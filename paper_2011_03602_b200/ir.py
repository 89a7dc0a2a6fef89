"""Read-only view of a program in the reference's IR document format.

The evaluator receives live ``gpuoffload.model.ProgramModel`` objects from the
reference GA; it serialises them once with the reference's own
``irdoc.model_to_document`` (``src/irdoc.py:95-166``) and every stage of this
package (compiler, analysis, tests, and the CPU oracle) reads that document
through this module.  Field meanings follow ``src/model.py``:

* expressions ``Num/VarRef/ArrayRef/BinOp`` (``src/model.py:45-71``) become
  tuples ``("num", value, is_float)``, ``("var", id)``, ``("arr", id, index)``
  and ``("bin", op, left, right)``;
* statements ``DeclStmt/Assign/CallStmt/LoopStmt/ReplacedBlock``
  (``src/model.py:131-181``) become :class:`Stmt` records;
* occurrences keep their define/set/read kind and the region they belong to
  (``src/model.py:97-104``); loop-header occurrences are attached to the loop
  (``src/model.py:195-211``).
"""

from __future__ import annotations

import hashlib
import json
import sys
from dataclasses import dataclass, field

DEFINE, SET, READ = "define", "set", "read"


def _expr(doc: dict):
    if "num" in doc:
        return ("num", doc["num"], bool(doc.get("float", False)))
    if "var" in doc:
        return ("var", doc["var"])
    if "array" in doc:
        return ("arr", doc["array"], _expr(doc["index"]))
    return ("bin", doc["op"], _expr(doc["left"]), _expr(doc["right"]))


def expr_vars(e) -> list[int]:
    """Variable ids referenced by an expression, in syntactic order
    (mirrors ``expr_var_ids``, ``src/model.py:74-90``)."""
    out: list[int] = []

    def walk(x):
        if x[0] == "var":
            out.append(x[1])
        elif x[0] == "arr":
            out.append(x[1])
            walk(x[2])
        elif x[0] == "bin":
            walk(x[2])
            walk(x[3])

    walk(e)
    return out


@dataclass(frozen=True)
class Var:
    id: int
    name: str
    base_type: str  # "int" | "float"
    is_array: bool
    length: int


@dataclass
class Stmt:
    kind: str  # decl | assign | loop | call | replaced
    region: int
    index: int
    var: int | None = None          # decl
    init: tuple | None = None       # decl initializer
    target: tuple | None = None     # assign target expression
    value: tuple | None = None      # assign value expression
    loop: int | None = None         # loop statement
    call: int | None = None         # call statement
    replaced: dict | None = None    # replaced block payload
    occurrences: list = field(default_factory=list)  # (var, kind)
    uid: int = -1                   # document-order statement number


@dataclass
class Loop:
    id: int
    parent: int | None
    body: int
    index_var: int
    lower: tuple
    upper: tuple
    iter_count: int
    header_occurrences: list = field(default_factory=list)


@dataclass
class Call:
    id: int
    name: str
    subtree: int
    arg_types: tuple
    return_type: str
    arg_vars: tuple
    pure: bool


@dataclass
class Region:
    id: int
    enclosing_loop: int | None
    statements: list


class Program:
    """Parsed IR document with the structural queries the compiler needs."""

    def __init__(self, doc: dict):
        self.doc = doc
        self.language = doc.get("language", "c_like")
        self.root = doc.get("root_region", 0)
        self.vars = [Var(v["id"], v["name"], v["type"], bool(v.get("array", False)),
                         int(v.get("length", 0))) for v in doc["variables"]]
        self.loops = [Loop(l["id"], l["parent"], l["body"], l["index_var"], _expr(l["lower"]),
                           _expr(l["upper"]), int(l["iter_count"])) for l in doc["loops"]]
        self.calls = [Call(c["id"], c["name"], c["subtree"], tuple(c["arg_types"]),
                           c["return_type"], tuple(c.get("arg_vars", [])),
                           bool(c.get("pure", False))) for c in doc["calls"]]
        stmt_occ: dict[tuple[int, int], list] = {}
        for o in doc["occurrences"]:
            site = o["site"]
            if "stmt" in site:
                stmt_occ.setdefault(tuple(site["stmt"]), []).append((o["var"], o["kind"]))
            else:
                self.loops[site["loop_header"]].header_occurrences.append((o["var"], o["kind"]))
        self.regions: dict[int, Region] = {}
        for r in doc["regions"]:
            stmts = []
            for idx, s in enumerate(r["statements"]):
                occ = stmt_occ.get((r["id"], idx), [])
                if "decl" in s:
                    st = Stmt("decl", r["id"], idx, var=s["decl"],
                              init=_expr(s["init"]) if "init" in s else None)
                elif "assign" in s:
                    st = Stmt("assign", r["id"], idx, target=_expr(s["assign"]), value=_expr(s["value"]))
                elif "loop" in s:
                    st = Stmt("loop", r["id"], idx, loop=s["loop"])
                elif "call" in s:
                    st = Stmt("call", r["id"], idx, call=s["call"])
                else:
                    st = Stmt("replaced", r["id"], idx, replaced={
                        "name": s["replaced"], "args": list(s["args"]), "record": s.get("record"),
                        "speedup_hint": s.get("speedup_hint"), "base_cpu_time": s.get("base_cpu_time")})
                st.occurrences = occ
                stmts.append(st)
            self.regions[r["id"]] = Region(r["id"], r["enclosing_loop"], stmts)
        # document-order statement numbering and loop sites
        self.loop_site: dict[int, tuple[int, int]] = {}
        self.stmts: list[Stmt] = []
        for st in self.walk():
            st.uid = len(self.stmts)
            self.stmts.append(st)
            if st.kind == "loop":
                self.loop_site[st.loop] = (st.region, st.index)
        self.var_by_name = {v.name: v for v in self.vars}

    # -- traversal ---------------------------------------------------------

    def walk(self, region: int | None = None):
        """Statements in document pre-order, descending into loop bodies and
        call subtrees (``ProgramModel.walk_statements``, src/model.py:280-291)."""
        rid = self.root if region is None else region
        for st in self.regions[rid].statements:
            yield st
            if st.kind == "loop":
                yield from self.walk(self.loops[st.loop].body)
            elif st.kind == "call":
                yield from self.walk(self.calls[st.call].subtree)

    def subtree_regions(self, loop_id: int) -> list[int]:
        body = self.loops[loop_id].body
        out = [body]
        for st in self.walk(body):
            if st.kind == "loop":
                out.append(self.loops[st.loop].body)
            elif st.kind == "call":
                out.append(self.calls[st.call].subtree)
        return out

    def subtree_loops(self, loop_id: int) -> list[int]:
        return [loop_id] + [st.loop for st in self.walk(self.loops[loop_id].body) if st.kind == "loop"]

    def children(self, loop_id: int | None) -> list[int]:
        return [l.id for l in self.loops if l.parent == loop_id]

    def ancestors(self, loop_id: int) -> list[int]:
        out = []
        p = self.loops[loop_id].parent
        while p is not None:
            out.append(p)
            p = self.loops[p].parent
        return out

    def is_opaque_call(self, call_id: int) -> bool:
        return not self.regions[self.calls[call_id].subtree].statements

    # -- access sets ----------------------------------------------------------

    def stmt_access(self, st: Stmt) -> tuple[set[int], set[int]]:
        """(read, written) variable ids of one statement, from its expressions.
        Opaque calls read their arguments (``src/build.py:166-183``); the
        outputs of external bindings are added by the compiler."""
        reads: set[int] = set()
        writes: set[int] = set()
        if st.kind == "decl":
            if st.init is not None:
                writes.add(st.var)
                reads.update(expr_vars(st.init))
        elif st.kind == "assign":
            t = st.target
            writes.add(t[1])
            if t[0] == "arr":
                reads.update(expr_vars(t[2]))
            reads.update(expr_vars(st.value))
        elif st.kind == "call":
            if self.is_opaque_call(st.call):
                reads.update(self.calls[st.call].arg_vars)
        elif st.kind == "replaced":
            for v, kind in st.occurrences:
                (writes if kind == SET else reads).add(v)
            reads.update(st.replaced["args"])
        return reads, writes

    def loop_header_access(self, loop_id: int) -> tuple[set[int], set[int]]:
        l = self.loops[loop_id]
        reads = set(expr_vars(l.lower)) | set(expr_vars(l.upper)) | {l.index_var}
        return reads, {l.index_var}

    def subtree_access(self, loop_id: int, extra_writes=None) -> tuple[set[int], set[int]]:
        reads, writes = self.loop_header_access(loop_id)
        for st in self.walk(self.loops[loop_id].body):
            if st.kind == "loop":
                r, w = self.loop_header_access(st.loop)
            else:
                r, w = self.stmt_access(st)
                if extra_writes is not None and st.kind == "call":
                    w = w | extra_writes(st)
            reads |= r
            writes |= w
        return reads, writes

    # -- identity --------------------------------------------------------------

    def digest(self) -> str:
        return document_digest(self.doc)


def document_digest(doc: dict) -> str:
    blob = json.dumps(doc, sort_keys=True, separators=(",", ":")).encode()
    return hashlib.sha256(blob).hexdigest()


def document_of(model) -> dict:
    """IR document for a live reference model (via the reference's own
    serializer, ``irdoc.model_to_document``) or an already-serialised one."""
    if isinstance(model, dict):
        return model
    if isinstance(model, Program):
        return model.doc
    irdoc = sys.modules.get("gpuoffload.irdoc")
    if irdoc is None:
        import importlib

        irdoc = importlib.import_module("gpuoffload.irdoc")
    return irdoc.model_to_document(model)
