"""Python loop-nest subset -> IR document tagged ``python_like``.

Accepted (anything else raises FrontendError with the line):

* module level
  - ``N = 1024`` (int literal, never reassigned in a function): a compile-time
    constant, substituted by value so index expressions keep literal
    coefficients;
  - ``omega = 0.8`` / ``n: int`` / ``x: float = 0.0``: scalar variables;
  - ``a = [0.0] * (N * N)``, ``a = [0] * N``, ``a = np.zeros(N, dtype=np.float32)``
    (also ``np.empty``; dtype float32/float64/float -> float, int32/int64/int
    -> int): zero-initialised arrays (inputs come from the app spec, SURVEY.md
    Appendix A.2);
* functions: ``def main():`` (the entry) and helpers whose parameters are
  bound to module-level names at their call sites (the mini language expands
  them inline, src/minilang.py:464-488); ``global`` statements are ignored;
* statements: ``for v in range(stop)`` / ``range(start, stop)`` /
  ``range(start, stop, 1)``; ``x = e``; ``a[e] = e``; ``+= -= *= /=``; bare
  calls ``f(a, b)`` with name arguments (unknown callees stay opaque
  external calls, e.g. ``gemm(ma, mb, mc)`` for the block matcher); ``pass``;
* expressions: ``+ - * / //``, unary ``-``/``+``, int/float literals, names,
  1-D subscripts.  ``/`` is Python's true division: int / int is lowered as
  ``(a * 1.0) / b``; ``//`` on ints is C division (the subset assumes
  non-negative operands, where floor and truncation agree).

Variables first assigned inside a function (loop indices, temporaries) are
hoisted to top-level declarations, as the mini language requires; their type
is int for ``range`` indices and the type of their first assigned value
otherwise.
"""

from __future__ import annotations

import ast

from . import FrontendError, to_document
from .common import Unit, binop, num

_FLOAT_DTYPES = {"float32", "float64", "float", "double", "single"}
_INT_DTYPES = {"int32", "int64", "int", "intc"}


def _const_eval(node, consts, line):
    if isinstance(node, ast.Constant) and isinstance(node.value, int) and not isinstance(node.value, bool):
        return node.value
    if isinstance(node, ast.Name) and node.id in consts and isinstance(consts[node.id], int):
        return consts[node.id]
    if isinstance(node, ast.BinOp) and isinstance(node.op, (ast.Add, ast.Sub, ast.Mult, ast.FloorDiv)):
        a, b = _const_eval(node.left, consts, line), _const_eval(node.right, consts, line)
        return {ast.Add: a + b, ast.Sub: a - b, ast.Mult: a * b}.get(type(node.op), a // b if b else 0)
    raise FrontendError("array length must be an integer constant expression", line)


def _dtype_name(node) -> str | None:
    if isinstance(node, ast.Attribute):
        return node.attr
    if isinstance(node, ast.Name):
        return node.id
    if isinstance(node, ast.Constant) and isinstance(node.value, str):
        return node.value
    return None


class _Lower:
    def __init__(self, tree: ast.Module, entry: str):
        self.tree = tree
        self.entry = entry
        self.u = Unit()
        self.funcs: dict[str, ast.FunctionDef] = {}
        self.assigned_in_funcs: set[str] = set()
        self.params: dict = {}  # parameters of the helper being lowered: name -> Decl

    def lookup(self, n: str):
        return self.params.get(n) or self.u.decls.get(n)

    # -- module level ---------------------------------------------------------

    def run(self) -> str:
        for node in self.tree.body:
            if isinstance(node, ast.FunctionDef):
                self.funcs[node.name] = node
        for f in self.funcs.values():
            for n in ast.walk(f):
                if isinstance(n, (ast.Assign, ast.AugAssign, ast.AnnAssign)):
                    for t in (n.targets if isinstance(n, ast.Assign) else [n.target]):
                        if isinstance(t, ast.Name):
                            self.assigned_in_funcs.add(t.id)
                elif isinstance(n, ast.For) and isinstance(n.target, ast.Name):
                    self.assigned_in_funcs.add(n.target.id)
        for node in self.tree.body:
            if isinstance(node, ast.FunctionDef):
                continue
            if isinstance(node, (ast.Import, ast.ImportFrom)):
                continue
            if isinstance(node, ast.Expr) and isinstance(node.value, ast.Constant):
                continue  # docstring
            if isinstance(node, ast.Assign) and len(node.targets) == 1 and isinstance(node.targets[0], ast.Name):
                self.module_assign(node.targets[0].id, node.value, None, node.lineno)
            elif isinstance(node, ast.AnnAssign) and isinstance(node.target, ast.Name):
                self.module_assign(node.target.id, node.value, node.annotation, node.lineno)
            elif isinstance(node, ast.If) and _is_main_guard(node):
                continue
            else:
                raise FrontendError(f"unsupported module-level statement {type(node).__name__}", node.lineno)
        if self.entry not in self.funcs:
            raise FrontendError(f"no entry function {self.entry!r}")
        if self.funcs[self.entry].args.args:
            raise FrontendError(f"entry function {self.entry!r} must take no parameters", self.funcs[self.entry].lineno)
        self.emitted: set[str] = set()
        body = self.block(self.funcs[self.entry].body, 1, {})
        self.u.funcs.append("func main() {\n" + body + "}")
        return self.u.text()

    def module_assign(self, name: str, value, ann, line):
        ann_t = _dtype_name(ann) if ann is not None else None
        if value is None:
            if ann_t not in ("int", "float"):
                raise FrontendError(f"annotation of {name!r} must be int or float", line)
            self.u.declare(name, ann_t, line=line)
            return
        if isinstance(value, ast.Constant) and isinstance(value.value, (int, float)) \
                and not isinstance(value.value, bool):
            v = value.value
            base = "float" if isinstance(v, float) or ann_t == "float" else "int"
            if base == "int" and name not in self.assigned_in_funcs:
                self.u.consts[name] = v
                return
            self.u.declare(name, base, init=num(float(v) if base == "float" else v), line=line)
            return
        if isinstance(value, ast.UnaryOp) and isinstance(value.op, ast.USub) and isinstance(value.operand, ast.Constant):
            self.module_assign(name, ast.Constant(-value.operand.value), ann, line)
            return
        # [c] * n
        if isinstance(value, ast.BinOp) and isinstance(value.op, ast.Mult):
            lst, n = (value.left, value.right) if isinstance(value.left, ast.List) else (value.right, value.left)
            if isinstance(lst, ast.List) and len(lst.elts) == 1 and isinstance(lst.elts[0], ast.Constant):
                c = lst.elts[0].value
                if c != 0:
                    raise FrontendError("arrays start zeroed; give inputs in the app spec", line)
                self.u.declare(name, "float" if isinstance(c, float) else "int",
                               _const_eval(n, self.u.consts, line), line=line)
                return
        # np.zeros(n, dtype=...)
        if isinstance(value, ast.Call) and isinstance(value.func, ast.Attribute) and value.func.attr in ("zeros", "empty"):
            if not value.args:
                raise FrontendError("np.zeros needs a length", line)
            length = _const_eval(value.args[0], self.u.consts, line)
            dt = "float64"
            for kw in value.keywords:
                if kw.arg == "dtype":
                    dt = _dtype_name(kw.value)
            if len(value.args) > 1:
                dt = _dtype_name(value.args[1])
            if dt in _FLOAT_DTYPES:
                base = "float"
            elif dt in _INT_DTYPES:
                base = "int"
            else:
                raise FrontendError(f"unsupported dtype {dt!r}", line)
            self.u.declare(name, base, length, line=line)
            return
        raise FrontendError(f"unsupported initialiser for {name!r}", line)

    # -- statements -----------------------------------------------------------

    def block(self, stmts, ind: int, subst: dict) -> str:
        return "".join(self.stmt(s, ind, subst) for s in stmts)

    def stmt(self, s, ind: int, subst: dict) -> str:
        pad = "  " * ind
        if isinstance(s, (ast.Global, ast.Nonlocal, ast.Pass)):
            return ""
        if isinstance(s, ast.Expr) and isinstance(s.value, ast.Constant):
            return ""  # docstring
        if isinstance(s, ast.For):
            if s.orelse:
                raise FrontendError("for-else is not supported", s.lineno)
            if not isinstance(s.target, ast.Name):
                raise FrontendError("loop target must be a name", s.lineno)
            it = s.iter
            if not (isinstance(it, ast.Call) and isinstance(it.func, ast.Name) and it.func.id == "range"
                    and not it.keywords and 1 <= len(it.args) <= 3):
                raise FrontendError("only 'for v in range(...)' loops are supported", s.lineno)
            args = it.args
            if len(args) == 3 and not (isinstance(args[2], ast.Constant) and args[2].value == 1):
                raise FrontendError("range step must be 1", s.lineno)
            lo = self.expr(args[0], subst, s.lineno) if len(args) >= 2 else ("0", "int")
            hi = self.expr(args[-1] if len(args) == 1 else args[1], subst, s.lineno)
            if lo[1] != "int" or hi[1] != "int":
                raise FrontendError("range bounds must be integers", s.lineno)
            v = self.name(s.target.id, subst)
            self.u.declare(v, "int", line=s.lineno)
            body = self.block(s.body, ind + 1, subst)
            return f"{pad}for ({v} = {lo[0]}; {v} < {hi[0]}; {v}++) {{\n{body}{pad}}}\n"
        if isinstance(s, ast.Assign):
            if len(s.targets) != 1:
                raise FrontendError("chained / tuple assignment is not supported", s.lineno)
            return pad + self.assign(s.targets[0], s.value, None, subst, s.lineno)
        if isinstance(s, ast.AugAssign):
            op = {ast.Add: "+", ast.Sub: "-", ast.Mult: "*", ast.Div: "/"}.get(type(s.op))
            if op is None:
                raise FrontendError("unsupported augmented assignment", s.lineno)
            return pad + self.assign(s.target, s.value, op, subst, s.lineno)
        if isinstance(s, ast.AnnAssign) and s.value is not None:
            return pad + self.assign(s.target, s.value, None, subst, s.lineno)
        if isinstance(s, ast.Expr) and isinstance(s.value, ast.Call):
            return self.call(s.value, ind, subst, s.lineno)
        raise FrontendError(f"unsupported statement {type(s).__name__}", getattr(s, "lineno", None))

    def assign(self, target, value, aug: str | None, subst: dict, line) -> str:
        rhs = self.expr(value, subst, line)
        if isinstance(target, ast.Name):
            name = self.name(target.id, subst)
            if name in self.u.consts:
                raise FrontendError(f"assignment to constant {name!r}", line)
            d = self.lookup(name)
            if d is None:
                d = self.u.declare(name, rhs[1], line=line)
            if d.length is not None:
                raise FrontendError(f"array {name!r} assigned without an index", line)
            lhs = (name, d.base)
        elif isinstance(target, ast.Subscript) and isinstance(target.value, ast.Name):
            name = self.name(target.value.id, subst)
            d = self.lookup(name)
            if d is None or d.length is None:
                raise FrontendError(f"{name!r} is not a declared array", line)
            idx = self.expr(_index(target), subst, line)
            if idx[1] != "int":
                raise FrontendError("array index must be an integer expression", line)
            lhs = (f"{name}[{idx[0]}]", d.base)
        else:
            raise FrontendError("unsupported assignment target", line)
        if aug is not None:
            rhs = self.arith(aug, lhs, rhs, line)
        return f"{lhs[0]} = {rhs[0]};\n"

    def call(self, c: ast.Call, ind: int, subst: dict, line) -> str:
        if not isinstance(c.func, ast.Name) or c.keywords:
            raise FrontendError("only calls 'f(a, b, ...)' with name arguments are supported", line)
        args = []
        for a in c.args:
            if not isinstance(a, ast.Name):
                raise FrontendError("call arguments must be variable names", line)
            n = self.name(a.id, subst)
            if self.lookup(n) is None:
                raise FrontendError(f"call argument {n!r} is not a declared variable", line)
            args.append(n)
        f = self.funcs.get(c.func.id)
        pad = "  " * ind
        if f is None:
            return f"{pad}{c.func.id}({', '.join(args)});\n"
        params = [p.arg for p in f.args.args]
        if len(params) != len(args):
            raise FrontendError(f"{c.func.id!r} expects {len(params)} arguments", line)
        if c.func.id not in self.emitted:
            # helper: parameters typed by this (first) call site
            self.emitted.add(c.func.id)
            from .common import Decl

            ps, local = [], {}
            for p, a in zip(params, args):
                d = self.lookup(a)
                local[p] = Decl(p, d.base, d.length)
                ps.append(f"{d.base} {p}[{d.length}]" if d.length is not None else f"{d.base} {p}")
            saved, self.params = self.params, local
            try:
                body = self.block(f.body, 1, {})
            finally:
                self.params = saved
            self.u.funcs.insert(0, f"func {c.func.id}({', '.join(ps)}) {{\n{body}}}")
        return f"{pad}{c.func.id}({', '.join(args)});\n"

    # -- expressions ----------------------------------------------------------

    def name(self, n: str, subst: dict) -> str:
        return subst.get(n, n)

    def arith(self, op: str, a, b, line):
        if op == "/" and a[1] == "int" and b[1] == "int":
            # Python true division of ints
            return binop("/", (f"({a[0]} * 1.0)", "float"), b)
        return binop(op, a, b)

    def expr(self, e, subst: dict, line) -> tuple[str, str]:
        if isinstance(e, ast.Constant):
            if isinstance(e.value, bool) or not isinstance(e.value, (int, float)):
                raise FrontendError(f"unsupported literal {e.value!r}", line)
            return num(e.value), "float" if isinstance(e.value, float) else "int"
        if isinstance(e, ast.Name):
            n = self.name(e.id, subst)
            if n in self.u.consts and n not in self.params:
                v = self.u.consts[n]
                return num(v), "int" if isinstance(v, int) else "float"
            d = self.lookup(n)
            if d is None:
                raise FrontendError(f"undeclared name {n!r}", line)
            if d.length is not None:
                raise FrontendError(f"array {n!r} used without an index", line)
            return n, d.base
        if isinstance(e, ast.Subscript) and isinstance(e.value, ast.Name):
            n = self.name(e.value.id, subst)
            d = self.lookup(n)
            idx = self.expr(_index(e), subst, line)
            if idx[1] != "int":
                raise FrontendError("array index must be an integer expression", line)
            if d is None or d.length is None:
                raise FrontendError(f"{n!r} is not a declared array", line)
            return f"{n}[{idx[0]}]", d.base
        if isinstance(e, ast.UnaryOp):
            v = self.expr(e.operand, subst, line)
            if isinstance(e.op, ast.UAdd):
                return v
            if isinstance(e.op, ast.USub):
                zero = "0.0" if v[1] == "float" else "0"
                return f"({zero} - {v[0]})", v[1]
            raise FrontendError("unsupported unary operator", line)
        if isinstance(e, ast.BinOp):
            a, b = self.expr(e.left, subst, line), self.expr(e.right, subst, line)
            if isinstance(e.op, ast.FloorDiv):
                if a[1] != "int" or b[1] != "int":
                    raise FrontendError("'//' is supported on integers only", line)
                return binop("/", a, b)
            op = {ast.Add: "+", ast.Sub: "-", ast.Mult: "*", ast.Div: "/"}.get(type(e.op))
            if op is None:
                raise FrontendError(f"unsupported operator {type(e.op).__name__}", line)
            return self.arith(op, a, b, line)
        raise FrontendError(f"unsupported expression {type(e).__name__}", line)


def _index(sub: ast.Subscript):
    idx = sub.slice
    if isinstance(idx, (ast.Tuple, ast.Slice)):
        raise FrontendError("only 1-D integer subscripts are supported", getattr(sub, "lineno", None))
    return idx


def _is_main_guard(node: ast.If) -> bool:
    t = node.test
    return isinstance(t, ast.Compare) and isinstance(t.left, ast.Name) and t.left.id == "__name__"


def python_to_mini(source: str, entry: str = "main") -> str:
    """Mini-language text of a Python program (the subset above)."""
    try:
        tree = ast.parse(source)
    except SyntaxError as exc:
        raise FrontendError(f"Python syntax error: {exc.msg}", exc.lineno) from exc
    return _Lower(tree, entry).run()


def python_to_document(source: str, entry: str = "main") -> dict:
    """IR document (``language: python_like``) of a Python program."""
    return to_document(python_to_mini(source, entry), "python_like")
