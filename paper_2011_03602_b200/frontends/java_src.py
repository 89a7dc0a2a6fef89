"""Java loop-nest subset -> IR document tagged ``java_like``.

Accepted (anything else raises FrontendError with the line):

* one top-level ``class`` (``package``/``import`` lines are skipped); its
  ``static`` members:
  - ``static final int N = 258;`` -- a compile-time constant, substituted by
    value (index expressions keep literal coefficients);
  - ``static float omega = 0.25f;``, ``static float ca0 = 0.0f - 8.0f / 3.0f;``
    (initialiser expressions become declaration initialisers),
    ``static int it;``, ``static double x;``, several declarators per line;
  - ``static float[] u = new float[N * N * N];`` (also ``float u[] = ...``):
    zero-initialised arrays (inputs come from the app spec);
* methods: the entry (``main`` by default, its ``String[] args`` ignored) and
  ``static void`` helpers whose parameters are bound at their call sites
  (expanded inline by the mini language, src/minilang.py:464-488);
* statements: ``for (int i = a; i < b; i++)`` (also ``i = a``, ``++i``,
  ``i += 1``; a braced block or a single statement), local declarations
  ``int i;`` / ``float s = e;`` (hoisted to top level), ``x = e;``,
  ``a[e] = e;``, ``+= -= *= /=``, ``x++``, calls ``f(a, b);`` with name
  arguments (unknown callees stay opaque external calls), nested blocks;
* expressions: ``+ - * /`` (Java int division truncates, like C), unary
  ``-``/``+``, parentheses, int and float literals (``0.8f``, ``1e-3``,
  ``2.0d``), names, 1-D subscripts.

``double`` and ``float`` both map to the IR's ``float``; a program that uses
``double`` reports ``precision = "fp64"`` (``java_precision``) for its app
spec, as the IR keeps one float width per program.
"""

from __future__ import annotations

import re

from . import FrontendError, to_document
from .common import Decl, Unit, binop, num

_TOKEN = re.compile(r"""
    (?P<ws>\s+|//[^\n]*|/\*.*?\*/)
  | (?P<num>(?:\d+\.\d*|\.\d+|\d+)(?:[eE][+-]?\d+)?[fFdDlL]?)
  | (?P<id>[A-Za-z_$][A-Za-z0-9_$]*)
  | (?P<op>\+\+|--|\+=|-=|\*=|/=|==|<=|>=|!=|&&|\|\||[{}()\[\];,=<>+\-*/.!%&|?:@])
""", re.S | re.X)

_TYPES = {"int": "int", "long": "int", "short": "int", "byte": "int", "float": "float", "double": "float"}
_MODIFIERS = {"public", "private", "protected", "static", "final", "strictfp", "synchronized"}


def _tokens(src: str):
    pos, line, out = 0, 1, []
    while pos < len(src):
        m = _TOKEN.match(src, pos)
        if not m:
            raise FrontendError(f"unexpected character {src[pos]!r}", line)
        kind = m.lastgroup
        text = m.group()
        if kind != "ws":
            out.append((kind, text, line))
        line += text.count("\n")
        pos = m.end()
    out.append(("eof", "", line))
    return out


class _Parser:
    def __init__(self, src: str, entry: str):
        self.t = _tokens(src)
        self.i = 0
        self.entry = entry
        self.u = Unit()
        self.methods: dict[str, tuple] = {}  # name -> (params [(type, is_array, name)], body token range)
        self.params: dict[str, Decl] = {}
        self.saw_double = False
        self.emitted: set[str] = set()

    # -- token helpers --------------------------------------------------------

    def peek(self, k: int = 0):
        return self.t[min(self.i + k, len(self.t) - 1)]

    def line(self) -> int:
        return self.peek()[2]

    def take(self, text: str | None = None, kind: str | None = None):
        tok = self.peek()
        if (text is not None and tok[1] != text) or (kind is not None and tok[0] != kind):
            raise FrontendError(f"expected {text or kind!r}, found {tok[1]!r}", tok[2])
        self.i += 1
        return tok

    def accept(self, text: str) -> bool:
        if self.peek()[1] == text:
            self.i += 1
            return True
        return False

    def lookup(self, n: str):
        return self.params.get(n) or self.u.decls.get(n)

    # -- class level ----------------------------------------------------------

    def program(self) -> str:
        while self.peek()[1] in ("package", "import"):
            while not self.accept(";"):
                self.i += 1
        while self.peek()[1] in _MODIFIERS or self.peek()[1] == "@":
            self.i += 1
        self.take("class")
        self.take(kind="id")
        if self.peek()[1] in ("extends", "implements"):
            raise FrontendError("class inheritance is not supported", self.line())
        self.take("{")
        while not self.accept("}"):
            self.member()
        if self.peek()[0] != "eof":
            raise FrontendError("one top-level class expected", self.line())
        if self.entry not in self.methods:
            raise FrontendError(f"no entry method {self.entry!r}")
        params, start, end = self.methods[self.entry]
        if params and not (self.entry == "main" and len(params) == 1 and params[0][0] == "String"):
            raise FrontendError(f"entry method {self.entry!r} must take no parameters (or String[] args)")
        body = self.body_at(start, end, 1)
        self.u.funcs.append("func main() {\n" + body + "}")
        return self.u.text()

    def member(self):
        mods = set()
        while self.peek()[1] in _MODIFIERS:
            mods.add(self.take()[1])
        line = self.line()
        tname = self.take(kind="id")[1]
        if tname == "void" or (self.peek()[0] == "id" and self.peek(1)[1] == "("):
            name = self.take(kind="id")[1]
            self.method(name, line)
            return
        if tname not in _TYPES:
            raise FrontendError(f"unsupported field type {tname!r}", line)
        if "static" not in mods:
            raise FrontendError("only static fields are supported", line)
        arr = self.accept("[")
        if arr:
            self.take("]")
        while True:
            name = self.take(kind="id")[1]
            is_arr = arr
            if self.accept("["):
                self.take("]")
                is_arr = True
            self.field(name, tname, is_arr, "final" in mods, line)
            if not self.accept(","):
                break
        self.take(";")

    def field(self, name, tname, is_arr, final, line):
        base = _TYPES[tname]
        self.saw_double |= tname == "double"
        if is_arr:
            if not self.accept("="):
                raise FrontendError(f"array {name!r} needs 'new {tname}[n]'", line)
            self.take("new")
            et = self.take(kind="id")[1]
            if _TYPES.get(et) != base:
                raise FrontendError("array element type mismatch", line)
            self.take("[")
            length = self.const_expr()
            self.take("]")
            self.u.declare(name, base, length, line=line)
            return
        if self.accept("="):
            if base == "int" and final:
                self.u.consts[name] = self.const_expr()
                return
            # initialiser expression over literals and earlier fields: a
            # mini-language declaration initialiser, run in declaration order
            # (src/build.py:83-87)
            text, t = self.expr()
            if base == "int" and t != "int":
                raise FrontendError(f"int field {name!r} with a float initialiser", line)
            self.u.declare(name, base, init=text, line=line)
        else:
            self.u.declare(name, base, line=line)

    def const_expr(self) -> int:
        text, t = self.expr()
        if t != "int":
            raise FrontendError("constant expression must be an integer", self.line())
        if not re.fullmatch(r"[0-9()+\-*/ ]+", text):
            raise FrontendError(f"not a constant expression: {text}", self.line())
        # digits and operators only (checked above); Java int division truncates
        v = eval(text.replace("/", "//"), {"__builtins__": {}}, {})  # noqa: S307
        return int(v)

    def method(self, name, line):
        self.take("(")
        params = []
        if not self.accept(")"):
            while True:
                tname = self.take(kind="id")[1]
                arr = False
                while self.accept("["):
                    self.take("]")
                    arr = True
                pname = self.take(kind="id")[1]
                if self.accept("["):
                    self.take("]")
                    arr = True
                params.append((tname, arr, pname))
                if self.accept(")"):
                    break
                self.take(",")
        if self.peek()[1] == "throws":
            raise FrontendError("throws clauses are not supported", self.line())
        start = self.i
        self.skip_block()
        self.methods[name] = (params, start, self.i)

    def skip_block(self):
        self.take("{")
        depth = 1
        while depth:
            tok = self.take()
            if tok[0] == "eof":
                raise FrontendError("unbalanced braces", tok[2])
            depth += {"{": 1, "}": -1}.get(tok[1], 0)

    def body_at(self, start, end, ind) -> str:
        saved = self.i
        self.i = start
        self.take("{")
        out = []
        while not self.accept("}"):
            out.append(self.stmt(ind))
        self.i = saved
        return "".join(out)

    # -- statements -----------------------------------------------------------

    def stmt(self, ind: int) -> str:
        pad = "  " * ind
        tok = self.peek()
        line = tok[2]
        if tok[1] == "{":
            self.take("{")
            out = []
            while not self.accept("}"):
                out.append(self.stmt(ind))
            return "".join(out)
        if tok[1] == ";":
            self.take(";")
            return ""
        if tok[1] == "for":
            return self.for_stmt(ind)
        if tok[1] in ("if", "while", "do", "return", "switch", "break", "continue"):
            raise FrontendError(f"'{tok[1]}' is not supported in the loop-nest subset", line)
        if tok[1] == "final":
            self.take()
            tok = self.peek()
        if tok[0] == "id" and tok[1] in _TYPES and self.peek(1)[0] == "id":
            return self.local_decl(ind)
        if tok[0] == "id" and self.peek(1)[1] == "(":
            return self.call_stmt(ind)
        text = self.simple_assign()
        self.take(";")
        return pad + text

    def local_decl(self, ind: int) -> str:
        pad = "  " * ind
        line = self.line()
        tname = self.take(kind="id")[1]
        self.saw_double |= tname == "double"
        base = _TYPES[tname]
        out = []
        while True:
            name = self.take(kind="id")[1]
            if self.peek()[1] == "[":
                raise FrontendError("local arrays are not supported (declare them static)", line)
            self.u.declare(name, base, line=line)
            if self.accept("="):
                rhs = self.expr()
                out.append(f"{pad}{name} = {rhs[0]};\n")
            if not self.accept(","):
                break
        self.take(";")
        return "".join(out)

    def for_stmt(self, ind: int) -> str:
        pad = "  " * ind
        line = self.line()
        self.take("for")
        self.take("(")
        if self.peek()[1] in _TYPES:
            t = self.take()[1]
            if _TYPES[t] != "int":
                raise FrontendError("loop index must be an integer", line)
        v = self.take(kind="id")[1]
        d = self.lookup(v) or self.u.declare(v, "int", line=line)
        if d.base != "int" or d.length is not None:
            raise FrontendError(f"loop index {v!r} must be an int scalar", line)
        self.take("=")
        lo = self.expr()
        self.take(";")
        if self.take(kind="id")[1] != v:
            raise FrontendError("the loop condition must test the index", line)
        self.take("<")
        hi = self.expr()
        self.take(";")
        if self.accept("++"):
            ok = self.take(kind="id")[1] == v
        else:
            ok = self.take(kind="id")[1] == v and (self.accept("++") or (self.accept("+=") and self.take(kind="num")[1] == "1"))
        if not ok:
            raise FrontendError("loop step must be i++", line)
        self.take(")")
        if lo[1] != "int" or hi[1] != "int":
            raise FrontendError("loop bounds must be integers", line)
        body = self.stmt(ind + 1)
        return f"{pad}for ({v} = {lo[0]}; {v} < {hi[0]}; {v}++) {{\n{body}{pad}}}\n"

    def simple_assign(self) -> str:
        line = self.line()
        name = self.take(kind="id")[1]
        if name in self.u.consts and name not in self.params:
            raise FrontendError(f"assignment to constant {name!r}", line)
        d = self.lookup(name)
        if d is None:
            raise FrontendError(f"undeclared variable {name!r}", line)
        if self.accept("["):
            if d.length is None:
                raise FrontendError(f"{name!r} is not an array", line)
            idx = self.expr()
            self.take("]")
            if idx[1] != "int":
                raise FrontendError("array index must be an integer expression", line)
            lhs = (f"{name}[{idx[0]}]", d.base)
        else:
            if d.length is not None:
                raise FrontendError(f"array {name!r} assigned without an index", line)
            lhs = (name, d.base)
        op = self.take()[1]
        if op == "=":
            rhs = self.expr()
        elif op in ("+=", "-=", "*=", "/="):
            rhs = binop(op[0], lhs, self.expr())
        elif op in ("++", "--"):
            rhs = binop("+" if op == "++" else "-", lhs, ("1", "int"))
        else:
            raise FrontendError(f"unsupported assignment operator {op!r}", line)
        return f"{lhs[0]} = {rhs[0]};\n"

    def call_stmt(self, ind: int) -> str:
        pad = "  " * ind
        line = self.line()
        name = self.take(kind="id")[1]
        self.take("(")
        args = []
        if not self.accept(")"):
            while True:
                a = self.take(kind="id")[1]
                if self.lookup(a) is None:
                    raise FrontendError(f"call argument {a!r} is not a declared variable", line)
                args.append(a)
                if self.accept(")"):
                    break
                self.take(",")
        self.take(";")
        m = self.methods.get(name)
        if m is not None and name not in self.emitted:
            params, start, end = m
            if len(params) != len(args):
                raise FrontendError(f"{name!r} expects {len(params)} arguments", line)
            self.emitted.add(name)
            local, ps = {}, []
            for (tname, arr, pname), a in zip(params, args):
                d = self.lookup(a)
                if _TYPES.get(tname) != d.base or arr != (d.length is not None):
                    raise FrontendError(f"argument {a!r} does not match parameter {pname!r}", line)
                local[pname] = Decl(pname, d.base, d.length)
                ps.append(f"{d.base} {pname}[{d.length}]" if arr else f"{d.base} {pname}")
            saved, self.params = self.params, local
            try:
                body = self.body_at(start, end, 1)
            finally:
                self.params = saved
            self.u.funcs.insert(0, f"func {name}({', '.join(ps)}) {{\n{body}}}")
        return f"{pad}{name}({', '.join(args)});\n"

    # -- expressions (precedence climbing) -------------------------------------

    def expr(self):
        a = self.term()
        while self.peek()[1] in ("+", "-"):
            op = self.take()[1]
            a = binop(op, a, self.term())
        return a

    def term(self):
        a = self.unary()
        while self.peek()[1] in ("*", "/"):
            op = self.take()[1]
            a = binop(op, a, self.unary())
        return a

    def unary(self):
        if self.accept("-"):
            v = self.unary()
            return (f"({'0.0' if v[1] == 'float' else '0'} - {v[0]})", v[1])
        if self.accept("+"):
            return self.unary()
        return self.factor()

    def factor(self):
        kind, text, line = self.peek()
        if text == "(":
            self.take("(")
            if self.peek()[1] in _TYPES and self.peek(1)[1] == ")":
                raise FrontendError("casts are not supported", line)
            v = self.expr()
            self.take(")")
            return (f"({v[0]})", v[1])
        if kind == "num":
            self.take()
            v = _num_value(text, line)
            self.saw_double |= isinstance(v, float) and text[-1:] not in "fF"
            return (num(v), "float" if isinstance(v, float) else "int")
        if kind == "id":
            self.take()
            if self.peek()[1] in ("(", "."):
                raise FrontendError(f"method calls in expressions are not supported ({text})", line)
            if text in self.u.consts and text not in self.params:
                return (num(self.u.consts[text]), "int")
            d = self.lookup(text)
            if d is None:
                raise FrontendError(f"undeclared name {text!r}", line)
            if self.accept("["):
                idx = self.expr()
                self.take("]")
                if d.length is None:
                    raise FrontendError(f"{text!r} is not an array", line)
                if idx[1] != "int":
                    raise FrontendError("array index must be an integer expression", line)
                return (f"{text}[{idx[0]}]", d.base)
            if d.length is not None:
                raise FrontendError(f"array {text!r} used without an index", line)
            return (text, d.base)
        raise FrontendError(f"unexpected {text!r} in expression", line)


def _num_value(text: str, line):
    t = text
    if t[-1] in "lL":
        raise FrontendError("long literals are not supported", line)
    is_float = t[-1] in "fFdD" or "." in t or "e" in t.lower()
    if t[-1] in "fFdD":
        t = t[:-1]
    return float(t) if is_float else int(t)


def java_to_mini(source: str, entry: str = "main") -> str:
    """Mini-language text of a Java program (the subset above)."""
    return _Parser(source, entry).program()


def java_precision(source: str, entry: str = "main") -> str:
    """``fp64`` when the program uses ``double``, else ``fp32``."""
    p = _Parser(source, entry)
    p.program()
    return "fp64" if p.saw_double else "fp32"


def java_to_document(source: str, entry: str = "main") -> dict:
    """IR document (``language: java_like``) of a Java program."""
    return to_document(java_to_mini(source, entry), "java_like")
