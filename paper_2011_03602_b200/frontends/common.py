"""Shared lowering helpers: typed expressions rendered as mini-language
text (fully parenthesised, no unary minus: ``-e`` becomes ``(0 - e)``)."""

from __future__ import annotations

from dataclasses import dataclass, field

from . import FrontendError

RESERVED = {"for", "func", "int", "float"}


@dataclass
class Decl:
    name: str
    base: str                 # "int" | "float"
    length: int | None = None  # arrays
    init: str | None = None    # scalar initializer (mini text)


@dataclass
class Unit:
    """A program being lowered: top-level declarations (every variable is
    top-level in the mini language), constants substituted by value, and
    function bodies as mini text."""

    decls: dict[str, Decl] = field(default_factory=dict)
    consts: dict[str, int | float] = field(default_factory=dict)
    funcs: list[str] = field(default_factory=list)

    def declare(self, name: str, base: str, length: int | None = None, init: str | None = None, line=None):
        if name in RESERVED:
            raise FrontendError(f"{name!r} is a reserved word of the mini language", line)
        old = self.decls.get(name)
        if old is not None:
            if (old.base, old.length) != (base, length):
                raise FrontendError(f"{name!r} redeclared with another type", line)
            return old
        d = Decl(name, base, length, init)
        self.decls[name] = d
        return d

    def text(self) -> str:
        out = []
        for d in self.decls.values():
            if d.length is not None:
                out.append(f"{d.base} {d.name}[{d.length}];")
            elif d.init is not None:
                out.append(f"{d.base} {d.name} = {d.init};")
            else:
                out.append(f"{d.base} {d.name};")
        return "\n".join(out) + "\n\n" + "\n".join(self.funcs) + "\n"


def num(v: int | float) -> str:
    """Mini-language literal (floats keep a '.', negatives become 0 - x)."""
    if isinstance(v, bool):
        raise FrontendError("booleans are not supported")
    if isinstance(v, int):
        return str(v) if v >= 0 else f"(0 - {-v})"
    s = repr(float(v))
    if "inf" in s or "nan" in s:
        raise FrontendError(f"literal {v!r} is not representable")
    if "." not in s and "e" not in s:
        s += ".0"
    return s if v >= 0 else f"(0.0 - {s[1:]})"


def _int_lit(text: str) -> int | None:
    if text.isdigit():
        return int(text)
    if text.startswith("(0 - ") and text.endswith(")") and text[5:-1].isdigit():
        return -int(text[5:-1])
    return None


def binop(op: str, a: tuple[str, str], b: tuple[str, str]) -> tuple[str, str]:
    """(text, type) of ``a op b`` under C's usual conversions.  Integer
    literal operands are folded (C semantics, division truncates toward zero)
    so bounds like ``N - 1`` stay constants: the reference derives trip
    counts, hence transfer multiplicities, only from constant bounds
    (pkg/docs/mini_language.md "Trip counts")."""
    t = "float" if "float" in (a[1], b[1]) else "int"
    x, y = _int_lit(a[0]), _int_lit(b[0])
    if t == "int" and x is not None and y is not None and not (op == "/" and y == 0):
        if op == "+":
            return num(x + y), "int"
        if op == "-":
            return num(x - y), "int"
        if op == "*":
            return num(x * y), "int"
        if op == "/":
            q = abs(x) // abs(y)
            return num(q if (x >= 0) == (y >= 0) else -q), "int"
    return f"({a[0]} {op} {b[0]})", t
