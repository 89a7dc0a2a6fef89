"""Himeno benchmark (19-point Jacobi) written in the reference's mini-language.

Two forms, both following SURVEY.md Appendix B:

* ``inline`` (the default, the form the GA can offload): the Jacobi nest has
  no scalar temporaries; it writes ``gs[idx] = SS*SS`` and
  ``wrk2[idx] = p[idx] + omega*SS`` with ``SS`` expanded textually, and the
  ``gosa`` reduction is a separate host nest.  The reference screen
  (``src/screen.py:57-68``) then admits Jacobi i/j/k and copy i/j/k, so the
  genome length is 6.
* ``temps``: the textbook form with ``s0``/``ss``/``gosa`` inside the nest; the
  screen rejects it (``loop_carried_scalar``) and only the copy nest enters the
  genome (a=3).  Kept for parity tests of screen-rejected host nests.

Sizes are the Himeno grid sizes (array extents); the interior is
``[1, n-1)`` in every dimension, as in SURVEY.md §2.2 K1 (M: 127*127*255
interior points).  Inputs follow the standard ``initmt``.
"""

from __future__ import annotations

SIZES = {
    "XS": (9, 9, 17),
    "S": (65, 65, 129),
    "M": (129, 129, 257),
    "L": (257, 257, 513),
}

ARRAYS = ("p", "a0", "a1", "a2", "a3", "b0", "b1", "b2", "c0", "c1", "c2", "bnd", "wrk1", "wrk2")


def _idx(J: int, K: int, di: int = 0, dj: int = 0, dk: int = 0) -> str:
    def term(name: str, d: int) -> str:
        if d == 0:
            return name
        return f"({name} + {d})" if d > 0 else f"({name} - {-d})"

    return f"({term('i', di)} * {J} + {term('j', dj)}) * {K} + {term('k', dk)}"


def _s0(J: int, K: int) -> str:
    c = lambda di, dj, dk: f"p[{_idx(J, K, di, dj, dk)}]"  # noqa: E731
    x = _idx(J, K)
    return (
        f"a0[{x}] * {c(1, 0, 0)}"
        f" + a1[{x}] * {c(0, 1, 0)}"
        f" + a2[{x}] * {c(0, 0, 1)}"
        f" + b0[{x}] * ({c(1, 1, 0)} - {c(1, -1, 0)} - {c(-1, 1, 0)} + {c(-1, -1, 0)})"
        f" + b1[{x}] * ({c(0, 1, 1)} - {c(0, -1, 1)} - {c(0, 1, -1)} + {c(0, -1, -1)})"
        f" + b2[{x}] * ({c(1, 0, 1)} - {c(-1, 0, 1)} - {c(1, 0, -1)} + {c(-1, 0, -1)})"
        f" + c0[{x}] * {c(-1, 0, 0)}"
        f" + c1[{x}] * {c(0, -1, 0)}"
        f" + c2[{x}] * {c(0, 0, -1)}"
        f" + wrk1[{x}]"
    )


def source(size: str | tuple[int, int, int] = "M", nn: int = 4, form: str = "inline", read_p: bool = True) -> str:
    """``read_p=False`` drops the final host read of ``p``: the reference plan
    then never fetches ``p``, the hole the coherent variable
    manager repairs."""
    I, J, K = SIZES[size] if isinstance(size, str) else size
    n = I * J * K
    x = _idx(J, K)
    loops = lambda body, ind="    ": (  # noqa: E731
        f"{ind}for (i = 1; i < {I - 1}; i++) {{\n"
        f"{ind}  for (j = 1; j < {J - 1}; j++) {{\n"
        f"{ind}    for (k = 1; k < {K - 1}; k++) {{\n"
        + "".join(f"{ind}      {line}\n" for line in body)
        + f"{ind}    }}\n{ind}  }}\n{ind}}}\n"
    )
    decls = ["int n;", "int i;", "int j;", "int k;", f"int nn = {nn};",
             "float omega = 0.8;", "float gosa;", "float chk;"]
    if form == "temps":
        decls += ["float s0;", "float ss;"]
    decls += [f"float {a}[{n}];" for a in ARRAYS]
    if form == "inline":
        decls.append(f"float gs[{n}];")
    out = "\n".join(decls) + "\n\nfunc main() {\n  for (n = 0; n < nn; n++) {\n    gosa = 0.0;\n"
    if form == "inline":
        ss = f"(({_s0(J, K)}) * a3[{x}] - p[{x}]) * bnd[{x}]"
        out += loops([f"gs[{x}] = ({ss}) * ({ss});", f"wrk2[{x}] = p[{x}] + omega * ({ss});"])
        out += loops([f"gosa = gosa + gs[{x}];"])
    elif form == "temps":
        out += loops([
            f"s0 = {_s0(J, K)};",
            f"ss = (s0 * a3[{x}] - p[{x}]) * bnd[{x}];",
            "gosa = gosa + ss * ss;",
            f"wrk2[{x}] = p[{x}] + omega * ss;",
        ])
    else:
        raise ValueError(f"unknown Himeno form {form!r}")
    out += loops([f"p[{x}] = wrk2[{x}];"])
    tail = "gosa + p[0] + gs[0]" if form == "inline" else "gosa + p[0]"
    if not read_p:
        tail = tail.replace(" + p[0]", "")
    out += f"  }}\n  chk = {tail};\n}}\n"
    return out


def spec(size: str | tuple[int, int, int] = "M", form: str = "inline", precision: str = "fp32",
         reductions: bool = False) -> dict:
    """App spec: standard initmt inputs, outputs read by the final host
    statement, fp32 tolerance 1e-5 (BASELINE.md parity tolerances).

    ``reductions=True`` is the opt-in of reductions.py (gosa reduced on the
    GPU): the tree-ordered sum differs from the sequential fp32 sum by the
    latter's rounding error -- at size M the sequential fp32 gosa is 2.5 %
    above the exact (float64) sum of the same gs values, while the GPU tree
    sum agrees with it to ~1e-7 (tests/test_reductions.py) -- so ``gosa`` and
    ``chk`` are compared at 5e-2 (documented deviation; p and gs keep 1e-5)."""
    I, J, K = SIZES[size] if isinstance(size, str) else size
    inputs = {
        "p": {"kind": "himeno_p", "dims": [I, J, K]},
        "a0": {"kind": "fill", "value": 1.0},
        "a1": {"kind": "fill", "value": 1.0},
        "a2": {"kind": "fill", "value": 1.0},
        "a3": {"kind": "fill", "value": 1.0 / 6.0},
        "c0": {"kind": "fill", "value": 1.0},
        "c1": {"kind": "fill", "value": 1.0},
        "c2": {"kind": "fill", "value": 1.0},
        "bnd": {"kind": "fill", "value": 1.0},
        # b0..b2 and wrk1 are zero (file-scope zero init)
    }
    outs = ["p", "gosa", "chk"] + (["gs"] if form == "inline" else [])
    rel = 1e-5 if precision == "fp32" else 1e-12
    out = {
        "name": f"himeno_{form}_{'x'.join(map(str, (I, J, K)))}",
        "precision": precision,
        "inputs": inputs,
        "outputs": {o: {"rel_tol": rel} for o in outs},
    }
    if reductions:
        out["reductions"] = True
        out["name"] += "_red"
        for o in ("gosa", "chk"):
            out["outputs"][o]["rel_tol"] = 5e-2 if precision == "fp32" else 1e-9
    return out


def interior_points(size: str | tuple[int, int, int] = "M") -> int:
    I, J, K = SIZES[size] if isinstance(size, str) else size
    return (I - 2) * (J - 2) * (K - 2)


#: algorithmic HBM bytes per interior point per sweep.  The
#: inline Jacobi nest reads 13 fp32 streams exactly once (p, a0..a3, b0..b2,
#: c0..c2, bnd, wrk1; p's 18 neighbour reads are cache hits) and writes two
#: (wrk2, gs): 15 * 4 = 60 B.  SURVEY/BASELINE quote 64 B (14 reads + wrk2
#: write, the textbook count); we report the smaller, exact figure.  The copy
#: nest reads wrk2 and writes p: 8 B.
JACOBI_BYTES_PER_POINT = 60
COPY_BYTES_PER_POINT = 8
