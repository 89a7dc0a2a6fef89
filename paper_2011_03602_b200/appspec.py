"""App specs: what the reference model does not carry.

The reference model has no numeric semantics for inputs, outputs, element
widths or opaque library calls.  An app spec fixes
them, by variable *name* (names survive ``apply_replacements`` while ids of
loops do not, ``src/blocks.py:480-563``):

* ``precision``: ``fp32`` (model ``float`` -> C ``float``) or ``fp64``;
  ``int`` is always C ``int`` (Appendix A.1).
* ``inputs``: initial values, everything else is zero (C file scope, A.2).
* ``outputs``: variables compared against the reference run, each with a
  ``rel_tol`` and a ``compare`` mode (``elementwise`` is the reference rule
  ``|c-r| <= max(rel*|r|, 1e-12)``, ``src/evaluators.py:129-139``;
  ``normwise`` is the documented deviation for FFT/GEMM outputs).
* ``externals``: CPU semantics of opaque calls (``gemm``/``fft``/``histogram``), A.5.
* ``blocks``: shapes of replaced function blocks (``cublas_gemm``/``cufft_exec``/
  ``cuda_histogram``).
"""

from __future__ import annotations

import math

import numpy as np

from .ir import Program

# per-precision default of an output's rel_tol when the spec names none.  The
# reference's validate_output default is 1e-6 (src/evaluators.py:129-139,
# a harness for doubles printed as text); fp32 apps default to 1e-5 (SURVEY.md
# Appendix A.8: the reference's own C text computes them in float), a
# documented deviation.  Every golden app spells its tolerance out.
DEFAULT_REL_TOL = {"fp32": 1e-5, "fp64": 1e-12}


def np_dtype(base_type: str, precision: str):
    if base_type == "int":
        return np.int32
    return np.float32 if precision == "fp32" else np.float64


def _fill_input(var, dtype, desc: dict) -> np.ndarray:
    n = var.length if var.is_array else 1
    kind = desc.get("kind", "fill")
    if kind == "fill":
        return np.full(n, desc.get("value", 0), dtype=dtype)
    if kind == "uniform":
        rng = np.random.default_rng(int(desc.get("seed", 0)))
        lo, hi = float(desc.get("lo", 0.0)), float(desc.get("hi", 1.0))
        return (rng.random(n) * (hi - lo) + lo).astype(dtype)
    if kind == "randint":
        rng = np.random.default_rng(int(desc.get("seed", 0)))
        return rng.integers(int(desc.get("lo", 0)), int(desc.get("hi", 2)), n).astype(dtype)
    if kind == "himeno_p":
        I, J, K = desc["dims"]
        i = np.arange(n) // (J * K)
        # initmt: p[i][j][k] = (float)(i*i) / (float)((imax-1)*(imax-1))
        if dtype == np.float32:
            return (i.astype(np.float32) * i.astype(np.float32)) / np.float32((I - 1) * (I - 1))
        return (i * i).astype(np.float64) / float((I - 1) * (I - 1))
    if kind == "arange":
        return (np.arange(n) * float(desc.get("scale", 1.0)) + float(desc.get("offset", 0.0))).astype(dtype)
    raise ValueError(f"unknown input kind {kind!r}")


def initial_state(prog: Program, spec: dict) -> dict[int, np.ndarray]:
    """Pristine value of every variable (1-element arrays for scalars)."""
    precision = spec.get("precision", "fp32")
    inputs = spec.get("inputs", {})
    unknown = set(inputs) - set(prog.var_by_name)
    if unknown:
        raise ValueError(f"app spec names unknown variables {sorted(unknown)}")
    state = {}
    for v in prog.vars:
        dtype = np_dtype(v.base_type, precision)
        if v.name in inputs:
            state[v.id] = np.ascontiguousarray(_fill_input(v, dtype, inputs[v.name]))
        else:
            state[v.id] = np.zeros(v.length if v.is_array else 1, dtype=dtype)
    return state


def outputs_of(prog: Program, spec: dict) -> list[tuple[int, float, str]]:
    """(var id, rel_tol, compare mode) for every declared output present in
    this program variant."""
    precision = spec.get("precision", "fp32")
    out = []
    for name, desc in spec.get("outputs", {}).items():
        if name not in prog.var_by_name:
            continue
        rel = float(desc.get("rel_tol", DEFAULT_REL_TOL[precision]))
        out.append((prog.var_by_name[name].id, rel, desc.get("compare", "elementwise")))
    return out


EXTERNAL_KINDS = ("gemm", "fft2d", "histogram")
BLOCK_KINDS = {"cublas_gemm": "gemm", "cufft_exec": "fft2d", "cuda_histogram": "histogram"}


def external_binding(spec: dict, name: str) -> dict | None:
    ext = spec.get("externals", {})
    return ext.get(name)


def block_binding(prog: Program, spec: dict, stmt) -> dict:
    """Operand binding and shape of a replaced block.

    The output is the argument with a ``set`` occurrence (similarity path,
    first-occurrence order ``cublas_gemm(mc, ma, mb)``) or, when the block
    came from an opaque call whose occurrences are all reads (name path,
    ``cublas_gemm(ma, mb, mc)``), the position the app spec gives for the
    original callee (default: last).  Inputs keep their order.
    """
    rb = stmt.replaced
    name = rb["name"]
    args = list(rb["args"])
    desc = dict(spec.get("blocks", {}).get(name, {}))
    kind = desc.get("kind") or BLOCK_KINDS.get(name)
    if kind is None:
        raise ValueError(f"no block semantics for replacement {name!r}")
    set_vars = [v for v, k in stmt.occurrences if k == "set" and v in args]
    if len(set_vars) == 1:
        out = set_vars[0]
    else:
        out = args[int(desc.get("out", len(args) - 1))]
    ins = [a for a in args if a != out]
    binding = {"kind": kind, "out": out, "ins": ins}
    _shape(prog, binding, desc)
    return binding


def _shape(prog: Program, binding: dict, desc: dict) -> None:
    """Operand shapes of a gemm / fft2d / histogram binding, checked against
    the operand lengths (a mismatch is a ValueError, which the compiler
    reports as compile_error: never an out-of-bounds library call)."""
    kind, out, ins = binding["kind"], binding["out"], binding["ins"]
    if kind == "gemm":
        if len(ins) < 2:
            raise ValueError("gemm needs two input operands")
        a, b = ins[0], ins[1]
        la, lb, lc = (prog.vars[x].length for x in (a, b, out))
        if "m" in desc:
            m, n, k = int(desc["m"]), int(desc["n"]), int(desc["k"])
        else:
            n = math.isqrt(lc)
            m, k = n, n
        if min(m, n, k) <= 0 or m * k != la or k * n != lb or m * n != lc:
            raise ValueError(f"gemm shape {m}x{n}x{k} does not match operand lengths {la},{lb},{lc}")
        binding.update(m=m, n=n, k=k)
    elif kind == "fft2d":
        if not ins:
            raise ValueError("fft2d needs an input operand")
        lx = prog.vars[ins[0]].length
        n = int(desc.get("n", math.isqrt(lx // 2)))
        if n <= 0 or 2 * n * n != lx or prog.vars[out].length != lx:
            raise ValueError(f"fft2d size {n} does not match operand lengths")
        binding.update(n=n)
    elif kind == "histogram":
        _histogram_shape(prog, binding)
    else:
        raise ValueError(f"unknown external kind {kind!r}")


def _histogram_shape(prog: Program, binding: dict) -> None:
    """``cuda_histogram(d, h)`` (fixtures/sample_db.json:20-28, interface
    ``int[], int[]``): ``h[d[i]] += 1`` for every element of ``d``; bins =
    len(h).  Values outside [0, bins) are skipped (the original C loop would
    write out of bounds)."""
    d = binding["ins"][0]
    if prog.vars[d].base_type != "int":
        raise ValueError("histogram data must be an int array")
    binding.update(m=prog.vars[binding["out"]].length, n=prog.vars[d].length)


def external_call_binding(prog: Program, spec: dict, call) -> dict:
    """CPU binding of an opaque call (Appendix A.5): same operand rules as a
    name-matched block; the output position comes from the spec."""
    desc = external_binding(spec, call.name)
    if desc is None:
        raise ValueError(f"opaque call {call.name!r} has no CPU binding in the app spec")
    args = list(call.arg_vars)
    out = args[int(desc.get("out", len(args) - 1))]
    ins = [a for a in args if a != out]
    binding = {"kind": desc["kind"], "out": out, "ins": ins}
    _shape(prog, binding, desc)  # the same length checks as a replaced block
    return binding
