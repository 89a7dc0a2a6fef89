"""ORACLE — test infrastructure only.

Reference semantics of opaque library calls and replaced function blocks
(the reference gives them no body, ``src/build.py:166-183``,
and the fixture ``fft`` body is a placeholder, ``fixtures/three_loops_fft.mini:11-15``):

* ``gemm``: C[m,n] = sum_k A[m,k] B[k,n], row-major, accumulated in float64
  and rounded once to the element type;
* ``fft2d``: y = forward, unnormalised 2-D DFT of x (``numpy.fft.fft2``
  convention), both interleaved complex ``[re, im]`` row-major ``n x n``,
  computed in complex128;
* ``histogram``: ``h[d[i]] += 1`` over every element of the int array ``d``
  in order (the DB comparison snippet ``h[d[n]] = h[d[n]] + 1.0``,
  fixtures/sample_db.json:23), values outside ``[0, len(h))`` skipped.

Operand binding mirrors ``paper_2011_03602_b200.appspec`` but is restated here
so the checker does not import the product.
"""

from __future__ import annotations

import math

import numpy as np

BLOCK_KINDS = {"cublas_gemm": "gemm", "cufft_exec": "fft2d", "cuda_histogram": "histogram"}


def gemm(a: np.ndarray, b: np.ndarray, m: int, n: int, k: int, dtype) -> np.ndarray:
    A = a.astype(np.float64).reshape(m, k)
    B = b.astype(np.float64).reshape(k, n)
    return (A @ B).reshape(-1).astype(dtype)


def fft2d(x: np.ndarray, n: int, dtype) -> np.ndarray:
    z = x.astype(np.float64).reshape(n, n, 2)
    c = z[..., 0] + 1j * z[..., 1]
    f = np.fft.fft2(c)
    out = np.empty((n, n, 2), dtype=np.float64)
    out[..., 0] = f.real
    out[..., 1] = f.imag
    return out.reshape(-1).astype(dtype)


def _apply(kind: str, out: int, ins: list[int], state, spec_desc: dict) -> None:
    dtype = state[out].dtype
    if kind == "gemm":
        lc = state[out].shape[0]
        if "m" in spec_desc:
            m, n, k = int(spec_desc["m"]), int(spec_desc["n"]), int(spec_desc["k"])
        else:
            n = math.isqrt(lc)
            m = k = n
        state[out][:] = gemm(state[ins[0]], state[ins[1]], m, n, k, dtype)
    elif kind == "fft2d":
        n = int(spec_desc.get("n", math.isqrt(state[ins[0]].shape[0] // 2)))
        state[out][:] = fft2d(state[ins[0]], n, dtype)
    elif kind == "histogram":
        d = state[ins[0]].astype(np.int64)
        bins = state[out].shape[0]
        d = d[(d >= 0) & (d < bins)]
        counts = np.bincount(d, minlength=bins)
        state[out][:] = (state[out].astype(np.float64) + counts).astype(dtype) if dtype != np.int32 \
            else (state[out] + counts.astype(np.int32))
    else:
        raise ValueError(f"unknown external kind {kind!r}")


def make_binder(doc: dict, spec: dict):
    """Callback used by the interpreter and by the C oracle for opaque calls
    and replaced blocks."""
    occ_by_site: dict[tuple[int, int], list] = {}
    for o in doc["occurrences"]:
        if "stmt" in o["site"]:
            occ_by_site.setdefault(tuple(o["site"]["stmt"]), []).append((o["var"], o["kind"]))

    def bind(what: str, obj: dict, state) -> None:
        if what == "call":
            desc = spec.get("externals", {}).get(obj["name"])
            if desc is None:
                raise RuntimeError(f"no external binding for {obj['name']!r}")
            args = list(obj["arg_vars"])
            out = args[int(desc.get("out", len(args) - 1))]
            _apply(desc["kind"], out, [a for a in args if a != out], state, desc)
        else:
            desc = dict(spec.get("blocks", {}).get(obj["name"], {}))
            kind = desc.get("kind") or BLOCK_KINDS[obj["name"]]
            args = list(obj["args"])
            sets = [v for v, k in occ_by_site.get((obj["rid"], obj["index"]), []) if k == "set" and v in args]
            out = sets[0] if len(sets) == 1 else args[int(desc.get("out", len(args) - 1))]
            _apply(kind, out, [a for a in args if a != out], state, desc)

    return bind
