"""Function-block app (BASELINE config 3): a program calling ``gemm`` and
``fft`` as opaque library calls, which the reference's name matcher pairs with
the ``matmul``/``fft`` records of ``fixtures/sample_db.json`` and replaces by
``cublas_gemm`` / ``cufft_exec`` (``src/blocks.py:275-291``).

CPU semantics of the original calls: ``gemm(A, B, C)``
is C = A B (n x n, row-major); ``fft(x, y)`` is y = FFT2(x), interleaved
complex ``float[2 n^2]``.  ``mc`` is compared element-wise (the reference
rule, src/evaluators.py:129-139); ``y`` norm-wise (documented deviation,
SURVEY.md Appendix A.8: FFT outputs near zero have no meaningful relative
error).
"""

from __future__ import annotations


def source(n_gemm: int = 4096, n_fft: int = 4096) -> str:
    return (
        f"float ma[{n_gemm * n_gemm}];\nfloat mb[{n_gemm * n_gemm}];\nfloat mc[{n_gemm * n_gemm}];\n"
        f"float x[{2 * n_fft * n_fft}];\nfloat y[{2 * n_fft * n_fft}];\nfloat chk;\n\n"
        "func main() {\n  gemm(ma, mb, mc);\n  fft(x, y);\n  chk = mc[0] + y[0];\n}\n"
    )


def spec(n_gemm: int = 4096, n_fft: int = 4096, seed: int = 20240817) -> dict:
    return {
        "name": f"blocks_gemm{n_gemm}_fft{n_fft}",
        "precision": "fp32",
        "inputs": {
            "ma": {"kind": "uniform", "seed": seed, "lo": 0.0, "hi": 1.0},
            "mb": {"kind": "uniform", "seed": seed + 1, "lo": 0.0, "hi": 1.0},
            "x": {"kind": "uniform", "seed": seed + 2, "lo": -1.0, "hi": 1.0},
        },
        "outputs": {
            "mc": {"rel_tol": 1e-5},  # element-wise, the reference rule (3xTF32: 1.5e-6 at 4096^3)
            "y": {"rel_tol": 1e-5, "compare": "normwise"},
        },
        "externals": {"gemm": {"kind": "gemm", "out": 2}, "fft": {"kind": "fft2d", "out": 1}},
        "blocks": {"cublas_gemm": {"kind": "gemm"}, "cufft_exec": {"kind": "fft2d"}},
    }


def gemm_flops(n: int) -> int:
    return 2 * n ** 3


def fft_flops(n: int) -> float:
    import math

    return 5.0 * n * n * math.log2(n * n)
