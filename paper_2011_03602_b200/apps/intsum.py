"""Integer reduction app for the opt-in reduction screen (reductions.py,
SURVEY.md §8 f4): an int sum and a float sum over the same data, then a nest
that reads the int total.  Integer reductions reassociate exactly, so the
GPU result is bit-identical to the sequential loop; the float one is compared
at the tolerance its spec gives."""

from __future__ import annotations


def source(n: int = 1 << 16) -> str:
    return (
        "int i;\nint j;\nint cnt;\nfloat fs;\nint tot;\n"
        f"int d[{n}];\nfloat x[{n}];\nint e[{n}];\n\n"
        "func main() {\n  cnt = 0;\n  fs = 0.0;\n"
        f"  for (i = 0; i < {n}; i++) {{\n    cnt = cnt + d[i] * 3;\n    fs = fs + x[i];\n  }}\n"
        f"  for (j = 0; j < {n}; j++) {{\n    e[j] = d[j] + cnt;\n  }}\n"
        "  tot = cnt + e[0];\n}\n"
    )


def spec(n: int = 1 << 16, seed: int = 77) -> dict:
    return {
        "name": f"intsum_{n}",
        "precision": "fp32",
        "reductions": True,
        "inputs": {"d": {"kind": "randint", "seed": seed, "lo": -1000, "hi": 1000},
                   "x": {"kind": "uniform", "seed": seed + 1, "lo": 0.0, "hi": 1.0}},
        "outputs": {"cnt": {"rel_tol": 0.0}, "e": {"rel_tol": 0.0}, "tot": {"rel_tol": 0.0},
                    "fs": {"rel_tol": 1e-4}},
    }
