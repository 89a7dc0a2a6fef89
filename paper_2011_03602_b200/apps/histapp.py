"""Histogram app for the third record of the reference pattern DB
(``histogram`` -> ``cuda_histogram``, interface ``int[], int[]``,
fixtures/sample_db.json:20-28).

The program bins ``d`` twice: once with a loop the similarity matcher pairs
with the record's comparison snippet ``h[d[n]] = h[d[n]] + 1.0``
(``src/blocks.py`` loop path), once through an opaque ``histogram(d2, h2)``
call the name matcher pairs with the record's trigger names.  Both are
interface-compatible (all operands ``int[]``), so the block search measures
all four subsets; the unreplaced loop is also a GA gene (the reference screen
admits ``h[d[n]]`` because the write index mentions ``n``), and running it on
the GPU races on the bins, which the fitness reports as ``numeric_mismatch``
(SURVEY.md Appendix A.7).
"""

from __future__ import annotations


def source(n: int = 1 << 24, bins: int = 256) -> str:
    return (
        "int n;\nint chk;\n"
        f"int d[{n}];\nint h[{bins}];\nint d2[{n}];\nint h2[{bins}];\n\n"
        "func main() {\n"
        f"  for (n = 0; n < {n}; n++) {{\n    h[d[n]] = h[d[n]] + 1;\n  }}\n"
        "  histogram(d2, h2);\n"
        f"  chk = h[0] + h2[{bins - 1}];\n"
        "}\n"
    )


def spec(n: int = 1 << 24, bins: int = 256, seed: int = 1103) -> dict:
    return {
        "name": f"histogram_{n}_{bins}",
        "precision": "fp32",
        "inputs": {
            "d": {"kind": "randint", "seed": seed, "lo": 0, "hi": bins},
            "d2": {"kind": "randint", "seed": seed + 1, "lo": 0, "hi": bins},
        },
        # integer counts: bit-exact (rel_tol 0)
        "outputs": {"h": {"rel_tol": 0.0}, "h2": {"rel_tol": 0.0}, "chk": {"rel_tol": 0.0}},
        "externals": {"histogram": {"kind": "histogram", "out": 1}},
        "blocks": {"cuda_histogram": {"kind": "histogram"}},
    }


#: algorithmic bytes per element of d: one 4-byte read (bins stay on chip)
BYTES_PER_ELEMENT = 4
