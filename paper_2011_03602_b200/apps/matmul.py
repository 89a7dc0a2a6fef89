"""Naive matmul loop nest (the reference fixture ``fixtures/matmul.mini``
scaled to N), plus a final host read so the result is
fetched.  Screen: i ok, j ok, k non_affine_array_write
(``tests/test_screen.py:42-46``), so a=2 and the GA sweeps 4 genomes
(``src/ga.py:262-264``)."""

from __future__ import annotations


def source(n: int = 1024) -> str:
    return (
        "int i;\nint j;\nint k;\n"
        f"float ma[{n * n}];\nfloat mb[{n * n}];\nfloat mc[{n * n}];\nfloat chk;\n\n"
        "func main() {\n"
        f"  for (i = 0; i < {n}; i++) {{\n"
        f"    for (j = 0; j < {n}; j++) {{\n"
        f"      mc[i * {n} + j] = 0.0;\n"
        f"      for (k = 0; k < {n}; k++) {{\n"
        f"        mc[i * {n} + j] = mc[i * {n} + j] + ma[i * {n} + k] * mb[k * {n} + j];\n"
        "      }\n    }\n  }\n"
        "  chk = mc[0];\n}\n"
    )


def python_source(n: int = 1024) -> str:
    """The same program as real Python (BASELINE config 1 is a *Python*
    matmul app): lowered by frontends/python_src.py to the same IR as
    :func:`source` (tests/test_frontends.py)."""
    return (
        '"""Naive matmul: the paper\'s Python loop-offload example shape."""\n'
        "import numpy as np\n\n"
        f"N = {n}\n"
        "ma = np.zeros(N * N, dtype=np.float32)\n"
        "mb = np.zeros(N * N, dtype=np.float32)\n"
        "mc = np.zeros(N * N, dtype=np.float32)\n"
        "chk = 0.0\n\n\n"
        "def main():\n"
        "    global chk\n"
        "    for i in range(N):\n"
        "        for j in range(N):\n"
        "            mc[i * N + j] = 0.0\n"
        "            for k in range(N):\n"
        "                mc[i * N + j] = mc[i * N + j] + ma[i * N + k] * mb[k * N + j]\n"
        "    chk = mc[0]\n\n\n"
        'if __name__ == "__main__":\n'
        "    main()\n"
    )


def spec(n: int = 1024, seed: int = 2011036021) -> dict:
    return {
        "name": f"matmul_{n}",
        "language": "python_like",
        "precision": "fp32",
        "inputs": {
            "ma": {"kind": "uniform", "seed": seed, "lo": 0.0, "hi": 1.0},
            "mb": {"kind": "uniform", "seed": seed + 1, "lo": 0.0, "hi": 1.0},
        },
        "outputs": {"mc": {"rel_tol": 1e-5}, "chk": {"rel_tol": 1e-5}},
    }


def flops(n: int) -> int:
    return 2 * n ** 3
