"""Seeded random mini-language programs for differential testing of the GPU
path against the C oracle (tests/test_fuzz_gpu.py; fixtures made by
tests/golden/make_golden.py through the reference's parser, screen and
planner).

Programs mix every construct the compiler lowers differently: 1-3 deep
nests with constant, offset and zero-trip bounds (flat, quad and sequential
kernels), straight-line array bodies, point-local read-modify-writes, scalar
temporaries (lastprivate), screen-rejected reductions (host), int arrays and
scalars read by value.  They are hazard-free by construction -- a nest never
reads an array it writes except at the written index -- so every genome must
reproduce the sequential program bit for bit.
"""

from __future__ import annotations

import random

N = 8                   # loop extent per level
L = N * N * N + 16      # array length (room for +1 offsets)


def program(seed: int) -> str:
    rng = random.Random(seed)
    farr = [f"f{k}" for k in range(4)]
    iarr = ["n0"]
    lines = ["int i;", "int j;", "int k;", "int m;", "float s0;", "float s1;", "float t;", "int q = 3;",
             "float w = 0.5;", "float chk;"]
    lines += [f"float {a}[{L}];" for a in farr] + [f"int {a}[{L}];" for a in iarr]
    body = []
    for _ in range(rng.randint(2, 4)):
        depth = rng.choice([1, 2, 2, 3])
        idx = ["i", "j", "k"][:depth]
        # bounds: lower 0 or 1, upper N, N-1 or (rarely) 0 / 1 (zero / one trip)
        bounds = []
        for _d in idx:
            lo = rng.choice([0, 0, 1])
            hi = rng.choice([N, N, N - 1, N - 1, 0, 1]) if rng.random() < 0.15 else rng.choice([N, N - 1])
            bounds.append((lo, hi))
        flat = idx[0] if depth == 1 else (f"{idx[0]} * {N} + {idx[1]}" if depth == 2 else
                                         f"({idx[0]} * {N} + {idx[1]}) * {N} + {idx[2]}")
        written = rng.sample(farr, rng.choice([1, 2]))
        readable = [a for a in farr if a not in written]
        stmts = []
        kind = rng.random()
        for dst in written:
            src = rng.choice(readable)
            off = rng.choice([0, 1, 2])
            e = rng.choice([
                f"{src}[{flat} + {off}] * w + {dst}[{flat}]",
                f"{src}[{flat} + {off}] - {rng.choice(readable)}[{flat}] * 2.0",
                f"({src}[{flat}] + {src}[{flat} + 1]) * 0.25",
                f"{src}[{flat} + {off}] + q",
            ])
            stmts.append(f"{dst}[{flat}] = {e};")
        if kind < 0.12:  # scalar temporary, then used (screen-rejected: host or sequential kernel)
            src = rng.choice(readable)
            stmts = [f"t = {src}[{flat}] * 3.0;", f"{written[0]}[{flat}] = t + 1.0;"] + stmts[1:]
        elif kind < 0.22:  # reduction (screen-rejected)
            stmts.append(f"s0 = s0 + {rng.choice(readable)}[{flat}];")
        elif kind < 0.4:  # lastprivate scalar write
            stmts.append(f"s1 = {rng.choice(readable)}[{flat} + 1];")
        if rng.random() < 0.3:
            stmts.append(f"n0[{flat}] = n0[{flat}] + q;")
        text = "\n".join("    " + "  " * depth + s for s in stmts)
        nest = text
        for d in reversed(range(depth)):
            pad = "    " + "  " * d
            lo, hi = bounds[d]
            nest = f"{pad}for ({idx[d]} = {lo}; {idx[d]} < {hi}; {idx[d]}++) {{\n{nest}\n{pad}}}"
        body.append(nest)
        if rng.random() < 0.3:
            body.append(f"    s1 = s1 + {rng.choice(farr)}[{rng.randint(0, L - 1)}];")
    # an outer repeat loop around everything sometimes (transfer hoisting, multiplicities)
    inner = "\n".join(body)
    if rng.random() < 0.5:
        inner = "  for (m = 0; m < 2; m++) {\n" + inner + "\n  }"
    tail = f"  chk = s0 + s1 + f0[{rng.randint(0, L - 1)}] + f3[{L - 1}] + n0[5];"
    return "\n".join(lines) + "\n\nfunc main() {\n" + inner + "\n" + tail + "\n}\n"


def spec(seed: int) -> dict:
    return {
        "name": f"fuzz_{seed}",
        "precision": "fp32",
        "inputs": {
            "f0": {"kind": "uniform", "seed": seed, "lo": -1.0, "hi": 1.0},
            "f1": {"kind": "uniform", "seed": seed + 1, "lo": -1.0, "hi": 1.0},
            "f2": {"kind": "uniform", "seed": seed + 2, "lo": 0.0, "hi": 1.0},
            "f3": {"kind": "uniform", "seed": seed + 3, "lo": 0.0, "hi": 2.0},
            "n0": {"kind": "randint", "seed": seed + 4, "lo": -5, "hi": 5},
        },
        "outputs": {o: {"rel_tol": 1e-5} for o in ("f0", "f1", "f2", "f3", "n0", "s0", "s1", "chk")},
    }


SEEDS = list(range(96))
