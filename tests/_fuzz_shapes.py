"""Seeded random programs aimed at the specialised kernel shapes (differential
testing against the C oracle; fixtures tests/golden/fuzz_shapes.json made by
tests/golden/make_golden.py through the reference's parser, screen and
planner):

* ``ktile``  -- (i, j) nests around a sequential k loop: random extents (not
  multiples of the 64 x 64 tile or the 32-deep stage), both operand layouts
  ((i, k) / (k, i) and (k, j) / (j, k)), accumulation with or without an
  initialising statement, subtraction, scalar factors, a post statement into
  a second accumulator, an outer repeat loop (compiler.ktile_plan);
* ``march``  -- 3-D stencils on n^3 grids with n even (plane stride a multiple
  of the quad), random subsets of the 27 neighbours, optionally a correction
  nest and an outer repeat loop (compiler.march_plan);
* ``reduce`` -- fp32 scalar reductions s = s + e / s = s - e with a float
  term over 1- to 3-deep nests, run under the opt-in reduction screen
  (reductions.py): summed exactly in loop order on the GPU (b2o_xsum.cu).

Every program is hazard-free, so every genome must leave the oracle's final
state bit for bit.
"""

from __future__ import annotations

import random

SEEDS = list(range(90))  # 12 per original family, 18 per second-generation family


def family(seed: int) -> str:
    if seed < 36:
        return ("ktile", "march", "reduce")[seed % 3]
    return ("ktile2", "march2", "reduce2")[seed % 3]


def _ktile(rng: random.Random) -> str:
    ni, nj, nk = rng.choice([33, 64, 70]), rng.choice([17, 64, 80]), rng.choice([16, 31, 40, 65])
    a = rng.choice([f"a[i * {nk} + k]", f"a[k * {ni} + i]"])
    b = rng.choice([f"b[k * {nj} + j]", f"b[j * {nk} + k]"])
    c = f"c[i * {nj} + j]"
    upd = rng.choice([f"{c} = {c} + {a} * {b};", f"{c} = {c} - {a} * {b};", f"{c} = {c} + {a} * {b} * w;",
                      f"{c} = {c} + ({a} + w) * {b};"])
    init = rng.choice(["", f"{c} = 0.0;", f"{c} = d[i * {nj} + j] * w;"])
    post = rng.choice(["", f"e[i * {nj} + j] = {c} * 2.0;"])
    n = max(ni, nj, nk) ** 2
    lines = ["int i;", "int j;", "int k;", "int m;", "float w = 0.75;", "float chk;"]
    lines += [f"float {x}[{n}];" for x in "abcde"]
    nest = (f"    for (i = 0; i < {ni}; i++) {{\n      for (j = 0; j < {nj}; j++) {{\n"
            + (f"        {init}\n" if init else "")
            + f"        for (k = 0; k < {nk}; k++) {{\n          {upd}\n        }}\n"
            + (f"        {post}\n" if post else "") + "      }\n    }\n")
    if rng.random() < 0.4:
        nest = "  for (m = 0; m < 2; m++) {\n" + nest + "  }\n"
    return "\n".join(lines) + "\n\nfunc main() {\n" + nest + f"  chk = c[{nj + 1}] + e[3];\n}}\n"


def _march(rng: random.Random) -> str:
    n = rng.choice([12, 16, 20])

    def ix(d3=0, d2=0, d1=0):
        def t(name, d):
            return name if d == 0 else (f"({name} + {d})" if d > 0 else f"({name} - {-d})")
        return f"({t('i3', d3)} * {n} + {t('i2', d2)}) * {n} + {t('i1', d1)}"

    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1) if (a, b, c) != (0, 0, 0)]
    pick = rng.sample(offs, rng.randint(4, 12))
    if all(o[0] == 0 for o in pick):
        pick.append((1, 0, 0))
    terms = " + ".join(f"u[{ix(*o)}]" for o in pick)
    res = f"r[{ix()}] = v[{ix()}] - c0 * u[{ix()}] - c1 * ({terms});"
    corr = f"u[{ix()}] = u[{ix()}] + w * r[{ix()}];"

    def nest(line):
        return (f"    for (i3 = 1; i3 < {n - 1}; i3++) {{\n      for (i2 = 1; i2 < {n - 1}; i2++) {{\n"
                f"        for (i1 = 1; i1 < {n - 1}; i1++) {{\n          {line}\n        }}\n      }}\n    }}\n")

    body = nest(res) + (nest(corr) if rng.random() < 0.6 else "")
    if rng.random() < 0.5:
        body = "  for (it = 0; it < 2; it++) {\n" + body + "  }\n"
    m = n ** 3
    return ("int it;\nint i1;\nint i2;\nint i3;\nfloat c0 = 0.0 - 8.0 / 3.0;\nfloat c1 = 1.0 / 12.0;\n"
            f"float w = 0.25;\nfloat chk;\nfloat u[{m}];\nfloat v[{m}];\nfloat r[{m}];\n\nfunc main() {{\n"
            + body + f"  chk = r[{n * n + n + 1}] + u[0];\n}}\n")


def _reduce(rng: random.Random) -> str:
    n = rng.choice([40, 64, 96])
    lines = ["int i;", "int j;", "int k;", "int m;", "float w = 0.5;", "float s0;", "float s1;", "float chk;"]
    lines += [f"float {x}[{n * n * n}];" for x in "abd"]
    body = []
    for _ in range(rng.randint(1, 3)):
        depth = rng.choice([1, 2, 3])
        idx = ["i", "j", "k"][:depth]
        flat = idx[0] if depth == 1 else (f"{idx[0]} * {n} + {idx[1]}" if depth == 2 else
                                         f"({idx[0]} * {n} + {idx[1]}) * {n} + {idx[2]}")
        s = rng.choice(["s0", "s1"])
        term = rng.choice([f"a[{flat}] * b[{flat}]", f"a[{flat}]", f"b[{flat}] * w", f"a[{flat}] - b[{flat}]"])
        op = rng.choice(["+", "+", "-"])
        stmts = [f"{s} = {s} {op} {term};"]
        if rng.random() < 0.4:
            stmts.append(f"d[{flat}] = a[{flat}] + w;")
        rng.shuffle(stmts)
        text = "\n".join("    " + "  " * depth + x for x in stmts)
        for d in reversed(range(depth)):
            pad = "    " + "  " * d
            lo = rng.choice([0, 1])
            text = f"{pad}for ({idx[d]} = {lo}; {idx[d]} < {n}; {idx[d]}++) {{\n{text}\n{pad}}}"
        if rng.random() < 0.5:
            text = f"    {s} = {rng.choice(['0.0', 'w', '2.0'])};\n" + text
        body.append(text)
    inner = "\n".join(body)
    if rng.random() < 0.4:
        inner = "  for (m = 0; m < 2; m++) {\n" + inner + "\n  }"
    return "\n".join(lines) + "\n\nfunc main() {\n" + inner + "\n  chk = s0 + s1 + d[7];\n}\n"


def _ktile2(rng: random.Random) -> str:
    """Several k-loop statements: two updates of one accumulator, a second
    accumulator, constant operand offsets."""
    ni, nj, nk = rng.choice([40, 64, 72]), rng.choice([24, 64, 66]), rng.choice([8, 33, 48])
    a = rng.choice([f"a[i * {nk} + k]", f"a[k * {ni} + i + 1]"])
    b = rng.choice([f"b[k * {nj} + j]", f"b[j * {nk} + k + 2]"])
    c, e = f"c[i * {nj} + j]", f"e[i * {nj} + j]"
    body = [f"{c} = {c} + {a} * {b};"]
    body.append(rng.choice([f"{c} = {c} - {a} * w;", f"{e} = {e} + {b};", f"{e} = {e} * w + {a};"]))
    if rng.random() < 0.5:
        body.append(f"{c} = {c} * 0.5 + {b};")
    init = rng.choice(["", f"{c} = 1.0;\n        {e} = 0.0;", f"{e} = d[i * {nj} + j];"])
    n = (max(ni, nj, nk) + 4) ** 2
    lines = ["int i;", "int j;", "int k;", "float w = 0.625;", "float chk;"] + [f"float {x}[{n}];" for x in "abcde"]
    nest = (f"    for (i = 0; i < {ni}; i++) {{\n      for (j = 0; j < {nj}; j++) {{\n"
            + (f"        {init}\n" if init else "")
            + f"        for (k = 0; k < {nk}; k++) {{\n" + "".join(f"          {x}\n" for x in body) + "        }\n"
            + "      }\n    }\n")
    return "\n".join(lines) + "\n\nfunc main() {\n" + nest + f"  chk = c[{nj + 1}] + e[3];\n}}\n"


def _march2(rng: random.Random) -> str:
    """Two statements per point (two outputs from the same neighbours), plane
    offsets of two arrays."""
    n = rng.choice([12, 16])

    def ix(d3=0, d2=0, d1=0):
        def t(name, d):
            return name if d == 0 else (f"({name} + {d})" if d > 0 else f"({name} - {-d})")
        return f"({t('i3', d3)} * {n} + {t('i2', d2)}) * {n} + {t('i1', d1)}"

    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]
    pu = rng.sample(offs, rng.randint(3, 8)) + [(1, 0, 0)]
    pv = rng.sample(offs, rng.randint(1, 4))
    tu = " + ".join(f"u[{ix(*o)}]" for o in pu)
    tv = " + ".join(f"v[{ix(*o)}]" for o in pv)
    lines = [f"r[{ix()}] = c1 * ({tu}) - {tv};", f"q[{ix()}] = u[{ix()}] * c0 + v[{ix(1, 0, 0)}];"]
    rng.shuffle(lines)
    body = (f"    for (i3 = 1; i3 < {n - 1}; i3++) {{\n      for (i2 = 1; i2 < {n - 1}; i2++) {{\n"
            f"        for (i1 = 1; i1 < {n - 1}; i1++) {{\n" + "".join(f"          {x}\n" for x in lines)
            + "        }\n      }\n    }\n")
    m = n ** 3
    return ("int i1;\nint i2;\nint i3;\nfloat c0 = 0.5;\nfloat c1 = 1.0 / 6.0;\nfloat chk;\n"
            f"float u[{m}];\nfloat v[{m}];\nfloat r[{m}];\nfloat q[{m}];\n\nfunc main() {{\n"
            + body + f"  chk = r[{n * n + n + 1}] + q[{n * n + n + 2}];\n}}\n")


def _reduce2(rng: random.Random) -> str:
    """Two fp32 reductions and an int reduction in one nest."""
    n = rng.choice([32, 48, 64])
    lines = ["int i;", "int j;", "int k;", "int cnt;", "float w = 0.5;", "float s0;", "float s1;", "float chk;",
             f"float a[{n * n * n}];", f"float b[{n * n * n}];", f"int t[{n * n * n}];"]
    depth = rng.choice([2, 3])
    idx = ["i", "j", "k"][:depth]
    flat = f"{idx[0]} * {n} + {idx[1]}" if depth == 2 else f"({idx[0]} * {n} + {idx[1]}) * {n} + {idx[2]}"
    stmts = [f"s0 = s0 + a[{flat}] * w;", f"s1 = s1 - b[{flat}];", f"cnt = cnt + t[{flat}];"]
    rng.shuffle(stmts)
    text = "\n".join("    " + "  " * depth + x for x in stmts)
    for d in reversed(range(depth)):
        pad = "    " + "  " * d
        text = f"{pad}for ({idx[d]} = 0; {idx[d]} < {n}; {idx[d]}++) {{\n{text}\n{pad}}}"
    return "\n".join(lines) + "\n\nfunc main() {\n" + text + "\n  chk = s0 + s1 + cnt;\n}\n"


def program(seed: int) -> str:
    rng = random.Random(1000 + seed)
    return {"ktile": _ktile, "march": _march, "reduce": _reduce, "ktile2": _ktile2, "march2": _march2,
            "reduce2": _reduce2}[family(seed)](rng)


def spec(seed: int) -> dict:
    fam = family(seed)
    arrays = {"ktile": "abcde", "march": ("u", "v", "r"), "reduce": "abd", "ktile2": "abcde",
              "march2": ("u", "v", "r", "q"), "reduce2": ("a", "b", "t")}[fam]
    inputs = {x: {"kind": "uniform", "seed": 7 * seed + i, "lo": -1.0 if i % 2 else 0.0, "hi": 1.0}
              for i, x in enumerate(arrays)}
    if fam == "reduce2":
        inputs["t"] = {"kind": "randint", "seed": 7 * seed + 9, "lo": -3, "hi": 4}
    outs = list(arrays) + ["chk"] + (["s0", "s1"] if fam.startswith("reduce") else []) + \
        (["cnt"] if fam == "reduce2" else [])
    sp = {"name": f"shapes_{seed}", "precision": "fp32", "inputs": inputs,
          "outputs": {o: {"rel_tol": 1e-5} for o in outs}}
    if fam.startswith("reduce"):
        sp["reductions"] = True
    return sp
