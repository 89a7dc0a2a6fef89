"""NAS-MG-style residual app for the Java-source path (BASELINE config 4).

The ``resid`` kernel of NPB MG (r = v - A u with the 27-point operator,
coefficients a = (-8/3, 0, 1/6, 1/12), so the a(1) face terms vanish) written
inline (no temporaries, no unary minus: constants come from initialised
scalars), followed by a correction nest ``u = u + omega * r``, iterated
``nit`` times.  Layout is C row-major ``(i3 * n + i2) * n + i1`` with i1
fastest (Fortran ``u(i1,i2,i3)``).  The program enters the pipeline as an IR
document tagged ``language: java_like`` (SPEC.md §3.1 multi-language core).
"""

from __future__ import annotations


def _ix(n: int, d3: int = 0, d2: int = 0, d1: int = 0) -> str:
    def t(name, d):
        return name if d == 0 else (f"({name} + {d})" if d > 0 else f"({name} - {-d})")

    return f"({t('i3', d3)} * {n} + {t('i2', d2)}) * {n} + {t('i1', d1)}"


def source(n: int = 258, nit: int = 4) -> str:
    u = lambda d3, d2, d1: f"u[{_ix(n, d3, d2, d1)}]"  # noqa: E731
    u1 = lambda d: f"({u(0, -1, d)} + {u(0, 1, d)} + {u(-1, 0, d)} + {u(1, 0, d)})"  # noqa: E731
    u2 = lambda d: f"({u(-1, -1, d)} + {u(-1, 1, d)} + {u(1, -1, d)} + {u(1, 1, d)})"  # noqa: E731
    x = _ix(n)
    resid = (f"r[{x}] = v[{x}] - ca0 * {u(0, 0, 0)} - ca2 * ({u2(0)} + {u1(-1)} + {u1(1)})"
             f" - ca3 * ({u2(-1)} + {u2(1)});")
    corr = f"u[{x}] = u[{x}] + omega * r[{x}];"

    def nest(line):
        return (f"    for (i3 = 1; i3 < {n - 1}; i3++) {{\n"
                f"      for (i2 = 1; i2 < {n - 1}; i2++) {{\n"
                f"        for (i1 = 1; i1 < {n - 1}; i1++) {{\n"
                f"          {line}\n        }}\n      }}\n    }}\n")

    m = n ** 3
    return (
        "int it;\nint i1;\nint i2;\nint i3;\n"
        f"int nit = {nit};\n"
        "float ca0 = 0.0 - 8.0 / 3.0;\nfloat ca2 = 1.0 / 6.0;\nfloat ca3 = 1.0 / 12.0;\n"
        "float omega = 0.25;\nfloat chk;\n"
        f"float u[{m}];\nfloat v[{m}];\nfloat r[{m}];\n\n"
        "func main() {\n  for (it = 0; it < nit; it++) {\n"
        + nest(resid) + nest(corr)
        + f"  }}\n  chk = r[{n * n + n + 1}] + u[0];\n}}\n"
    )


def java_source(n: int = 258, nit: int = 4) -> str:
    """The same program as a Java class (NPB-JAV style: static arrays, the
    27-point operator inline), for the java frontend
    (frontends/java_src.py); it lowers to an IR whose oracle results equal
    :func:`source`'s bit for bit (tests/test_frontends.py)."""
    def ix(d3=0, d2=0, d1=0):
        def t(name, d):
            return name if d == 0 else (f"({name} + {d})" if d > 0 else f"({name} - {-d})")
        return f"({t('i3', d3)} * N + {t('i2', d2)}) * N + {t('i1', d1)}"

    u = lambda d3, d2, d1: f"u[{ix(d3, d2, d1)}]"  # noqa: E731
    u1 = lambda d: f"({u(0, -1, d)} + {u(0, 1, d)} + {u(-1, 0, d)} + {u(1, 0, d)})"  # noqa: E731
    u2 = lambda d: f"({u(-1, -1, d)} + {u(-1, 1, d)} + {u(1, -1, d)} + {u(1, 1, d)})"  # noqa: E731
    x = ix()
    resid = (f"r[{x}] = v[{x}] - ca0 * {u(0, 0, 0)} - ca2 * ({u2(0)} + {u1(-1)} + {u1(1)})"
             f" - ca3 * ({u2(-1)} + {u2(1)});")

    def nest(line):
        return ("            for (i3 = 1; i3 < N - 1; i3++) {\n"
                "                for (i2 = 1; i2 < N - 1; i2++) {\n"
                "                    for (i1 = 1; i1 < N - 1; i1++) {\n"
                f"                        {line}\n"
                "                    }\n                }\n            }\n")

    return (
        "package npb;\n\n/** NAS-MG resid + correction (NPB-JAV style). */\n"
        "public class MGResid {\n"
        f"    static final int N = {n};\n"
        "    static int it, i1, i2, i3;\n"
        f"    static int nit = {nit};\n"
        "    static float ca0 = 0.0f - 8.0f / 3.0f, ca2 = 1.0f / 6.0f, ca3 = 1.0f / 12.0f;\n"
        "    static float omega = 0.25f;\n"
        "    static float chk;\n"
        "    static float[] u = new float[N * N * N];\n"
        "    static float[] v = new float[N * N * N];\n"
        "    static float[] r = new float[N * N * N];\n\n"
        "    public static void main(String[] args) {\n"
        "        for (it = 0; it < nit; it++) {\n"
        + nest(resid) + nest(f"u[{x}] = u[{x}] + omega * r[{x}];")
        + "        }\n"
        f"        chk = r[{n * n + n + 1}] + u[0];\n"
        "    }\n}\n"
    )


def spec(n: int = 258, seed: int = 550) -> dict:
    return {
        "name": f"nasmg_resid_{n}",
        "language": "java_like",
        "precision": "fp32",
        "inputs": {
            "u": {"kind": "uniform", "seed": seed, "lo": 0.0, "hi": 1.0},
            "v": {"kind": "uniform", "seed": seed + 1, "lo": 0.0, "hi": 1.0},
        },
        "outputs": {"u": {"rel_tol": 1e-5}, "r": {"rel_tol": 1e-5}, "chk": {"rel_tol": 1e-5}},
    }


#: algorithmic bytes per interior point: resid reads u (neighbours cached) and
#: v, writes r; the correction reads u and r and writes u.
RESID_BYTES_PER_POINT = 12
CORR_BYTES_PER_POINT = 12
