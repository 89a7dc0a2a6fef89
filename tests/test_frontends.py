"""Language edges: Python and Java sources lowered to the
reference's IR document through its own parser.

* The Python matmul (BASELINE config 1 is a *Python* app) and the Java NAS-MG
  class (config 4 is a *Java* app) lower to programs whose oracle results
  equal the mini-language apps' bit for bit, with the same screen verdicts,
  genome and transfer plans as computed by the reference.
* The lowering is checked against the source language itself: a Python
  program run by CPython (float64 numpy arrays) equals the C oracle of its IR
  at fp64 exactly.
* Unsupported constructs fail with the offending line.
"""

import json

import numpy as np
import pytest

from conftest import has_reference
from oracle.cgen import CProgram
from oracle.interp import run_program
from paper_2011_03602_b200 import appspec
from paper_2011_03602_b200.apps import matmul, nasmg
from paper_2011_03602_b200.frontends import FrontendError
from paper_2011_03602_b200.frontends.java_src import java_precision, java_to_mini
from paper_2011_03602_b200.frontends.python_src import python_to_mini
from paper_2011_03602_b200.ir import Program

pytestmark = pytest.mark.skipif(not has_reference(), reason="reference parser not importable")


def _doc(mini, language=None):
    from gpuoffload.irdoc import model_to_document
    from gpuoffload.minilang import parse_mini_source

    from paper_2011_03602_b200.frontends import to_document

    return to_document(mini, language) if language else model_to_document(parse_mini_source(mini))


def _final(doc, spec):
    st = appspec.initial_state(Program(doc), spec)
    return CProgram(doc, spec.get("precision", "fp32")).run(st)


def _by_name(doc, state):
    return {v["name"]: state[v["id"]] for v in doc["variables"]}


def _plans(doc):
    from gpuoffload.irdoc import load_ir_document
    from gpuoffload.patterns import build_genome_space, pattern_from_genome
    from gpuoffload.screen import screen_model
    from gpuoffload.transfers import plan_transfers

    m = load_ir_document(json.dumps(doc))
    verdicts = screen_model(m)
    space = build_genome_space(m, verdicts)
    out = {}
    for g in space.all_genomes():
        p = pattern_from_genome(m, space, g)
        plan = plan_transfers(m, p)
        out[p.genome_text] = sorted((m.var(d.var_id).name, d.direction, d.multiplicity) for d in plan.directives)
    return [v.reason for v in verdicts], out


@pytest.mark.parametrize("lang", ["python", "java"])
def test_source_apps_equal_mini_apps(lang):
    if lang == "python":
        src_doc = _doc(python_to_mini(matmul.python_source(24)), "python_like")
        mini_doc = _doc(matmul.source(24))
        spec = matmul.spec(24)
    else:
        src = nasmg.java_source(10, 2)
        assert java_precision(src) == "fp32"
        src_doc = _doc(java_to_mini(src), "java_like")
        mini_doc = _doc(nasmg.source(10, 2))
        spec = nasmg.spec(10)
    assert src_doc["language"] == ("python_like" if lang == "python" else "java_like")
    a = _by_name(src_doc, _final(src_doc, spec))
    b = _by_name(mini_doc, _final(mini_doc, spec))
    for name in spec["outputs"]:
        assert np.array_equal(a[name], b[name]), name
    assert _plans(src_doc) == _plans(mini_doc)


PY_PROGRAM = '''
import numpy as np
N = 12
K = 3
x = np.zeros(N * N, dtype=np.float64)
y = np.zeros(N * N, dtype=np.float64)
hist = [0] * N
alpha = 0.75
total: float = 0.0
cnt: int


def smooth(a, b):
    for i in range(1, N - 1):
        for j in range(1, N - 1):
            b[i * N + j] = (a[(i - 1) * N + j] + a[(i + 1) * N + j] + a[i * N + j - 1] + a[i * N + j + 1]) / 4.0


def main():
    global total, cnt
    for t in range(K):
        smooth(x, y)
        for i in range(N * N):
            x[i] = y[i] * alpha - -x[i] / 3
    for i in range(N):
        for j in range(N):
            total += x[i * N + j] * (i + 1) / (j + 1)
    cnt = 0
    for i in range(N * N):
        cnt += (i * 7) // 5 - i // 2
        hist[i // N] = hist[i // N] + 1
'''


def test_python_lowering_matches_cpython():
    mini = python_to_mini(PY_PROGRAM)
    doc = _doc(mini, "python_like")
    prog = Program(doc)
    spec = {"precision": "fp64", "inputs": {"x": {"kind": "uniform", "seed": 5, "lo": -1.0, "hi": 1.0}}}
    st = appspec.initial_state(prog, spec)
    got = _by_name(doc, run_program(doc, st, "fp64"))
    ns: dict = {}
    exec(compile(PY_PROGRAM, "<program>", "exec"), ns)  # noqa: S102 - the test program above
    ns["x"][:] = st[prog.var_by_name["x"].id]
    ns["main"]()
    for name in ("x", "y"):
        assert np.array_equal(got[name], ns[name]), name
    assert got["total"][0] == ns["total"]
    assert int(got["cnt"][0]) == ns["cnt"]
    assert np.array_equal(got["hist"], np.asarray(ns["hist"]))


@pytest.mark.parametrize("src,where", [
    ("def main():\n    while True:\n        pass\n", 2),
    ("a = [0.0] * 4\ndef main():\n    for i in range(0, 4, 2):\n        a[i] = 1.0\n", 3),
    ("a = [0.0] * 4\ndef main():\n    a[0], a[1] = 1.0, 2.0\n", 3),
    ("a = [1.0] * 4\ndef main():\n    pass\n", 1),
    ("a = [0.0] * 4\ndef main():\n    a[0] = 2.0 // 3.0\n", 3),
    ("a = [0.0] * 4\ndef main():\n    if a[0]:\n        a[1] = 1.0\n", 3),
])
def test_python_rejects_outside_subset(src, where):
    with pytest.raises(FrontendError) as e:
        python_to_mini(src)
    assert e.value.line == where


@pytest.mark.parametrize("body,where", [
    ("while (it < 3) { it++; }", 5),
    ("if (it < 3) { it = 1; }", 5),
    ("x = Math.sqrt(x);", 5),
    ("x = (float) it;", 5),
    ("for (it = 0; it < 4; it += 2) { x = 1.0f; }", 5),
])
def test_java_rejects_outside_subset(body, where):
    src = ("class T {\n  static int it;\n  static float x;\n  public static void main(String[] a) {\n"
           f"    {body}\n  }}\n}}\n")
    with pytest.raises(FrontendError) as e:
        java_to_mini(src)
    assert e.value.line == where


def test_java_double_program_reports_fp64():
    src = "class T {\n static double s;\n static void main() {\n  s = s + 1.5;\n }\n}\n"
    assert java_precision(src) == "fp64"
    assert "float s;" in java_to_mini(src)


@pytest.mark.gpu
@pytest.mark.parametrize("lang", ["python", "java"])
def test_source_apps_on_b200(lang):
    """Every genome of the Python matmul / Java NAS-MG (reference screen and
    planner) runs on the B200 and matches the C oracle."""
    from gpuoffload.irdoc import load_ir_document
    from gpuoffload.patterns import build_genome_space, pattern_from_genome
    from gpuoffload.screen import screen_model
    from gpuoffload.transfers import plan_transfers

    from gpuoffload.evaluators import EvaluationRequest

    from paper_2011_03602_b200.evaluator import B200Evaluator, payload_from_request

    if lang == "python":
        doc, spec = _doc(python_to_mini(matmul.python_source(48)), "python_like"), matmul.spec(48)
    else:
        doc, spec = _doc(java_to_mini(nasmg.java_source(18, 2)), "java_like"), nasmg.spec(18)
    want = _by_name(doc, _final(doc, spec))
    m = load_ir_document(json.dumps(doc))
    space = build_genome_space(m, screen_model(m))
    ev = B200Evaluator(spec, devices=[0])
    app = ev.app_for(doc)
    prog = Program(doc)
    for g in space.all_genomes():
        p = pattern_from_genome(m, space, g)
        req = EvaluationRequest(m, p, plan_transfers(m, p), "", "c_openacc")
        r = ev.measure_payloads(doc, [payload_from_request(req)])[0]
        assert r["validity"] == "valid", (lang, p.genome_text, r["diag"])
        for name in spec["outputs"]:
            got = app.read(prog.var_by_name[name].id, worker=r["worker"])
            np.testing.assert_allclose(got, want[name], rtol=1e-5, atol=1e-12)
