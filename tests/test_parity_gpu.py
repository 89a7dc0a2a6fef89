"""GPU parity: every genome of every small app, executed through the C ABI
(B200Evaluator -> libb2o.so -> compiled sm_100a kernels), must reproduce the C
oracle's final state (oracle/cgen.py, itself pinned to oracle/interp.py) and
execute exactly the plan's directive multiplicities
(``TransferDirective.multiplicity``, src/transfers.py:176-188)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import SMALL_APPS, golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oracle_cache():
    return {}


def _oracle_state(name, g, cache):
    if name not in cache:
        from oracle.cgen import CProgram
        from oracle.externals import make_binder
        from paper_2011_03602_b200 import appspec
        from paper_2011_03602_b200.ir import Program

        prog = Program(g["doc"])
        state = appspec.initial_state(prog, g["spec"])
        cache[name] = (prog, CProgram(g["doc"], g["spec"].get("precision", "fp32")).run(
            state, make_binder(g["doc"], g["spec"])))
    return cache[name]


@pytest.fixture(scope="module")
def evaluators():
    from paper_2011_03602_b200.evaluator import B200Evaluator

    made = {}

    def get(name, spec, **kw):
        key = (name, tuple(sorted(kw.items())))
        if key not in made:
            made[key] = B200Evaluator(spec, devices=[0], **kw)
        return made[key]

    return get


def _close(a, b, rel):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.all(np.abs(a - b) <= np.maximum(rel * np.abs(b), 1e-12))


@pytest.mark.parametrize("name", SMALL_APPS)
def test_all_genomes_match_oracle(name, evaluators, oracle_cache):
    g = golden(name)
    prog, want = _oracle_state(name, g, oracle_cache)
    ev = evaluators(name, g["spec"])
    genomes = sorted(g["patterns"])
    payloads = [g["patterns"][x] for x in genomes]
    results = ev.measure_payloads(g["doc"], payloads)
    app = ev.app_for(g["doc"])
    outputs = [prog.var_by_name[o].id for o in g["spec"]["outputs"]]
    for x, r in zip(genomes, results):
        assert r["validity"] == "valid", (name, x, r["diag"])
        assert r["time_s"] > 0
        execs = sum(d["multiplicity"] for d in g["patterns"][x]["directives"])
        assert r["directive_execs"] == execs, (name, x)
        if any(b == "1" for b in x):
            assert r["launches"] > 0, (name, x)
        else:
            assert r["launches"] == 0
    # replay each genome alone to read its final state and compare with the oracle
    for x in genomes:
        r = ev.measure_payloads(g["doc"], [g["patterns"][x]])[0]
        for vid in outputs:
            got = app.read(vid, worker=r["worker"])
            assert _close(got, want[vid], 1e-5), (name, x, prog.vars[vid].name)


def test_himeno_bit_exact(evaluators, oracle_cache):
    """Kernels are compiled without FMA contraction (exact C semantics, the
    compiler default): the GPU evaluates the same expression tree in the same
    order as the CPU oracle, so results are bit-identical."""
    g = golden("himeno_17x9x33")
    spec = g["spec"]
    prog, want = _oracle_state("himeno_17x9x33", g, oracle_cache)
    ev = evaluators("himeno_17x9x33", spec)
    app = ev.app_for(g["doc"])
    for x in ("100100", "010010", "001001"):
        r = ev.measure_payloads(g["doc"], [g["patterns"][x]])[0]
        assert r["validity"] == "valid" and r["max_rel_err"] == 0.0, r
        for name in ("p", "gs", "gosa"):
            vid = prog.var_by_name[name].id
            assert np.array_equal(app.read(vid, worker=r["worker"]), want[vid]), (x, name)


def test_literal_mode_exposes_unfetched_output(evaluators):
    """without a final host read of ``p`` the reference plan
    for genome 100100 never brings ``p`` back (src/transfers.py:105-110).
    Executed literally the host copy is stale; the coherent manager fetches it
    and reports the bytes as epilogue (untimed) traffic."""
    g = golden("himeno_xs_noread")
    pat = g["patterns"]["100100"]
    from paper_2011_03602_b200.ir import Program

    pid = Program(g["doc"]).var_by_name["p"].id
    assert not any(d["var"] == pid and d["dir"] == "d2h" for d in pat["directives"])
    lit = evaluators("noread_literal", g["spec"], mode="literal").measure_payloads(g["doc"], [pat])[0]
    coh = evaluators("noread_coherent", g["spec"]).measure_payloads(g["doc"], [pat])[0]
    assert lit["validity"] == "numeric_mismatch", lit
    assert coh["validity"] == "valid" and coh["epilogue_bytes"] > 0, coh


def test_literal_equals_coherent_when_plan_is_complete(evaluators):
    """For Himeno with the final read, every plan is sufficient: literal and
    coherent execution agree and the coherent manager adds no unplanned
    traffic beyond write-only first touches."""
    g = golden("himeno_17x9x33")
    lit = evaluators("h_literal", g["spec"], mode="literal")
    for x in ("100100", "100000", "000100", "001001", "111111"):
        r = lit.measure_payloads(g["doc"], [g["patterns"][x]])[0]
        assert r["validity"] == "valid" and r["stale_reads"] == 0, (x, r)


def test_hoisted_plan_moves_fewer_bytes_than_unhoisted(evaluators):
    """The hoisting rule (src/transfers.py:120-191) realised on the device:
    the four_loops genome-101 plan executes fewer directive instances."""
    g = golden("four_loops")
    ev = evaluators("four_loops", g["spec"])
    hoisted, raw = ev.measure_payloads(g["doc"], [g["patterns"]["101"], g["unhoisted"]["101"]])
    assert hoisted["validity"] == raw["validity"] == "valid"
    assert hoisted["directive_execs"] < raw["directive_execs"]
    assert hoisted["directive_execs"] == sum(d["multiplicity"] for d in g["patterns"]["101"]["directives"])


def test_timeout_maps_to_timeout(evaluators):
    g = golden("himeno_17x9x33")
    ev = evaluators("himeno_timeout", g["spec"], timeout_seconds=1e-6)
    r = ev.measure_payloads(g["doc"], [g["patterns"]["000000"]])[0]
    assert r["validity"] == "timeout", r


def test_pattern_for_another_program_is_rejected(evaluators):
    """A pattern naming loops the program does not have never raises out of
    the evaluator: it comes back infeasible (src/evaluators.py:23-27)."""
    g = golden("blocks_nest64")
    variant = next(v for v in g["variants"] if v["subset"])
    ev = evaluators("blocks_nest64", g["spec"])
    r = ev.measure_payloads(variant["doc"], [{"gpu_roots": [0], "directives": []}])[0]
    assert r["validity"] in ("compile_error", "runtime_error"), r
