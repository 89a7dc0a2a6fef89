"""GPU parity: every genome of every small app, executed through the C ABI
(B200Evaluator -> libb2o.so -> compiled sm_100a kernels), must reproduce, bit for bit,
the final state of the reference's own C emission (oracle/_ref; the C
restatement oracle/cgen.py where none was prebuilt, pinned to it by
tests/test_refc.py) and
execute exactly the plan's directive multiplicities
(``TransferDirective.multiplicity``, src/transfers.py:176-188)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import SMALL_APPS, golden, oracle_final

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oracle_cache():
    return {}


def _oracle_state(name, g, cache):
    if name not in cache:
        from paper_2011_03602_b200.ir import Program

        cache[name] = (Program(g["doc"]), oracle_final(g["doc"], g["spec"]))
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
            assert got.tobytes() == np.asarray(want[vid], dtype=got.dtype).tobytes(), (name, x, prog.vars[vid].name)


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
    # coherent: p is current in HBM, so it is compared there (no epilogue
    # download of data the program never read on the host)
    assert coh["validity"] == "valid" and coh["epilogue_bytes"] == 0, coh


def test_literal_equals_coherent_when_plan_is_complete(evaluators):
    """For Himeno with the final read, every plan is sufficient: literal and
    coherent execution agree and the coherent manager adds no unplanned
    traffic beyond write-only first touches."""
    g = golden("himeno_17x9x33")
    lit = evaluators("h_literal", g["spec"], mode="literal")
    for x in ("100100", "100000", "000100", "001001", "111111"):
        r = lit.measure_payloads(g["doc"], [g["patterns"][x]])[0]
        assert r["validity"] == "valid" and r["stale_reads"] == 0, (x, r)


@pytest.mark.parametrize("mode", ["coherent", "literal"])
def test_job_results_do_not_depend_on_the_previous_job(evaluators, mode):
    """The reset between jobs restores host copies lazily (b2o_runtime.cu
    reset_state / host_fresh): a job's verdict, comparison and final state
    must not depend on which pattern ran before it on the same replica, in
    either mode.  12 Himeno XS genomes, each on a fresh replica, then all of
    them forward and backward on one replica."""
    from paper_2011_03602_b200.ir import Program

    g = golden("himeno_xs_inline")
    pats = g["patterns"]
    order = sorted(pats)[::5][:12]
    prog = Program(g["doc"])
    outs = [prog.var_by_name[o].id for o in g["spec"]["outputs"]]
    fresh = {}
    for x in order:
        ev = evaluators(f"order_{mode}_{x}", g["spec"], mode=mode)
        r = ev.measure_payloads(g["doc"], [pats[x]])[0]
        fresh[x] = (r, [ev.app_for(g["doc"]).read(v, worker=r["worker"]).tobytes() for v in outs])
    ev = evaluators(f"order_{mode}_chain", g["spec"], mode=mode)
    app = ev.app_for(g["doc"])
    for x in order + order[::-1]:
        r = ev.measure_payloads(g["doc"], [pats[x]])[0]
        f, fstate = fresh[x]
        assert (r["validity"], r["mismatches"], r["max_rel_err"], r["stale_reads"]) == \
            (f["validity"], f["mismatches"], f["max_rel_err"], f["stale_reads"]), (mode, x, r, f)
        assert [app.read(v, worker=r["worker"]).tobytes() for v in outs] == fstate, (mode, x)


def test_literal_noread_repeats_identically(evaluators):
    """The literal no-read genome reads a host copy of p that the coherent
    path would have refreshed: run after run on one replica it must see the
    same (pristine) bytes, whatever the previous run left there."""
    g = golden("himeno_xs_noread")
    ev = evaluators("noread_literal_repeat", g["spec"], mode="literal")
    rs = [ev.measure_payloads(g["doc"], [g["patterns"]["100100"]])[0] for _ in range(3)]
    assert len({(r["validity"], r["mismatches"], r["max_rel_err"], r["stale_reads"]) for r in rs}) == 1, rs


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


RESET_SRC = """int i;
int j;
float a[4096];
float b[4096];
float c[4096];

func main() {
  for (i = 0; i < 2048; i++) {
    b[i] = a[i] * 2.0;
  }
  for (j = 0; j < 4096; j++) {
    c[j] = b[j] + 1.0;
  }
  for (i = 2048; i < 4096; i++) {
    b[i] = a[i] * 3.0;
  }
}
"""


def test_reset_restores_device_only_intermediates():
    """an array a kernel writes but the host never reads
    (b: not an output, never downloaded) must be back to its pristine value
    on the device at the start of the next job.  Nest 1 writes b's first
    half, nest 2 reads all of b, nest 3 writes the second half: the second
    and later runs of the same pattern on the same worker used to read the
    previous run's second half."""
    from gpuoffload.evaluators import EvaluationRequest
    from gpuoffload.irdoc import model_to_document
    from gpuoffload.minilang import parse_mini_source
    from gpuoffload.patterns import build_genome_space, pattern_from_genome
    from gpuoffload.screen import screen_model
    from gpuoffload.transfers import plan_transfers

    from paper_2011_03602_b200.evaluator import B200Evaluator, payload_from_request
    from paper_2011_03602_b200.ir import Program

    model = parse_mini_source(RESET_SRC)
    doc = model_to_document(model)
    spec = {"precision": "fp32", "inputs": {"a": {"kind": "uniform", "seed": 5}}, "outputs": {"c": {"rel_tol": 0.0}}}
    space = build_genome_space(model, screen_model(model))
    ev = B200Evaluator(spec, devices=[0])
    want = oracle_final(doc, spec)
    cid = Program(doc).var_by_name["c"].id
    app = ev.app_for(doc)
    for bits in [(1, 1, 1), (1, 1, 1), (1, 0, 1), (1, 1, 1), (0, 1, 0), (1, 1, 1)]:
        pat = pattern_from_genome(model, space, bits)
        req = EvaluationRequest(model, pat, plan_transfers(model, pat), "", "c_openacc")
        r = ev.measure_payloads(doc, [payload_from_request(req)])[0]
        assert r["validity"] == "valid", (bits, r["diag"])
        got = app.read(cid, worker=r["worker"])
        assert got.tobytes() == want[cid].tobytes(), bits


@pytest.mark.parametrize("name,genome,out,normwise", [("himeno_17x9x33", "100100", "p", False),
                                                     ("himeno_17x9x33", "000000", "p", False),
                                                     ("blocks_small", None, "y", True)])
def test_device_compare_equals_host_compare(name, genome, out, normwise):
    """The output check on the device (csrc/b2o_compare.cu) gives the host
    check's verdict, mismatch count and worst relative error (reference rule
    src/evaluators.py:129-139), for a reference perturbed by small and large
    relative errors and a NaN."""
    import os

    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.evaluator import B200Evaluator
    from paper_2011_03602_b200.ir import Program

    g = golden(name)
    if genome is None:
        v = next(x for x in g["variants"] if x["subset"])
        doc, pat = v["doc"], v["pattern"]
    else:
        doc, pat = g["doc"], g["patterns"][genome]
    prog = Program(doc)
    vid = prog.var_by_name[out].id
    good = oracle_final(doc, g["spec"])[vid] if genome else None
    if good is None:
        ev0 = B200Evaluator(g["spec"], devices=[0])
        ev0.measure_payloads(doc, [pat])
        good = ev0.app_for(doc).reference(vid)
    bad = np.array(good, dtype=np.float32, copy=True)
    idx = np.flatnonzero(np.abs(bad) > 0.1)
    bad[idx[:5]] *= np.float32(1 + 2e-6)      # within rel_tol 1e-5
    bad[idx[5:9]] *= np.float32(1.5 if normwise else 1 + 1e-3)  # mismatches
    if not normwise:
        bad[idx[9]] = np.nan
    got = {}
    for host in (False, True):
        if host:
            os.environ["B2O_HOST_COMPARE"] = "1"
        try:
            ev = B200Evaluator(g["spec"], devices=[0], reference_outputs={out: bad})
            r = ev.measure_payloads(doc, [pat])[0]
        finally:
            os.environ.pop("B2O_HOST_COMPARE", None)
        got[host] = (r["validity"], r["mismatches"], r["max_rel_err"])
    assert got[False] == got[True], got
    assert got[False][0] == "numeric_mismatch"
