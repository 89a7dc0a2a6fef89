"""IsolatedEvaluator (paper_2011_03602_b200/isolated.py): a sticky CUDA error
in one pattern kills the CUDA context of its process for good (in-process
cudaDeviceReset cannot bring it back: profiles/r02/reset_probe.log), so the
runtime runs in a child process that is replaced after the fault.  The
faulting pattern is runtime_error; the next patterns are measured valid on
the fresh child, against the same all-CPU reference outputs."""

import pytest

from conftest import golden, has_reference

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def iso():
    from paper_2011_03602_b200.isolated import IsolatedEvaluator

    g = golden("himeno_xs_inline")
    ev = IsolatedEvaluator(g["spec"], devices=[0], timeout_seconds=60)
    yield g, ev
    ev.close()


def test_fault_then_fresh_child(iso):
    g, ev = iso
    pat = g["patterns"]["100100"]
    r0 = ev.measure_payloads(g["doc"], [pat])[0]
    assert r0["validity"] == "valid", r0
    ev.inject_fault(0)
    r1 = ev.measure_payloads(g["doc"], [pat])[0]
    assert r1["validity"] == "runtime_error", r1
    before = ev.restarts
    r2 = ev.measure_payloads(g["doc"], [pat])[0]   # the dead device refuses: child replaced, job re-run
    assert r2["validity"] == "valid", r2
    assert ev.restarts == before + 1
    assert r2["directive_execs"] == r0["directive_execs"] and r2["launches"] == r0["launches"]


def test_batch_after_fault_every_other_pattern_valid(iso):
    g, ev = iso
    genomes = ["100100", "100000", "000100", "001001", "010010"]
    ev.inject_fault(0)
    res = ev.measure_payloads(g["doc"], [g["patterns"][x] for x in genomes])
    bad = [x for x, r in zip(genomes, res) if r["validity"] != "valid"]
    assert len(bad) <= 1, res          # only the job that trapped
    res2 = ev.measure_payloads(g["doc"], [g["patterns"][x] for x in genomes])
    assert all(r["validity"] == "valid" for r in res2), res2


@pytest.mark.skipif(not has_reference(), reason="reference not importable")
def test_plugin_protocol_through_child(iso):
    """measure_batch with reference requests: results in request order,
    program-level dedupe in the parent."""
    import json

    from gpuoffload.irdoc import load_ir_document
    from gpuoffload.patterns import build_genome_space, pattern_from_genome
    from gpuoffload.screen import screen_model
    from gpuoffload.transfers import plan_transfers
    from gpuoffload.evaluators import EvaluationRequest

    g, ev = iso
    model = load_ir_document(json.dumps(g["doc"]))
    space = build_genome_space(model, screen_model(model))
    reqs = []
    for bits in list(space.all_genomes())[:8]:
        pat = pattern_from_genome(model, space, bits)
        reqs.append(EvaluationRequest(model, pat, plan_transfers(model, pat), "", "c_openacc"))
    out = ev.measure_batch(reqs)
    assert len(out) == 8 and all(r.validity == "valid" and r.time_seconds > 0 for r in out)
    assert ev.parallel_width == 1


@pytest.mark.skipif(not has_reference(), reason="reference not importable")
def test_two_workers_ga_with_confirmation():
    """The throughput mode: the reference GA over two workers sharing the
    B200 in an isolated child, the fastest programs re-measured alone; the
    result is a valid genome whose confirmed time is a solo measurement."""
    import json

    from gpuoffload.ga import GAParams
    from gpuoffload.irdoc import load_ir_document
    from gpuoffload.screen import screen_model

    from paper_2011_03602_b200.isolated import IsolatedEvaluator
    from paper_2011_03602_b200.search import run_search_batched

    g = golden("himeno_17x9x33")
    model = load_ir_document(json.dumps(g["doc"]))
    ev = IsolatedEvaluator(g["spec"], devices=[0, 0], timeout_seconds=60)
    try:
        assert ev.parallel_width == 2
        stats = {}
        res = run_search_batched(model, screen_model(model), ev, GAParams(population_size=16, generations=4, seed=3),
                                 stats=stats, confirm_top=2, confirm_repeats=2)
    finally:
        ev.close()
    assert res.best_time is not None and res.best_time > 0
    rows = stats["confirmed"]
    assert 1 <= len(rows) <= 2 and all(s is not None for _, _, s in rows)
    assert res.best_time == min(s for _, _, s in rows)
