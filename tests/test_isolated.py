"""IsolatedEvaluator's recovery logic on CPU, with a child double that
behaves like the runtime after a sticky CUDA error (tests/_iso_double.py);
the real fault is injected on the GPU in tests/test_isolated_gpu.py."""

from paper_2011_03602_b200.isolated import IsolatedEvaluator

DOC = {"variables": [], "loops": []}


def pat(g):
    return {"genome": g, "gpu_roots": [], "directives": []}


def make(**kw):
    return IsolatedEvaluator({}, factory="_iso_double:FakeB200", start_timeout=60, **kw)


def test_sticky_fault_replaces_child_and_remeasures_refused_jobs():
    ev = make()
    try:
        r = ev.measure_payloads(DOC, [pat("a")])[0]
        assert r["validity"] == "valid"
        pid0 = r["pid"]
        ev.inject_fault(0)
        res = ev.measure_payloads(DOC, [pat("b"), pat("c"), pat("d")])
        # b faulted (kept), c and d were refused by the dead device: re-run on a fresh child
        assert [x["validity"] for x in res] == ["runtime_error", "valid", "valid"]
        assert ev.restarts == 1 and res[1]["pid"] != pid0
        assert ev.measure_payloads(DOC, [pat("e")])[0]["validity"] == "valid"
    finally:
        ev.close()


def test_crash_and_hang_are_isolated():
    ev = make(timeout_seconds=1.0)
    ev.start_timeout = 8.0
    try:
        res = ev.measure_payloads(DOC, [pat("a"), pat("crash"), pat("b")])
        assert [x["validity"] for x in res] == ["valid", "runtime_error", "valid"]
        r = ev.measure_payloads(DOC, [pat("hang")])[0]
        assert r["validity"] == "timeout"
        assert ev.measure_payloads(DOC, [pat("c")])[0]["validity"] == "valid"
        assert ev.restarts >= 3
    finally:
        ev.close()
