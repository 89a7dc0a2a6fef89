"""Differential fuzzing of the GPU path (tests/_fuzz.py programs; fixtures
with the reference's screen verdicts and hoisted plans for every genome,
tests/golden/fuzz.json).

CPU: the two oracles agree on every program (C restatement == pure-Python
interpreter, bit for bit), and the programs exercise every kernel shape the
compiler emits (quad, flat, sequential, zero-trip bounds).
GPU: every genome of every program is valid and leaves exactly the oracle's
final state -- 3976 patterns, hazard-free programs, so bit-exact."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, oracle_final
from oracle.cgen import CProgram
from oracle.interp import run_program
from paper_2011_03602_b200 import appspec
from paper_2011_03602_b200.ir import Program

FUZZ = json.loads((GOLDEN / "fuzz.json").read_text())
SEEDS = sorted(FUZZ, key=int)


@pytest.fixture(scope="module")
def oracle_states():
    out = {}
    for s in SEEDS:
        r = FUZZ[s]
        st = appspec.initial_state(Program(r["doc"]), r["spec"])
        out[s] = CProgram(r["doc"]).run(st)
    return out


@pytest.mark.parametrize("seed", SEEDS)
def test_oracles_agree(seed, oracle_states):
    r = FUZZ[seed]
    st = appspec.initial_state(Program(r["doc"]), r["spec"])
    a = run_program(r["doc"], st)
    for k, v in oracle_states[seed].items():
        assert np.array_equal(a[k], v), (seed, k)


def test_fuzz_covers_kernel_shapes():
    from paper_2011_03602_b200.compiler import _Gen

    shapes = set()
    zero_trip = False
    for s in SEEDS:
        r = FUZZ[s]
        gen = _Gen(Program(r["doc"]), r["spec"])
        for n in gen.nests.values():
            if n.kernel:
                shapes.add((n.shape, len(n.chain) > 0))
        zero_trip |= "< 0;" in json.dumps(r["doc"]) or any(
            lo.get("upper", {}).get("num") == 0 for lo in r["doc"]["loops"])
    assert {("quad", True), ("flat", False)} <= shapes, shapes
    assert sum(len(FUZZ[s]["patterns"]) for s in SEEDS) > 800


def _trips(loop) -> int | None:
    lo, up = loop["lower"], loop["upper"]
    if "num" in lo and "num" in up:
        return max(0, int(up["num"]) - int(lo["num"]))
    return None


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_every_genome_bit_exact(seed):
    from paper_2011_03602_b200.evaluator import B200Evaluator

    r = FUZZ[seed]
    prog = Program(r["doc"])
    want = oracle_final(r["doc"], r["spec"])  # the reference's own C emission (oracle/_ref)
    ev = B200Evaluator(r["spec"], devices=[0])
    app = ev.app_for(r["doc"])
    outs = [prog.var_by_name[o].id for o in r["spec"]["outputs"]]
    genomes = sorted(r["patterns"])
    results = ev.measure_payloads(r["doc"], [r["patterns"][g] for g in genomes])
    # the reference clamps trip counts to >= 1 (src/minilang.py:505-517), so a
    # directive placed inside a zero-trip loop is counted in its multiplicity
    # but never executes: equality holds exactly when no loop is zero-trip
    zero_trip = any(lo["iter_count"] == 1 and _trips(lo) == 0 for lo in r["doc"]["loops"])
    for g, res in zip(genomes, results):
        assert res["validity"] == "valid", (seed, g, res["diag"])
        planned = sum(d["multiplicity"] for d in r["patterns"][g]["directives"])
        if zero_trip:
            assert res["directive_execs"] <= planned, (seed, g)
        else:
            assert res["directive_execs"] == planned, (seed, g)
    # final state of every genome, one at a time
    for g in genomes:
        res = ev.measure_payloads(r["doc"], [r["patterns"][g]])[0]
        for vid in outs:
            got = app.read(vid, worker=res["worker"])
            assert np.array_equal(got, want[vid]), (seed, g, prog.vars[vid].name)
