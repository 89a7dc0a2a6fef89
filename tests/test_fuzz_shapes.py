"""Differential fuzzing of the specialised kernels (tests/_fuzz_shapes.py:
register-tiled k-reductions, plane-marching quad stencils, exact in-order
fp32 reductions; fixtures with the reference's screen verdicts and hoisted
plans for every genome, tests/golden/fuzz_shapes.json).

CPU: the programs really exercise those shapes.  GPU: every genome of every
program is valid and leaves exactly the final state of the reference's own C emission
(oracle/_ref; tests/conftest.py oracle_final)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN, oracle_final
from paper_2011_03602_b200.ir import Program

SHAPES = json.loads((GOLDEN / "fuzz_shapes.json").read_text())
SEEDS = sorted(SHAPES, key=int)


def test_shapes_cover_specialised_kernels():
    from paper_2011_03602_b200.compiler import _Gen

    seen = {"ktile": 0, "march": 0, "exact": 0}
    for s in SEEDS:
        r = SHAPES[s]
        gen = _Gen(Program(r["doc"]), r["spec"])
        for n in gen.nests.values():
            if not n.kernel:
                continue
            seen["ktile"] += n.shape == "ktile"
            seen["march"] += n.shape == "quad" and bool(n.quad.get("march"))
            seen["exact"] += bool(n.exact)
    assert all(v >= 4 for v in seen.values()), seen
    assert sum(len(SHAPES[s]["patterns"]) for s in SEEDS) > 400


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_every_genome_bit_exact(seed):
    from paper_2011_03602_b200.evaluator import B200Evaluator

    r = SHAPES[seed]
    prog = Program(r["doc"])
    want = oracle_final(r["doc"], r["spec"])
    ev = B200Evaluator(r["spec"], devices=[0])
    app = ev.app_for(r["doc"])
    outs = [prog.var_by_name[o].id for o in r["spec"]["outputs"]]
    for g in sorted(r["patterns"]):
        res = ev.measure_payloads(r["doc"], [r["patterns"][g]])[0]
        assert res["validity"] == "valid", (seed, g, res["diag"])
        for vid in outs:
            got = app.read(vid, worker=res["worker"])
            assert got.tobytes() == np.asarray(want[vid], dtype=got.dtype).tobytes(), (seed, g, prog.vars[vid].name)
