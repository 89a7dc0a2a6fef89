"""fp64 precision on the GPU (north_star: 1e-12 for fp64): the same programs
compiled with ``precision: fp64`` (model ``float`` -> C ``double``: flat
kernels instead of the 4-byte quad / k-tile shapes, 8-byte transfers and
progressive downloads) must leave the final state of the reference's own C emission
compiled fp64 (oracle/_ref) bit for bit under every genome -- the kernels evaluate the same C expression trees
with -fmad=false.  Programs: the fuzz set (quad/flat/sequential shapes,
zero-trip bounds, lastprivate scalars, host reductions) and the small apps."""

import copy
import json

import pytest

from conftest import GOLDEN, oracle_final
from paper_2011_03602_b200.ir import Program

FUZZ = json.loads((GOLDEN / "fuzz.json").read_text())
APPS = ["four_loops", "nest2d", "stencil", "triple_nest", "himeno_xs_inline", "himeno_17x9x33", "matmul_48",
        "nasmg_18"]


def _cases():
    out = [(f"fuzz_{s}", FUZZ[s]["doc"], FUZZ[s]["spec"], FUZZ[s]["patterns"]) for s in sorted(FUZZ, key=int)[:16]]
    for a in APPS:
        g = json.loads((GOLDEN / f"{a}.json").read_text())
        out.append((a, g["doc"], g["spec"], g["patterns"]))
    return out


CASES = _cases()


def test_fp64_compiles_to_8_byte_kernels():
    from paper_2011_03602_b200.compiler import generate_sources

    name, doc, spec, _ = next(c for c in CASES if c[0] == "himeno_17x9x33")
    host, dev, hdr = generate_sources(doc, dict(spec, precision="fp64"))
    assert "double" in dev and "float4" not in dev  # no 16-byte quads of doubles


@pytest.mark.gpu
@pytest.mark.parametrize("name,doc,spec,patterns", CASES, ids=[c[0] for c in CASES])
def test_every_genome_bit_exact_fp64(name, doc, spec, patterns):
    from paper_2011_03602_b200.evaluator import B200Evaluator

    sp = dict(copy.deepcopy(spec), precision="fp64")
    for o in sp.get("outputs", {}).values():
        o["rel_tol"] = 1e-12
    prog = Program(doc)
    want = oracle_final(doc, sp)  # the reference's emission built with -Dfloat=double
    ev = B200Evaluator(sp, devices=[0])
    app = ev.app_for(doc)
    outs = [prog.var_by_name[o].id for o in sp["outputs"]]
    for g in sorted(patterns)[:64]:
        r = ev.measure_payloads(doc, [patterns[g]])[0]
        assert r["validity"] == "valid", (name, g, r["diag"])
        for vid in outs:
            got = app.read(vid, worker=r["worker"])
            assert got.dtype == want[vid].dtype and got.tobytes() == want[vid].tobytes(), (name, g, prog.vars[vid].name)
