"""The compiler's optional kernel shapes (measured and kept selectable,
DESIGN.md §4) stay correct: every genome of a few apps and fuzz programs,
compiled with each option, leaves the C oracle's final state bit for bit
(spec["stencil"] 2.5-D smem template, spec["brick"]-style k-blocking,
points per thread, two quads per thread, warp-shuffle neighbour exchange,
march prefetch, cp.async-staged march planes, k-tile stage fast path off, march / k-tile / progressive downloads switched off)."""

import copy
import json

import pytest

from conftest import GOLDEN, oracle_final
from paper_2011_03602_b200.ir import Program

OPTIONS = [
    {"stencil": True},
    {"flat_kblock": 4},
    {"flat_ppt": 2},
    {"quad_groups": 2},
    {"quad_shfl": True},
    {"quad_shfl": True, "quad_shfl_max": 4},
    {"march_prefetch": True},
    {"quad_march": 0},
    {"quad_march": 4, "march_block": 64},
    {"march_async": 2},
    {"march_async": 3, "march_block": 64},
    {"march_async": 2, "quad_march": 16},
    {"ktile_fast": False},
    {"ktile_ri": 8},
    {"ktile_prefetch": False, "ktile_swz": False},
    {"ktile": False},
    {"ktile_tile": 32},
    {"ktile_r": 8},
    {"progressive_d2h": False},
    {"flat_min_blocks": 2},
    {"march_tma": True, "quad_march": 32, "march_tma_stages": 4},
    {"march_tma": True},
    {"march_shfl": True},
    {"march_shfl": True, "quad_march": 5, "march_block": 64},
    {"march_chains": False},
    {"march_chains": False, "march_fill": False, "march_l2pf": 0},
    {"quad_nextpf": False},
]

FUZZ = json.loads((GOLDEN / "fuzz.json").read_text())


def _programs():
    out = []
    for a in ("himeno_17x9x33", "nasmg_18", "matmul_48", "stencil", "triple_nest"):
        g = json.loads((GOLDEN / f"{a}.json").read_text())
        out.append((a, g["doc"], g["spec"], g["patterns"]))
    for s in sorted(FUZZ, key=int)[:6]:
        out.append((f"fuzz_{s}", FUZZ[s]["doc"], FUZZ[s]["spec"], FUZZ[s]["patterns"]))
    return out


PROGRAMS = _programs()


def test_options_change_the_generated_kernels():
    from paper_2011_03602_b200.compiler import generate_sources

    name, doc, spec, _ = PROGRAMS[0]
    base = generate_sources(doc, spec)[1]
    changed = sum(generate_sources(doc, dict(spec, **o))[1] != base for o in OPTIONS)
    assert changed >= 6, changed


@pytest.mark.gpu
@pytest.mark.parametrize("opt", OPTIONS, ids=[json.dumps(o, sort_keys=True) for o in OPTIONS])
def test_option_every_genome_bit_exact(opt):
    from paper_2011_03602_b200.evaluator import B200Evaluator

    for name, doc, spec, patterns in PROGRAMS:
        sp = dict(copy.deepcopy(spec), **opt)
        prog = Program(doc)
        want = oracle_final(doc, sp)
        ev = B200Evaluator(sp, devices=[0])
        app = ev.app_for(doc)
        outs = [prog.var_by_name[o].id for o in sp["outputs"]]
        for g in sorted(patterns)[:32]:
            r = ev.measure_payloads(doc, [patterns[g]])[0]
            assert r["validity"] == "valid", (opt, name, g, r["diag"])
            for vid in outs:
                got = app.read(vid, worker=r["worker"])
                assert got.tobytes() == want[vid].tobytes(), (opt, name, g, prog.vars[vid].name)
