"""Parity pinned to the reference itself (oracle/_ref, ``oracle/refc.py``).

The reference renders every program as C (``gpuoffload.codegen.pretty_print``,
src/gpuoffload/codegen.py:230-232).  That text, compiled with gcc behind a
two-line prelude and run on the app spec's inputs, must leave exactly the
final state of the C restatement ``oracle/cgen.py`` -- bit for bit, every
variable -- on every golden app, every block-search program variant, every
committed fuzz program (tests/_fuzz.py, tests/_fuzz_shapes.py), the fp64
builds, and Himeno M (BASELINE config 2).  The GPU suites compare the B200
path with ``oracle/cgen.py`` (tests/test_parity_gpu.py, test_fuzz*.py,
test_fullsize_gpu.py), so this file is what ties the GPU to the reference.

Also: the annotated ``c_openacc`` emission of a pattern (the text the
reference hands to a compiler for that genome, codegen.py:235-247) computes
the same program, and its OpenMP mapping (bench.py's reference arm) is
bit-identical to the sequential text.
"""

from __future__ import annotations

import json
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

from conftest import GOLDEN, SMALL_APPS, golden, has_reference

pytestmark = pytest.mark.skipif(not has_reference(), reason="reference package not importable (emission needs it)")

FUZZ = json.loads((GOLDEN / "fuzz.json").read_text())
SHAPES = json.loads((GOLDEN / "fuzz_shapes.json").read_text())
APPS = SMALL_APPS + ["himeno_xs_noread", "himeno_xs_red", "himeno_xs_temps_red", "intsum", "himeno_M_red"]
BLOCKS = ["blocks_small", "blocks_hist", "blocks_nest64", "blocks_f2", "blocks_hist_16m"]
FP64_APPS = ["four_loops", "nest2d", "stencil", "triple_nest", "himeno_xs_inline", "himeno_17x9x33", "matmul_48",
             "nasmg_18"]


def _cases():
    """(label, doc, spec) of every program checked here."""
    out = []
    for a in APPS:
        g = golden(a)
        out.append((a, g["doc"], g["spec"]))
    for b in BLOCKS:
        g = golden(b)
        for i, v in enumerate(g["variants"]):
            out.append((f"{b}/{i}", v["doc"], g["spec"]))
    for k in sorted(FUZZ, key=int):
        out.append((f"fuzz/{k}", FUZZ[k]["doc"], FUZZ[k]["spec"]))
    for k in sorted(SHAPES, key=int):
        out.append((f"shapes/{k}", SHAPES[k]["doc"], SHAPES[k]["spec"]))
    for k in sorted(FUZZ, key=int)[:16]:
        out.append((f"fuzz64/{k}", FUZZ[k]["doc"], dict(FUZZ[k]["spec"], precision="fp64")))
    for a in FP64_APPS:
        g = golden(a)
        out.append((f"{a}@fp64", g["doc"], dict(g["spec"], precision="fp64")))
    return out


CASES = _cases()


def _build(item) -> str:
    doc, prec = item
    from oracle import refc
    from oracle.cgen import CProgram

    CProgram(doc, prec)  # compiled into oracle/_build (cache)
    return str(refc.build(doc, prec))


@pytest.fixture(scope="module")
def built():
    items = [(doc, spec.get("precision", "fp32")) for _, doc, spec in CASES]
    with ProcessPoolExecutor(max(1, min(8, len(os.sched_getaffinity(0))))) as pool:
        return list(pool.map(_build, items, chunksize=4))


def _compare(doc, spec, so):
    from oracle.cgen import CProgram
    from oracle.externals import make_binder
    from oracle.refc import RefProgram
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.ir import Program

    prec = spec.get("precision", "fp32")
    st = appspec.initial_state(Program(doc), spec)
    binder = make_binder(doc, spec)
    outcome = []
    for run in (lambda: RefProgram(so).run(st, binder), lambda: CProgram(doc, prec).run(st, binder)):
        try:
            outcome.append(run())
        except RuntimeError as exc:  # an app spec that cannot bind an external
            outcome.append(exc)
    ref, ours = outcome
    if isinstance(ref, Exception) or isinstance(ours, Exception):
        # both oracles must refuse the same programs (blocks_f2's cufft_exec
        # variant: 64 floats are no n x n complex grid)
        return [] if isinstance(ref, Exception) and isinstance(ours, Exception) else [f"raised: {ref!r} / {ours!r}"]
    bad = [v["name"] for v in doc["variables"]
           if ref[v["id"]].tobytes() != np.asarray(ours[v["id"]], dtype=ref[v["id"]].dtype).tobytes()]
    return bad


def test_every_program_bit_identical_to_reference_emission(built):
    failures = {}
    for (label, doc, spec), so in zip(CASES, built):
        bad = _compare(doc, spec, so)
        if bad:
            failures[label] = bad
    assert not failures, failures
    assert len(CASES) >= 96 + 90 + 16 + 8 + len(APPS)


def test_himeno_M_bit_identical_to_reference_emission():
    """BASELINE config 2 at full size (129x129x257, 20 sweeps)."""
    from oracle import refc

    g = golden("himeno_M")
    so = refc.build(g["doc"], "fp32")
    assert _compare(g["doc"], g["spec"], so) == []


def test_reference_text_is_compiled_verbatim():
    """The .c file holds the reference's text unchanged after our header."""
    from gpuoffload import codegen, irdoc

    from oracle import refc

    g = golden("himeno_17x9x33")
    so = refc.build(g["doc"], "fp32")
    c = so.with_suffix(".c").read_text()
    text = codegen.pretty_print(irdoc.load_ir_document(json.dumps(g["doc"])))
    assert c.endswith(text)
    assert "func main() {" in text  # the reference's entry, mapped by the prelude


@pytest.mark.parametrize("name", ["four_loops", "himeno_17x9x33", "nasmg_18", "matmul_48", "three_loops_fft"])
def test_annotated_emission_same_program(name):
    """Every genome's annotated c_openacc text (acc pragmas ignored by gcc)
    computes the program's result (sampled genomes)."""
    from oracle import refc
    from oracle.externals import make_binder
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.ir import Program

    g = golden(name)
    st = appspec.initial_state(Program(g["doc"]), g["spec"])
    binder = make_binder(g["doc"], g["spec"])
    want = refc.RefProgram(refc.build(g["doc"])).run(st, binder)
    genomes = sorted(g["patterns"])
    for gen in genomes[:: max(1, len(genomes) // 6)] + genomes[-1:]:
        so = refc.build(g["doc"], "fp32", pattern=g["patterns"][gen], genome_loops=g["genome_loops"])
        c = so.with_suffix(".c").read_text()
        if any(x == "1" for x in gen):
            assert "#pragma acc" in c
        got = refc.RefProgram(so).run(st, binder)
        for k in want:
            assert got[k].tobytes() == want[k].tobytes(), (name, gen, k)


@pytest.mark.parametrize("name,genome", [("himeno_17x9x33", "100100"), ("nasmg_18", "100100"),
                                         ("matmul_48", "10"), ("four_loops", "111")])
def test_openmp_mapping_bit_identical(name, genome):
    from oracle import refc
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.ir import Program

    g = golden(name)
    st = appspec.initial_state(Program(g["doc"]), g["spec"])
    want = refc.RefProgram(refc.build(g["doc"])).run(st)
    so = refc.build(g["doc"], "fp32", pattern=g["patterns"][genome], genome_loops=g["genome_loops"], openmp=True)
    assert "#pragma omp parallel for" in so.with_suffix(".c").read_text()
    got = refc.RefProgram(so).run(st)
    for k in want:
        assert got[k].tobytes() == want[k].tobytes(), (name, k)


def test_runner_needs_only_the_sidecar(tmp_path):
    """A built .so runs from its JSON sidecar alone (the GPU box has no
    reference): the sidecar carries names, types, static initialisers and
    the external call sites in emission order."""
    from oracle import refc

    g = golden("three_loops_fft")
    so = refc.build(g["doc"])
    meta = json.loads(so.with_suffix(".json").read_text())
    assert {v["name"] for v in meta["variables"]} == {v["name"] for v in g["doc"]["variables"]}
    assert meta["static_init"], "N and s carry initialisers"
    assert refc.prebuilt(g["doc"]) == so
