"""Generate the golden fixtures from the reference itself.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every app it records what the reference computes on the hot path's input
side, so tests and bench can replay exact requests on a box without the
reference:

* the IR document (``irdoc.model_to_document``, ``src/irdoc.py:95-166``),
* the screen verdicts (``screen_model``, ``src/screen.py:82-84``) and the
  genome space (``build_genome_space``, ``src/patterns.py:38-48``),
* for each genome: placements and ``gpu_roots`` (``pattern_from_genome``,
  ``src/patterns.py:66-89``), the hoisted transfer plan (``plan_transfers``,
  ``src/transfers.py:194-199``) and the cost-model time
  (``cost_model_time``, ``src/evaluators.py:74-109``),
* for block apps: the replaced program variants (``apply_replacements``,
  ``src/blocks.py:463-563``) for every subset of the resolved candidates.

Numeric app outputs are NOT pinned here: the reference never executes
programs; see oracle/interp.py.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(ROOT))
if (REF / "src").exists():
    sys.path.insert(0, str(REF / "src"))

from gpuoffload.blocks import (  # noqa: E402
    apply_replacements,
    load_pattern_db,
    match_by_name,
    match_by_similarity,
    resolve_candidates,
)
from gpuoffload.evaluators import CostModelParams, EvaluationRequest, cost_model_time  # noqa: E402
from gpuoffload.irdoc import load_ir_document, model_to_document  # noqa: E402
from gpuoffload.minilang import ParseOptions, parse_mini_source  # noqa: E402
from gpuoffload.patterns import GenomeSpace, build_genome_space, pattern_from_genome  # noqa: E402
from gpuoffload.screen import screen_model  # noqa: E402
from gpuoffload.transfers import HOST_TO_DEVICE, TransferPlan, plan_transfers, unhoisted_plan  # noqa: E402

from paper_2011_03602_b200.apps import blockapp, histapp, himeno, intsum, matmul, nasmg  # noqa: E402
from paper_2011_03602_b200.reductions import screen_model_with_reductions  # noqa: E402


def fixture(name: str) -> str:
    return (REF / "fixtures" / name).read_text()


def uniform_spec(model, seed: int, outputs=None) -> dict:
    inputs = {}
    for v in model.variables:
        if v.is_array:
            inputs[v.name] = {"kind": "uniform", "seed": seed + v.id, "lo": 0.0, "hi": 1.0} \
                if v.base_type == "float" else {"kind": "randint", "seed": seed + v.id, "lo": 0, "hi": 4}
    outs = outputs or [v.name for v in model.variables]
    return {"precision": "fp32", "inputs": inputs, "outputs": {o: {"rel_tol": 1e-5} for o in outs}}


def plan_record(model, pattern, plan) -> dict:
    req = EvaluationRequest(model, pattern, plan, "", "c_openacc")
    cm = cost_model_time(req, CostModelParams())
    return {
        "genome": pattern.genome_text,
        "placements": {str(k): v for k, v in sorted(pattern.placements.items())},
        "gpu_roots": list(pattern.gpu_roots),
        "directives": [
            {
                "var": d.var_id,
                "dir": "h2d" if d.direction == HOST_TO_DEVICE else "d2h",
                "region": d.placement.region,
                "stmt_index": d.placement.stmt_index,
                "side": d.placement.side,
                "anchor_loop": d.placement.anchor_loop,
                "multiplicity": d.multiplicity,
                "batch": d.batch_id,
                "gpu_roots": list(d.gpu_roots),
            }
            for d in plan.directives
        ],
        "cost_model_time": cm.time_seconds,
        "cost_model_validity": cm.validity,
    }


def app_record(name: str, model, spec: dict, language: str | None = None, all_genomes_cap: int = 64,
               extra_genomes=(), unhoisted=(), screen=screen_model) -> dict:
    doc = model_to_document(model)
    if language:
        doc["language"] = language
        model = load_ir_document(json.dumps(doc))  # the reference validates the tagged document
        doc = model_to_document(model)
    verdicts = screen(model)
    space = build_genome_space(model, verdicts)
    genomes = list(space.all_genomes()) if 2 ** space.length <= all_genomes_cap else []
    for g in extra_genomes:
        bits = tuple(int(c) for c in g)
        if bits not in genomes:
            genomes.append(bits)
    patterns = {}
    for bits in genomes:
        pat = pattern_from_genome(model, space, bits)
        patterns[pat.genome_text] = plan_record(model, pat, plan_transfers(model, pat))
    unhoisted_rec = {}
    for g in unhoisted:
        pat = pattern_from_genome(model, space, tuple(int(c) for c in g))
        unhoisted_rec[g] = plan_record(model, pat, unhoisted_plan(model, pat))
    return {
        "name": name,
        "doc": doc,
        "spec": spec,
        "verdicts": [{"loop": v.loop_id, "reason": v.reason} for v in verdicts],
        "genome_loops": list(space.loop_ids),
        "patterns": patterns,
        "unhoisted": unhoisted_rec,
    }


def block_record(name: str, model, spec: dict) -> dict:
    db = load_pattern_db(REF / "fixtures" / "sample_db.json")
    cands, notes = resolve_candidates(model, match_by_name(model, db) + match_by_similarity(model, db))
    variants = []
    for mask in range(2 ** len(cands)):
        subset = [i for i in range(len(cands)) if mask >> i & 1]
        variant = apply_replacements(model, db, [cands[i] for i in subset]) if subset else model
        pat = pattern_from_genome(variant, GenomeSpace(0, ()), ())
        variants.append({
            "subset": subset,
            "doc": model_to_document(variant),
            "pattern": plan_record(variant, pat, TransferPlan(())),
        })
    return {
        "name": name,
        "spec": spec,
        "candidates": [{"block": f"{c.block.kind}:{c.block.id}", "record": c.record_id, "match": c.match_kind,
                        "score": c.similarity_score, "compatible": c.interface_compatible} for c in cands],
        "variants": variants,
    }


def shapes() -> None:
    """tests/_fuzz_shapes.py programs (k-tile, plane-march, exact-reduction
    kernels): all genomes, reference plans; the reduction family under the
    opt-in screen."""
    sys.path.insert(0, str(HERE.parent))
    import _fuzz_shapes

    rec = {}
    for seed in _fuzz_shapes.SEEDS:
        m = parse_mini_source(_fuzz_shapes.program(seed))
        sp = _fuzz_shapes.spec(seed)
        scr = screen_model_with_reductions if sp.get("reductions") else screen_model
        rec[str(seed)] = app_record(f"shapes_{seed}", m, sp, all_genomes_cap=512, screen=scr)
    (HERE / "fuzz_shapes.json").write_text(json.dumps(rec, sort_keys=True) + "\n")
    print("wrote fuzz_shapes.json:", {k: len(v["patterns"]) for k, v in rec.items()})


def main() -> None:
    if "--shapes" in sys.argv:
        shapes()
        return
    out: dict[str, dict] = {}
    for fx in ("four_loops", "nest2d", "stencil", "triple_nest", "matmul", "three_loops_fft"):
        m = parse_mini_source(fixture(f"{fx}.mini"))
        out[fx] = app_record(fx, m, uniform_spec(m, 7), unhoisted=("101",) if fx == "four_loops" else ())
    for form in ("inline", "temps"):
        m = parse_mini_source(himeno.source("XS", nn=3, form=form))
        out[f"himeno_xs_{form}"] = app_record(f"himeno_xs_{form}", m, himeno.spec("XS", form=form))
    m = parse_mini_source(himeno.source("XS", nn=2, read_p=False))
    out["himeno_xs_noread"] = app_record("himeno_xs_noread", m, himeno.spec("XS"), extra_genomes=("100100",),
                                         all_genomes_cap=1)
    m = parse_mini_source(himeno.source((17, 9, 33), nn=2))
    out["himeno_17x9x33"] = app_record("himeno_17x9x33", m, himeno.spec((17, 9, 33)))
    m = parse_mini_source(matmul.source(48))
    out["matmul_48"] = app_record("matmul_48", m, matmul.spec(48), language="python_like")
    m = parse_mini_source(nasmg.source(18, nit=2))
    out["nasmg_18"] = app_record("nasmg_18", m, nasmg.spec(18), language="java_like")
    for name, data in out.items():
        (HERE / f"{name}.json").write_text(json.dumps(data, sort_keys=True) + "\n")

    # configuration-sized apps (BASELINE.json configs): documents + plans only
    big = {
        "himeno_M": (parse_mini_source(himeno.source("M", nn=20)), himeno.spec("M"), None),
        "himeno_L": (parse_mini_source(himeno.source("L", nn=4)), himeno.spec("L"), None),
        "matmul_1024": (parse_mini_source(matmul.source(1024)), matmul.spec(1024), "python_like"),
        "nasmg_258": (parse_mini_source(nasmg.source(258, nit=4)), nasmg.spec(258), "java_like"),
    }
    for name, (m, spec, lang) in big.items():
        rec = app_record(name, m, spec, language=lang)
        (HERE / f"{name}.json").write_text(json.dumps(rec, sort_keys=True) + "\n")

    for name, (ng, nf) in {"blocks_small": (32, 16), "blocks_4096": (4096, 4096)}.items():
        m = parse_mini_source(blockapp.source(ng, nf))
        (HERE / f"{name}.json").write_text(json.dumps(block_record(name, m, blockapp.spec(ng, nf)),
                                                      sort_keys=True) + "\n")
    # similarity-matched GEMM nest (loop path of the block matcher) + the F2 fixture
    m = parse_mini_source(matmul.source(64))
    spec = matmul.spec(64)
    spec["outputs"] = {"mc": {"rel_tol": 1e-5}, "chk": {"rel_tol": 1e-4}}  # element-wise (reference rule)
    (HERE / "blocks_nest64.json").write_text(json.dumps(block_record("blocks_nest64", m, spec), sort_keys=True) + "\n")
    m = parse_mini_source(fixture("three_loops_fft.mini"))
    spec = uniform_spec(m, 11)  # x has 64 floats: no n with 2*n*n == 64, so the FFT variant cannot bind
    (HERE / "blocks_f2.json").write_text(json.dumps(block_record("blocks_f2", m, spec), sort_keys=True) + "\n")
    # cuda_histogram (third DB record): name path (opaque call) + similarity path (loop)
    # the reference's own pattern DB fixture as data, so the GPU box (no
    # /root/reference) can drive search_block_combination with it
    (HERE / "fixtures" / "sample_db.json").write_text((REF / "fixtures" / "sample_db.json").read_text())
    for name, (n, bins) in {"blocks_hist": (4096, 64), "blocks_hist_16m": (1 << 24, 256)}.items():
        m = parse_mini_source(histapp.source(n, bins))
        rec = block_record(name, m, histapp.spec(n, bins))
        rec["ga"] = app_record(name, m, histapp.spec(n, bins))
        (HERE / f"{name}.json").write_text(json.dumps(rec, sort_keys=True) + "\n")
    # opt-in reduction screen (reductions.py): the reference
    # planner and genome encoder run on the extended verdicts
    red = {
        "himeno_xs_red": (parse_mini_source(himeno.source("XS", nn=3)), himeno.spec("XS", reductions=True),
                          ("100100100", "000100000", "111111111", "001001001", "010010010", "000000000",
                           "100000100", "000100100")),
        "himeno_xs_temps_red": (parse_mini_source(himeno.source("XS", nn=3, form="temps")),
                                himeno.spec("XS", form="temps", reductions=True), ()),
        "himeno_M_red": (parse_mini_source(himeno.source("M", nn=20)), himeno.spec("M", reductions=True),
                         ("100100100", "100000100", "000000000")),
        "intsum": (parse_mini_source(intsum.source(1 << 16)), intsum.spec(1 << 16), ()),
    }
    for name, (m, spec, extra) in red.items():
        rec = app_record(name, m, spec, extra_genomes=extra, screen=screen_model_with_reductions,
                         all_genomes_cap=64 if not extra else 1)
        (HERE / f"{name}.json").write_text(json.dumps(rec, sort_keys=True) + "\n")
    # differential fuzz programs (tests/_fuzz.py): all genomes, reference plans
    sys.path.insert(0, str(HERE.parent))
    import _fuzz

    fuzz = {}
    for seed in _fuzz.SEEDS:
        m = parse_mini_source(_fuzz.program(seed))
        fuzz[str(seed)] = app_record(f"fuzz_{seed}", m, _fuzz.spec(seed), all_genomes_cap=256)
    (HERE / "fuzz.json").write_text(json.dumps(fuzz, sort_keys=True) + "\n")
    shapes()
    print("wrote", sorted(p.name for p in HERE.glob("*.json")))


if __name__ == "__main__":
    main()
