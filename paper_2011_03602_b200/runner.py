"""External-runner shim: lets the UNMODIFIED reference CLI drive B200.

The reference's ``ExternalCommandEvaluator`` (src/evaluators.py:268-293) writes
``candidate.<ext>`` and ``pattern.json`` into a fresh work directory, runs
``build_cmd`` then ``run_cmd`` there, and expects exactly one
``TIME_SECONDS=<float>`` line on stdout plus ``output.txt`` (one decimal per
line) when a reference output is configured (src/evaluators.py:167-242).
Use this module as the run command:

    gpuoffload --input app.mini --evaluator external --config cfg.txt
    # cfg.txt:  build_cmd = true
    #           run_cmd = python -m paper_2011_03602_b200.runner --spec /abs/app_spec.json

``pattern.json`` carries the genome and placements but no transfer anchors
(src/evaluators.py:245-261), so the runner rebuilds the program model (from
``--model`` IR document, or by stripping the c_openacc / python markers of the
candidate and re-parsing it, src/codegen.py:250-254) and re-derives the exact
plan with the reference's own planner (``plan_transfers``).  Non-valid B200
results exit non-zero (the harness maps that to runtime_error).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path


def _model(args):
    from gpuoffload.irdoc import load_ir_document
    from gpuoffload.minilang import parse_mini_source

    if args.model:
        return load_ir_document(Path(args.model).read_bytes())
    for ext, backend in (("c", "c_openacc"), ("py", "python_cuda_marker")):
        cand = Path(f"candidate.{ext}")
        if cand.exists():
            from gpuoffload.codegen import strip_annotations

            return parse_mini_source(strip_annotations(cand.read_text(), backend))
    raise SystemExit("runner: no --model and no strippable candidate (java_lambda_marker needs --model)")


def _ensure_reference_importable() -> None:
    try:
        import gpuoffload  # noqa: F401
    except ImportError:  # the repo's own install of the reference (baseline/_ref)
        ref = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
        if ref.exists():
            sys.path.append(str(ref))


def _reference_file(doc: dict, spec: dict) -> Path:
    """Where the all-CPU reference outputs of this program (and these inputs)
    are kept between runner invocations: the harness starts one runner
    process per pattern, and without the cache every one of them would re-run
    the whole program on the CPU at load (``b2o_app_finalize``) -- the
    reference outputs depend on the program and its inputs, never on the
    genome."""
    import hashlib

    from .compiler import CACHE
    from .ir import document_digest

    blob = json.dumps([document_digest(doc), spec.get("inputs"), spec.get("precision"), spec.get("externals"),
                       sorted(spec.get("outputs", {}))], sort_keys=True, default=str)
    return Path(CACHE) / "refs" / (hashlib.sha256(blob.encode()).hexdigest()[:24] + ".npz")


def _load_reference(path: Path) -> dict | None:
    import numpy as np

    try:
        with np.load(path) as z:
            return {k: z[k] for k in z.files}
    except (OSError, ValueError):
        return None


def _store_reference(path: Path, ev, doc: dict, spec: dict) -> None:
    """Written atomically (temp file + rename): concurrent runners may race."""
    import os
    import tempfile

    import numpy as np

    from . import appspec
    from .ir import Program

    try:
        app = ev.app_for(doc)
        prog = Program(doc)
        outs = {prog.vars[vid].name: app.reference(vid) for vid, _, _ in appspec.outputs_of(prog, spec)}
        path.parent.mkdir(parents=True, exist_ok=True)
        fd, tmp = tempfile.mkstemp(dir=path.parent, suffix=".npz")
        with os.fdopen(fd, "wb") as f:
            np.savez(f, **outs)
        os.replace(tmp, path)
    except Exception as exc:  # the cache is an optimisation: never fail the measurement over it
        print(f"runner: reference cache not written: {exc}", file=sys.stderr)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--spec", required=True, help="app spec JSON (inputs, outputs, externals, blocks)")
    ap.add_argument("--model", help="IR document of the program (else parsed from candidate.c/.py)")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--mode", default="coherent", choices=("coherent", "literal"))
    ap.add_argument("--outputs", help="comma-separated output variables written to output.txt (default: spec)")
    args = ap.parse_args(argv)
    _ensure_reference_importable()

    from gpuoffload.evaluators import EvaluationRequest
    from gpuoffload.patterns import build_genome_space, pattern_from_genome
    from gpuoffload.screen import screen_model
    from gpuoffload.transfers import plan_transfers

    from .evaluator import B200Evaluator, payload_from_request
    from .ir import document_of

    spec = json.loads(Path(args.spec).read_text())
    manifest = json.loads(Path("pattern.json").read_text())
    model = _model(args)
    space = build_genome_space(model, screen_model(model))
    bits = tuple(int(c) for c in manifest["genome"]) if manifest["genome"] else (0,) * space.length
    pattern = pattern_from_genome(model, space, bits)
    if {str(k): v for k, v in pattern.placements.items()} != manifest["placements"]:
        print("runner: placements in pattern.json do not match the rebuilt model", file=sys.stderr)
        return 3
    plan = plan_transfers(model, pattern)
    doc = document_of(model)
    ref_file = _reference_file(doc, spec)
    cached = _load_reference(ref_file)
    ev = B200Evaluator(spec, devices=[args.device], mode=args.mode, reference_outputs=cached)
    req = EvaluationRequest(model, pattern, plan, "", "c_openacc")
    res = ev.measure_payloads(doc, [payload_from_request(req)])[0]
    if cached is None:
        _store_reference(ref_file, ev, doc, spec)
    if res["validity"] != "valid":
        print(f"runner: {res['validity']}: {res.get('diag', '')}", file=sys.stderr)
        return 2
    app = ev.app_for(doc)
    names = args.outputs.split(",") if args.outputs else list(spec.get("outputs", {}))
    prog_vars = {v["name"]: v["id"] for v in doc["variables"]}
    lines = []
    for name in names:
        for x in app.read(prog_vars[name], worker=res["worker"]).tolist():
            lines.append(repr(float(x)))
    Path("output.txt").write_text("\n".join(lines) + "\n")
    print(f"TIME_SECONDS={res['time_s']!r}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
