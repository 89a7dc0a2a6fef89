"""The unmodified reference pipeline (run_pipeline, src/pipeline.py:190-327)
driven through its external-command evaluator with the B200 runner shim as
run_cmd: every genome is measured on the GPU, the report's winner is a
measured valid pattern, and output.txt parity holds against the all-CPU
reference output."""

import json
import sys

import pytest

from conftest import ROOT, golden, has_reference

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_reference(), reason="reference not importable")]


def test_cli_pipeline_through_runner(tmp_path):
    from gpuoffload.pipeline import PipelineConfig, run_pipeline

    from paper_2011_03602_b200.apps import himeno

    src = tmp_path / "himeno.mini"
    src.write_text(himeno.source("XS", nn=2))
    spec = himeno.spec("XS")
    spec["outputs"] = {"chk": {"rel_tol": 1e-5}}
    spec_path = tmp_path / "spec.json"
    spec_path.write_text(json.dumps(spec))
    run_cmd = f"PYTHONPATH={ROOT}:$PYTHONPATH {sys.executable} -m paper_2011_03602_b200.runner --spec {spec_path}"
    # reference output: the all-CPU program's chk, from the oracle
    from oracle.cgen import CProgram
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.ir import Program
    from gpuoffload.irdoc import model_to_document
    from gpuoffload.minilang import parse_mini_source

    doc = model_to_document(parse_mini_source(src.read_text()))
    prog = Program(doc)
    out = CProgram(doc).run(appspec.initial_state(prog, spec))
    ref = tmp_path / "ref.txt"
    ref.write_text(repr(float(out[prog.var_by_name["chk"].id][0])) + "\n")
    cfg = PipelineConfig(input_path=str(src), evaluator="external", exhaustive=True, out_dir=str(tmp_path / "out"),
                         build_cmd="true", run_cmd=run_cmd, reference_output=str(ref), timeout_seconds=120.0,
                         rel_tol=1e-5)
    report = run_pipeline(cfg)
    ga = [m for m in report.measurements if m["stage"] == "ga"]
    assert len(ga) == 64
    assert all(m["validity"] == "valid" for m in ga), [m for m in ga if m["validity"] != "valid"][:3]
    # the winner is the fastest valid measurement; on this tiny grid the
    # all-CPU program (block-stage baseline, genome None) may well win
    valid = [m["time"] for m in report.measurements if m["validity"] == "valid"]
    assert report.chosen["time"] == min(valid)
    # the all-CPU reference outputs were computed once and cached for the
    # later runner processes (one per pattern), keyed by program and inputs
    from paper_2011_03602_b200.runner import _load_reference, _reference_file

    cached = _load_reference(_reference_file(doc, spec))
    assert cached is not None and set(cached) == {"chk"}
    assert cached["chk"].tobytes() == out[prog.var_by_name["chk"].id].tobytes()
