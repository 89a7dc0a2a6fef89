"""Small driver for compute-sanitizer racecheck/memcheck over the k-tile and
plane-march kernels: every genome of matmul 48 (64x64 tiles with ragged
edges and a partial k stage), one of the 64-aligned k-tile fuzz shapes, and
NAS-MG 18's march pattern, each checked bit-exact against the C oracle."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle.cgen import CProgram  # noqa: E402
from paper_2011_03602_b200 import appspec  # noqa: E402
from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402
from paper_2011_03602_b200.ir import Program  # noqa: E402

cases = []
for name, genomes in (("matmul_48", None), ("nasmg_18", ["100100"])):
    g = json.loads((ROOT / "tests" / "golden" / f"{name}.json").read_text())
    cases.append((name, g["doc"], g["spec"], genomes or sorted(g["patterns"]), g["patterns"]))
shapes = json.loads((ROOT / "tests" / "golden" / "fuzz_shapes.json").read_text())
for seed in sorted(shapes, key=int)[:3]:
    r = shapes[seed]
    cases.append((f"shape_{seed}", r["doc"], r["spec"], sorted(r["patterns"])[:4], r["patterns"]))
for name, doc, spec, genomes, patterns in cases:
    prog = Program(doc)
    want = CProgram(doc, spec.get("precision", "fp32")).run(appspec.initial_state(prog, spec))
    ev = B200Evaluator(spec, devices=[0])
    app = ev.app_for(doc)
    for x in genomes:
        r = ev.measure_payloads(doc, [patterns[x]])[0]
        assert r["validity"] == "valid", (name, x, r["diag"])
        for o in spec["outputs"]:
            vid = prog.var_by_name[o].id
            assert app.read(vid, worker=r["worker"]).tobytes() == want[vid].tobytes(), (name, x, o)
    print(name, "ok", len(genomes), "genomes", flush=True)
