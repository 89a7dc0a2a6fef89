"""Sweep compiler kernel-shape options on one app and report the device time
of each generated kernel (b2o_bench_replay: back-to-back launches, CUDA
events).  Usage: python tools/kernel_sweep.py himeno_M 100100"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "himeno_M"
genome = sys.argv[2] if len(sys.argv) > 2 else "100100"
g = json.loads((ROOT / "tests" / "golden" / f"{name}.json").read_text())
variants = [json.loads(v) for v in sys.argv[3:]] or [
    {},
    {"flat_ppt": 2},
    {"flat_min_blocks": 4},
    {"flat_ppt": 2, "flat_min_blocks": 4},
    {"flat_min_blocks": 6},
    {"stencil": True},
]
for var in variants:
    spec = dict(g["spec"], **var)
    ev = B200Evaluator(spec, devices=[0])
    r = ev.measure_payloads(g["doc"], [g["patterns"][genome]])[0]
    app = ev.app_for(g["doc"])
    rep = app.bench_replay(g["patterns"][genome], warmup=3, steps=20)
    print(json.dumps({"variant": var, "validity": r["validity"], "ms_per_step": round(rep["ms_per_step"], 4),
                      "kernel_us": {k: round(v * 1e3, 2) for k, v in rep["kernel_ms"].items()}}), flush=True)
