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
# bring the GPU to its loaded clocks first (a cold start ramps for ~1 s)
_w = B200Evaluator(g["spec"], devices=[0])
_w.measure_payloads(g["doc"], [g["patterns"][genome]])
_wa = _w.app_for(g["doc"])
import time as _t  # noqa: E402
_t0 = _t.time()
import os as _os  # noqa: E402
while _t.time() - _t0 < (0.0 if _os.environ.get("KS_NOWARM") else 3.0):
    _wa.bench_replay(g["patterns"][genome], warmup=1, steps=50)
for var in variants:
    spec = dict(g["spec"], **var)
    ev = B200Evaluator(spec, devices=[0])
    r = ev.measure_payloads(g["doc"], [g["patterns"][genome]])[0]
    app = ev.app_for(g["doc"])
    rep = app.bench_replay(g["patterns"][genome], warmup=3, steps=20)
    print(json.dumps({"variant": var, "validity": r["validity"], "max_rel_err": r["max_rel_err"], "ms_per_step": round(rep["ms_per_step"], 4),
                      "kernel_us": {k: round(v * 1e3, 2) for k, v in rep["kernel_ms"].items()}}), flush=True)
