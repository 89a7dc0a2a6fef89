"""Where the per-call time of B200Evaluator.measure_payloads goes (Himeno M,
genome 100100 and the opt-in 100100100): Python wall per call vs the
runtime's own reset / run / fetch+compare split (B2O_TRACE=1)."""

import json
import os
import sys
import time
from pathlib import Path

os.environ["B2O_TRACE"] = "1"
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402

for name, genome in (("himeno_M", "100100"), ("himeno_M_red", "100100100")):
    g = json.loads((ROOT / "tests" / "golden" / f"{name}.json").read_text())
    ev = B200Evaluator(g["spec"], devices=[0])
    pat = g["patterns"][genome]
    ev.measure_payloads(g["doc"], [pat])
    for _ in range(3):
        t0 = time.perf_counter()
        r = ev.measure_payloads(g["doc"], [pat])[0]
        print(json.dumps({"app": name, "wall_ms": round((time.perf_counter() - t0) * 1e3, 3),
                          "time_ms": round(r["time_s"] * 1e3, 3)}), flush=True)
