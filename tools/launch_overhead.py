"""Per-launch cost of launch-bound patterns (Himeno L, k-rooted copy nest):
the pattern's own run (host walk + callbacks + cuLaunchKernel per k-row)
against a replay of the same recorded launches (cuLaunchKernel only)."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "himeno_L"
g = json.loads((ROOT / "tests" / "golden" / f"{name}.json").read_text())
ev = B200Evaluator(g["spec"], devices=[0], timeout_seconds=120)
app = ev.app_for(g["doc"])
for x in sys.argv[2:] or ["000001", "000100", "001000", "100000"]:
    r = ev.measure_payloads(g["doc"], [g["patterns"][x]])[0]
    rep = app.bench_replay(g["patterns"][x], warmup=1, steps=2)
    n = rep["launches_per_step"]
    print(json.dumps({"genome": x, "run_s": round(r["time_s"], 4), "launches": r["launches"],
                      "replay_ms": round(rep["ms_per_step"], 3),
                      "replay_us_per_launch": round(rep["ms_per_step"] * 1e3 / max(n, 1), 3)}), flush=True)
