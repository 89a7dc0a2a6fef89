"""The distinct programs of the Himeno L GA (config 5): one measurement per
(GPU roots, plan) with its time, launches and transfer bytes -- where the GA's
wall time goes."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402

g = json.loads((ROOT / "tests" / "golden" / "himeno_L.json").read_text())
ev = B200Evaluator(g["spec"], devices=[0], timeout_seconds=120)
ev.app_for(g["doc"])
seen = {}
for x in sorted(g["patterns"]):
    k = ev.run_key("L", g["patterns"][x])
    seen.setdefault(k, x)
rows = []
for k, x in seen.items():
    r = ev.measure_payloads(g["doc"], [g["patterns"][x]])[0]
    rows.append((r.get("time_s") or 0.0, x, g["patterns"][x]["gpu_roots"], r["launches"], r["validity"],
                 round((r["h2d_bytes"] + r["d2h_bytes"]) / 1e6, 1)))
tot = sum(r[0] for r in rows)
for t, x, roots, launches, val, mb in sorted(rows, reverse=True):
    print(json.dumps({"genome": x, "roots": roots, "time_s": round(t, 4), "share": round(t / tot, 3),
                      "launches": launches, "validity": val, "transfer_MB": mb}), flush=True)
print(json.dumps({"programs": len(rows), "sum_s": round(tot, 3)}))
