"""Launch-bound Himeno L programs with and without the next-launch L2
prefetch (spec quad_nextpf): run time, launches, validity."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402

g = json.loads((ROOT / "tests" / "golden" / "himeno_L.json").read_text())
for var in ({}, {"quad_nextpf": True}, {}, {"quad_nextpf": True}):
    ev = B200Evaluator(dict(g["spec"], **var), devices=[0], timeout_seconds=120)
    ev.app_for(g["doc"])
    for x in ("001001", "001000", "000001", "010001", "100100"):
        r = ev.measure_payloads(g["doc"], [g["patterns"][x]])[0]
        print(json.dumps({"variant": var, "genome": x, "validity": r["validity"], "run_s": round(r["time_s"] or -1, 4),
                          "launches": r["launches"]}), flush=True)
    ev.close()
