"""Where the per-call time of B200Evaluator.measure_payloads goes, per
BASELINE app: Python wall per call vs the runtime's own reset / run /
fetch+compare split (B2O_TRACE=1, printed on stderr), with inputs resident
and from host buffers."""

import json
import os
import sys
import time
from pathlib import Path

os.environ["B2O_TRACE"] = "1"
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402

CASES = [("himeno_M", "100100"), ("nasmg_258", "100100"), ("matmul_1024", "10"), ("himeno_M_red", "100100100")]
for name, genome in CASES[: int(sys.argv[1]) if len(sys.argv) > 1 else None]:
    g = json.loads((ROOT / "tests" / "golden" / f"{name}.json").read_text())
    ev = B200Evaluator(g["spec"], devices=[0])
    pat = g["patterns"][genome]
    ev.measure_payloads(g["doc"], [pat])
    for resident in (False, True):
        for _ in range(3):
            p = dict(pat, inputs_resident=resident)
            t0 = time.perf_counter()
            r = ev.measure_payloads(g["doc"], [p])[0]
            print(json.dumps({"app": name, "resident": resident, "wall_ms": round((time.perf_counter() - t0) * 1e3, 3),
                              "time_ms": round(r["time_s"] * 1e3, 3), "h2d_MB": round(r["h2d_bytes"] / 1e6, 1),
                              "d2h_MB": round(r["d2h_bytes"] / 1e6, 1), "epilogue_MB": round(r["epilogue_bytes"] / 1e6, 1)}),
                  flush=True)
            sys.stderr.flush()
