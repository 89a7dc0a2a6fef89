"""Subprocess body for test_worker_pool_gpu: the runtime is a process-wide
singleton, so the multi-worker configuration runs in its own interpreter."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402

name, devices = sys.argv[1], json.loads(sys.argv[2])
g = json.loads((ROOT / "tests" / "golden" / f"{name}.json").read_text())
ev = B200Evaluator(g["spec"], devices=devices)
genomes = sorted(g["patterns"])
res = ev.measure_payloads(g["doc"], [g["patterns"][x] for x in genomes])
print(json.dumps({"workers": ev.runtime.n_workers,
                  "results": [[x, r["validity"], r["worker"], r["directive_execs"], r["launches"]]
                              for x, r in zip(genomes, res)]}))
