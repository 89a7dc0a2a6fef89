"""Fitness drift under concurrency (SURVEY.md §8e risk:
host-core and DRAM contention among concurrently measured patterns).

The 16 distinct Himeno L programs of the config-5 GA are timed (a) one at a
time and (b) all at once, LPT-ordered over W workers that share the host
(W workers on device 0: the host-side contention of W ranks on a W-GPU
box, plus GPU sharing that a W-GPU box would not have -- an upper bound for
GPU-resident programs).  Prints per-program solo/concurrent times, the drift
ratio, and whether the GA's ranking (and its winner) survives.

Usage: python tools/ga_drift.py [W=8] [app=himeno_L]"""

import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
name = sys.argv[2] if len(sys.argv) > 2 else "himeno_L"
g = json.loads((ROOT / "tests" / "golden" / f"{name}.json").read_text())
ev = B200Evaluator(g["spec"], devices=[0] * W, timeout_seconds=300, dedupe=False)
ev.app_for(g["doc"])
progs = {}
for x in sorted(g["patterns"]):
    progs.setdefault(ev.run_key(name, g["patterns"][x]), x)
genomes = list(progs.values())
pats = [g["patterns"][x] for x in genomes]

# warm every program once (compile/load, first-touch of pinned buffers)
ev.measure_payloads(g["doc"], pats)

solo = {}
for x, p in zip(genomes, pats):
    ts = [ev.measure_payloads(g["doc"], [p])[0]["time_s"] for _ in range(2)]
    solo[x] = min(ts)
# concurrent: the whole set in one batch, longest first (the runtime's LPT
# queue by predicted cost), W at a time
order = sorted(genomes, key=lambda x: -solo[x])
t0 = time.perf_counter()
res = ev.measure_payloads(g["doc"], [g["patterns"][x] for x in order])
wall = time.perf_counter() - t0
conc = {x: r["time_s"] for x, r in zip(order, res)}
valid = all(r["validity"] == "valid" for r in res)
rows = []
for x in order:
    rows.append({"genome": x, "solo_s": round(solo[x], 4), "concurrent_s": round(conc[x], 4),
                 "drift": round(conc[x] / solo[x], 3)})
    print(json.dumps(rows[-1]), flush=True)
rank_solo = sorted(genomes, key=lambda x: solo[x])
rank_conc = sorted(genomes, key=lambda x: conc[x])
n = len(genomes)
pairs = [(a, b) for i, a in enumerate(genomes) for b in genomes[i + 1:]]
conc_pairs = sum(1 for a, b in pairs if (solo[a] - solo[b]) * (conc[a] - conc[b]) > 0)
tau = (2 * conc_pairs - len(pairs)) / len(pairs)
print(json.dumps({"workers": W, "programs": n, "all_valid": valid, "batch_wall_s": round(wall, 3),
                  "sum_solo_s": round(sum(solo.values()), 3),
                  "winner_solo": rank_solo[0], "winner_concurrent": rank_conc[0],
                  "top3_solo": rank_solo[:3], "top3_concurrent": rank_conc[:3],
                  "kendall_tau": round(tau, 3),
                  "max_drift": max(r["drift"] for r in rows), "median_drift": sorted(r["drift"] for r in rows)[n // 2]}))
