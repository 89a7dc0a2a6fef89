"""Measure BASELINE configs 1, 3 and 4 (config 2/5 live in bench.py) on one
B200 next to the CPU oracle (C restatement, OpenMP on all host cores).

  config 1  matmul 1024 loop GA: all 4 genomes (a=2 is swept, src/ga.py:262-264)
  config 3  block offload GEMM 4096^3 + FFT 4096^2: every replacement subset
  config 4  NAS-MG resid 258^3 from a java_like IR document, GPU genomes

Prints one JSON object per config.  Usage: python tools/apps_bench.py"""

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle.cgen import CProgram  # noqa: E402
from oracle.externals import fft2d, gemm, make_binder  # noqa: E402
from paper_2011_03602_b200 import appspec  # noqa: E402
from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402
from paper_2011_03602_b200.ir import Program  # noqa: E402


def golden(n):
    return json.loads((ROOT / "tests" / "golden" / f"{n}.json").read_text())


def cpu_time(g, runs=1):
    prog = Program(g["doc"])
    st = appspec.initial_state(prog, g["spec"])
    c = CProgram(g["doc"], openmp=True, opt="-O3")
    best = 1e30
    for _ in range(runs):
        t0 = time.perf_counter()
        c.run(st, make_binder(g["doc"], g["spec"]))
        best = min(best, time.perf_counter() - t0)
    return best


cores = len(os.sched_getaffinity(0))

# -- config 1 ----------------------------------------------------------------
g = golden("matmul_1024")
ev = B200Evaluator(g["spec"], devices=[0], repeats=3)
app = ev.app_for(g["doc"])
rows = {}
for x in sorted(g["patterns"]):
    r = ev.measure_payloads(g["doc"], [g["patterns"][x]])[0]
    rows[x] = {"validity": r["validity"], "time_ms": round(r["time_s"] * 1e3, 3), "launches": r["launches"]}
rep = app.bench_replay(g["patterns"]["10"], warmup=3, steps=10)
k_ms = rep["kernel_ms"][0]
cpu = cpu_time(g)
print(json.dumps({"config": 1, "workload": "matmul 1024 fp32 loop nest (python_like IR), all genomes",
                  "genomes": rows, "i_root_kernel_ms": round(k_ms, 3),
                  "i_root_gflops": round(2 * 1024**3 / (k_ms * 1e-3) / 1e9, 1),
                  "cpu_oracle_ms": round(cpu * 1e3, 1), "cpu_cores": cores,
                  "best_speedup_vs_cpu": round(cpu / (min(v["time_ms"] for v in rows.values()) * 1e-3), 1),
                  "reference_all_cpu_ms": round(app.reference_time * 1e3, 1)}), flush=True)

# -- config 4 ----------------------------------------------------------------
g = golden("nasmg_258")
ev = B200Evaluator(g["spec"], devices=[0], repeats=3)
app = ev.app_for(g["doc"])
rows = {}
for x in ("100100", "111111", "010010", "001001", "000000"):
    r = ev.measure_payloads(g["doc"], [g["patterns"][x]])[0]
    rows[x] = {"validity": r["validity"], "time_ms": round(r["time_s"] * 1e3, 3), "launches": r["launches"],
               "h2d_MB": round(r["h2d_bytes"] / 1e6, 1), "d2h_MB": round(r["d2h_bytes"] / 1e6, 1)}
rep = app.bench_replay(g["patterns"]["100100"], warmup=3, steps=10)
pts = 256 ** 3
kern = {f"b2o_k{k}": {"us": round(v * 1e3, 2), "GB/s": round(12 * pts / (v * 1e-3) / 1e9, 1)}
        for k, v in rep["kernel_ms"].items()}
cpu = cpu_time(g)
print(json.dumps({"config": 4, "workload": "NAS-MG resid+correction 258^3, java_like IR doc, nit=4",
                  "genomes": rows, "kernels": kern, "cpu_oracle_ms": round(cpu * 1e3, 1), "cpu_cores": cores,
                  "speedup_100100_vs_cpu": round(cpu / (rows["100100"]["time_ms"] * 1e-3), 1)}), flush=True)

# -- config 3 ----------------------------------------------------------------
g = golden("blocks_4096")
v0 = g["variants"][0]
prog = Program(v0["doc"])
st = appspec.initial_state(prog, g["spec"])
ids = {n: prog.var_by_name[n].id for n in ("ma", "mb", "x")}
ref = {"mc": gemm(st[ids["ma"]], st[ids["mb"]], 4096, 4096, 4096, np.float32),
       "y": fft2d(st[ids["x"]], 4096, np.float32)}
ev = B200Evaluator(g["spec"], devices=[0], reference_outputs=ref)
rows = {}
for v in g["variants"]:
    names = [g["candidates"][i]["record"] for i in v["subset"]]
    r = ev.measure_payloads(v["doc"], [v["pattern"]])[0]
    rows["+".join(names) or "none"] = {"validity": r["validity"], "time_ms": round(r["time_s"] * 1e3, 2),
                                       "normwise_err": r["max_rel_err"], "block_MB": round(r["block_bytes"] / 1e6, 1)}
print(json.dumps({"config": 3, "workload": "gemm 4096^3 + fft 4096^2 via sample_db name matches, every subset",
                  "subsets": rows, "speedup_best_vs_cpu_original": round(rows["none"]["time_ms"] /
                                                                          min(r["time_ms"] for r in rows.values()), 1)}),
      flush=True)
