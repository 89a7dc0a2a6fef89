#!/usr/bin/env python
"""Benchmark of the fitness-evaluation hot path on B200 (BASELINE.json).

Headline workload (BASELINE config 2): Himeno size M (129x129x257), inline
form, nn = 20 sweeps, executed under genome 100100 (Jacobi i-nest and copy
i-nest on the GPU, the gosa reduction nest on the host, as the reference's
screen requires) with the reference's hoisted transfer plan
(tests/golden/himeno_M.json, produced by the reference).  Metric: Himeno
algorithmic bytes per second of the whole app run, (60 + 8) B per interior
point per sweep.

* ``value``: one step = one whole run of the pattern (GPU launches, the
  plan's per-sweep ``gs`` downloads, the host gosa nest) with every input
  already resident in HBM (``inputs_resident``: the plan's input uploads are
  elided), timed by the runtime around the program run and its final stream
  synchronisation; W untimed warm-up steps, then K timed.  The 239 MB working
  set is larger than the 126 MB L2.
* ``e2e``: the same metric through the public plugin call
  (``B200Evaluator.measure_payloads``: host buffers, every H2D/D2H of the
  plan inside the timed call, output comparison), wall clock per call.
* ``gpu_launch_sequence`` / ``roofline``: the pattern's 40 kernel launches
  replayed on resident data, CUDA events on the worker stream; the roofline
  is the dominant kernel (Himeno Jacobi nest ``b2o_k1``).
* ``cpu_baseline``: the reference's own C emission of the same pattern
  (``gpuoffload.codegen.emit_annotated``, its ``#pragma acc`` nests run as
  OpenMP on every host core; oracle/refc.py), inputs loaded outside the timer.
* ``--impl reference``: that same reference program as the whole arm.
* ``apps``: BASELINE configs 1 (matmul 1024, python_like IR), 3 (GEMM 4096^3 +
  FFT 4096^2 through the block replacements) and 4 (NAS-MG resid 258^3,
  java_like IR), each with value / e2e / cpu_baseline / roofline.
* ``ga``: BASELINE config 5 (the reference GA, pop 64 x 20, on Himeno L) in
  patterns/s, with the reference GA + cost model (no program executed) timed
  beside it.

Under torchrun each rank drives its own GPU with its own replica (weak
scaling, no data-path collective); the step time is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# torchrun sets OMP_NUM_THREADS=1 per rank; the CPU reference arm (rank 0
# alone) and the N=1 cpu_baseline must use every host core they may, so the
# OpenMP runtime is sized before anything loads it
if "reference" in sys.argv or os.environ.get("WORLD_SIZE", "1") == "1":
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
for p in (ROOT / "baseline" / "_ref",):
    if p.exists():
        sys.path.append(str(p))

METRIC = "offloaded-app speedup vs CPU ref; Himeno GB/s; GA patterns evaluated/sec"
WORKLOAD = "himeno_M"
GENOME = "100100"
SIZE = (129, 129, 257)
BYTES_PER_POINT = 60 + 8  # Jacobi nest + copy nest (apps/himeno.py)


def golden(name: str) -> dict:
    return json.loads((ROOT / "tests" / "golden" / f"{name}.json").read_text())


def interior(size) -> int:
    return (size[0] - 2) * (size[1] - 2) * (size[2] - 2)


def decl_init(doc: dict, name: str) -> int:
    vid = next(v["id"] for v in doc["variables"] if v["name"] == name)
    for r in doc["regions"]:
        for s in r["statements"]:
            if s.get("decl") == vid and "init" in s:
                return int(s["init"]["num"])
    raise ValueError(f"{name} has no initialiser")


def sweeps_of(doc: dict) -> int:
    return decl_init(doc, "nn")


# ---------------------------------------------------------------------------
# plumbing
# ---------------------------------------------------------------------------


def visible_gpus() -> int:
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=30).stdout
        return max(1, sum(1 for ln in out.splitlines() if ln.startswith("GPU ")))
    except (OSError, subprocess.SubprocessError):
        return 1


class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        # one rank per GPU; more ranks than GPUs (testing on a 1-GPU box)
        # share devices round-robin
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0")) % visible_gpus()
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def _reduce(self, x: float, op) -> float:
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        return self._reduce(x, self.pg.ReduceOp.MAX) if self.pg else x

    def sum(self, x: float) -> float:
        return self._reduce(x, self.pg.ReduceOp.SUM) if self.pg else x

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


class Clocks:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.out,
                                         stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        # nvidia-smi takes a moment to start: the timed region begins once it
        # is sampling, so the samples cover the region
        t0 = time.time()
        while self.proc and time.time() - t0 < 5.0:
            self.out.flush()
            if Path(self.out.name).stat().st_size > 0:
                break
            time.sleep(0.02)
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        self.out.flush()
        rows = [ln.split(",") for ln in Path(self.out.name).read_text().splitlines() if ln.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for name, val in zip(names, r[5:9]):
                    if val.strip().lower() in ("active", "1"):
                        reasons.add(name)
            except (ValueError, IndexError):
                continue
        busy = [s for s in sm if s > 0.5 * mx] if mx else sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks() -> dict:
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        return dict(json.loads(f.read_text()), source="measured (MEASURED_PEAKS.json)")
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}


def compute_peaks() -> dict:
    """FP32 SIMT and TF32 rates measured on a pool B200 (profiles/r02)."""
    return json.loads((ROOT / "profiles" / "r02" / "compute_peaks.json").read_text())


def ncu_traffic(kernel: str) -> float | None:
    """dram bytes (read + write) per launch from the committed ncu capture."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if not f.exists():
        return None
    k = json.loads(f.read_text()).get("kernels", {}).get(kernel)
    return None if k is None else k.get("dram_bytes")


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# CPU side: the reference's own program (oracle/_ref)
# ---------------------------------------------------------------------------


def ref_cpu(g: dict, genome: str | None, runs: int, warm: int = 1, doc: dict | None = None,
            spec: dict | None = None) -> dict:
    """Time the reference's C emission of ``doc`` on the host: with a genome,
    its annotated c_openacc text with the acc compute nests run as OpenMP on
    every host core; without, the sequential pretty_print text on one core.
    Inputs are written into the program's globals before each run, outside
    the timer.  Falls back to the C restatement (kind "port") when neither a
    prebuilt object nor the reference package is available."""
    from oracle.externals import make_binder
    from oracle.refc import BASELINE_FLAGS, RefProgram, RefUnavailable
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.ir import Program

    doc = doc or g["doc"]
    spec = spec or g["spec"]
    prec = spec.get("precision", "fp32")
    state = appspec.initial_state(Program(doc), spec)
    binder = make_binder(doc, spec)
    openmp = genome is not None
    cores = len(os.sched_getaffinity(0)) if openmp else 1
    times = []
    try:
        rp = RefProgram.build(doc, prec, pattern=g["patterns"][genome] if openmp else None, openmp=openmp,
                              genome_loops=g.get("genome_loops"))
        kind = "reference"
        what = ("reference emission gpuoffload.codegen.emit_annotated(c_openacc) of genome "
                f"{genome}, acc nests as OpenMP, gcc {' '.join(BASELINE_FLAGS)}" if openmp
                else "reference emission gpuoffload.codegen.pretty_print, sequential, gcc -O2")
        for i in range(warm + runs):
            rp.load(state, binder)
            t0 = time.perf_counter()
            rp.execute()
            dt = time.perf_counter() - t0
            if i >= warm:
                times.append(dt)
    except RefUnavailable:
        from oracle.cgen import CProgram

        kind = "port"
        what = "C restatement oracle/cgen.py (reference emission unavailable), gcc -O2" + (" OpenMP" if openmp else "")
        prog = CProgram(doc, prec, openmp=openmp)
        for i in range(warm + runs):
            st = {k: v.copy() for k, v in state.items()}
            t0 = time.perf_counter()
            prog.run(st, binder, copy=False)
            dt = time.perf_counter() - t0
            if i >= warm:
                times.append(dt)
    return {"median_s": statistics.median(times), "min_s": min(times), "runs": len(times), "warm": warm,
            "cores": cores, "kind": kind, "what": what}


def cpu_line(value: float, unit: str, r: dict, sample: str) -> dict:
    return {"value": round(value, 3), "unit": unit, "cores": r["cores"], "kind": r["kind"],
            "sample": f"{sample}; {r['what']}; median of {r['runs']} runs after {r['warm']} warm-up, "
                      f"inputs loaded outside the timer", "cpu_model": cpu_model()}


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------


def resident_steps(ev, doc: dict, pat: dict, steps: int, warmup: int) -> dict:
    """W untimed + K timed whole-pattern runs with inputs resident in HBM;
    the runtime times each program run (host walk + kernels + transfers,
    final stream synchronisation)."""
    p = dict(pat, inputs_resident=True)
    for _ in range(warmup):
        r = ev.measure_payloads(doc, [p])[0]
        if r["validity"] != "valid":
            raise SystemExit(f"pattern {pat.get('genome')} invalid: {r}")
    runs = [ev.measure_payloads(doc, [p])[0] for _ in range(steps)]
    bad = [r for r in runs if r["validity"] != "valid"]
    if bad:
        raise SystemExit(f"pattern {pat.get('genome')} invalid: {bad[0]}")
    return {"ms_per_step": 1e3 * sum(r["time_s"] for r in runs) / len(runs),
            "launches_per_step": runs[-1]["launches"], "h2d_bytes": runs[-1]["h2d_bytes"],
            "d2h_bytes": runs[-1]["d2h_bytes"], "elided_bytes": runs[-1]["elided_bytes"]}


def e2e_calls(ev, doc: dict, pat: dict, n: int, warm: int = 1) -> dict:
    """Wall time of the public plugin call per step (host buffers)."""
    for _ in range(warm):
        ev.measure_payloads(doc, [pat])
    calls = []
    for _ in range(n):
        t0 = time.perf_counter()
        r = ev.measure_payloads(doc, [pat])[0]
        calls.append((time.perf_counter() - t0, r))
    last = calls[-1][1]
    if last["validity"] != "valid":
        raise SystemExit(f"pattern {pat.get('genome')} invalid: {last}")
    return {"s": statistics.median(t for t, _ in calls), "last": last}


def e2e_obj(value: float, unit: str, e: dict) -> dict:
    last = e["last"]
    return {"value": round(value, 3), "unit": unit, "h2d_bytes_per_step": int(last["h2d_bytes"]),
            "d2h_bytes_per_step": int(last["d2h_bytes"]), "ms_per_call": round(e["s"] * 1e3, 3),
            "app_run_ms": round(last["time_s"] * 1e3, 3), "call": "B200Evaluator.measure_payloads"}


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------


def reference_arm(args, dist: Dist) -> None:
    """The reference's own program for the same pattern on every host core
    (rank 0 only; other ranks exit without work)."""
    if dist.rank != 0:
        return
    g = golden(WORKLOAD)
    nn = sweeps_of(g["doc"])
    bytes_per_step = BYTES_PER_POINT * interior(SIZE) * nn
    r = ref_cpu(g, GENOME, runs=max(args.steps, 1), warm=max(args.warmup, 0))
    value = bytes_per_step / r["median_s"] / 1e9
    sample = f"one full Himeno M app run ({nn} sweeps) per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["median_s"] * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (Himeno initmt)",
        "config": {"workload": f"{WORKLOAD} inline nn={nn}, genome {GENOME} (the reference's acc nests on host cores)",
                   "size": list(SIZE), "sweeps": nn},
        "cpu_baseline": cpu_line(value, "GB/s", r, sample),
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def b200_arm(args, dist: Dist) -> None:
    from paper_2011_03602_b200.evaluator import B200Evaluator

    g = golden(WORKLOAD)
    nn = sweeps_of(g["doc"])
    pts = interior(SIZE)
    bytes_per_step = BYTES_PER_POINT * pts * nn
    pat = g["patterns"][GENOME]
    ev = B200Evaluator(g["spec"], devices=[dist.local_rank])
    app = ev.app_for(g["doc"])  # compile (cached) + load + reference run (untimed)
    check = ev.measure_payloads(g["doc"], [pat])[0]
    if check["validity"] != "valid":
        raise SystemExit(f"pattern {GENOME} invalid: {check}")
    dist.barrier()
    with Clocks(dist.local_rank) as clk:
        res = resident_steps(ev, g["doc"], pat, args.steps, max(args.warmup, 3))
        dist.barrier()
        rep = app.bench_replay(pat, warmup=max(args.warmup, 3), steps=args.steps)
        dist.barrier()
        e2e = e2e_calls(ev, g["doc"], pat, args.e2e_steps, warm=max(1, args.warmup // 2))
        dist.barrier()
    # the side measurements never cost the headline line: a failure is
    # reported in its own field
    apps = _guarded(apps_arm, args, dist) if args.apps else None
    red = _guarded(reductions_arm, args, dist) if args.reductions else None
    ga = _guarded(ga_arm, args, dist) if args.ga else None
    ops = _guarded(ops_arm, dist) if args.ops else None
    ms = dist.max(res["ms_per_step"])
    rep_ms = dist.max(rep["ms_per_step"])
    e2e_s = dist.max(e2e["s"])
    value = dist.world * bytes_per_step / (ms * 1e-3) / 1e9
    e2e_value = dist.world * bytes_per_step / e2e_s / 1e9
    pk = peaks()
    jac_loop = g["genome_loops"][0]  # the Jacobi i-loop is the first genome bit
    kms = rep["kernel_ms"].get(jac_loop)
    achieved = 60 * pts / (kms * 1e-3) / 1e9 if kms else None
    if dist.rank != 0:
        return
    # the CPU baseline is timed on rank 0 at N=1 only (other ranks would
    # contend for the same host cores)
    cpu = ref_cpu(g, GENOME, runs=5, warm=2) if dist.world == 1 else None
    cpu1 = ref_cpu(g, None, runs=2) if dist.world == 1 else None
    sample = f"one full Himeno M app run ({nn} sweeps)"
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (Himeno initmt)",
        "config": {"workload": f"{WORKLOAD} inline nn={nn}, genome {GENOME} (Jacobi+copy nests on GPU, gosa nest "
                               "on host), reference hoisted plan", "size": list(SIZE), "sweeps": nn,
                   "step": "one whole app run, inputs resident in HBM (plan's input uploads elided); per-sweep gs "
                           "downloads and the host gosa nest inside the step",
                   "timing": "runtime steady clock around the program run incl. final stream synchronisation "
                             "(a host+GPU program); kernels by CUDA events on the worker stream",
                   "l2": "inputs larger than L2 (239 MB working set > 126 MB)", "parallelism": f"replicas{dist.world}"},
        "gpu_launches": int(res["launches_per_step"] * args.steps),
        "e2e": e2e_obj(e2e_value, "GB/s", e2e),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                     "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4) if achieved else None,
                     "traffic": ncu_traffic(f"b2o_k{jac_loop}"), "kernel": f"b2o_k{jac_loop} (Himeno Jacobi nest)",
                     "kernel_us": round(kms * 1e3, 2) if kms else None, "bytes_per_launch": 60 * pts,
                     "peak_source": pk.get("source")},
        "gpu_launch_sequence": {"ms_per_step": round(rep_ms, 4),
                                "GBps": round(dist.world * bytes_per_step / (rep_ms * 1e-3) / 1e9, 1),
                                "share_of_step": round(rep_ms / ms, 4),
                                "launches_per_step": int(rep["launches_per_step"]),
                                "note": "the pattern's kernels replayed back to back on resident data (CUDA events); "
                                        "the rest of the step is the host gosa nest + gs downloads"},
        "kernels_us": {f"b2o_k{k}": round(v * 1e3, 2) for k, v in rep["kernel_ms"].items()},
        "step_transfers": {"h2d_bytes": int(res["h2d_bytes"]), "d2h_bytes": int(res["d2h_bytes"]),
                           "elided_bytes": int(res["elided_bytes"])},
        "cpu_baseline": cpu_line(bytes_per_step / cpu["median_s"] / 1e9, "GB/s", cpu, sample) if cpu else None,
        "cpu_baseline_1core": cpu_line(bytes_per_step / cpu1["median_s"] / 1e9, "GB/s", cpu1, sample)
        if cpu1 else None,
        "app_speedup_vs_cpu": {"e2e": round(cpu["median_s"] / e2e_s, 2), "value": round(cpu["median_s"] / (ms * 1e-3), 2)}
        if cpu else None,
        "app_speedup_vs_cpu_1core": {"e2e": round(cpu1["median_s"] / e2e_s, 2),
                                     "value": round(cpu1["median_s"] / (ms * 1e-3), 2)} if cpu1 else None,
        "apps": apps,
        "ga": ga,
        "ops": ops,
        "reductions_opt_in": red,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def _guarded(fn, *args) -> dict:
    try:
        return fn(*args)
    except Exception as exc:  # noqa: BLE001 -- reported, not raised
        import traceback

        traceback.print_exc(file=sys.stderr)
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


# ---------------------------------------------------------------------------
# BASELINE configs 1, 3, 4
# ---------------------------------------------------------------------------


def _app_entry(name: str, g: dict, genome: str, unit: str, work: float, args, dist: Dist, kernel_loop: int,
               kernel_work: float, kernel_bound: str, kernel_peak: float, peak_source: str, kernel_name: str,
               cpu_sample: str, cpu_runs: int = 5, cpu1_runs: int = 1, doc=None, pat=None, ev=None,
               cpu=None) -> dict:
    from paper_2011_03602_b200.evaluator import B200Evaluator

    doc = doc or g["doc"]
    pat = pat or g["patterns"][genome]
    ev = ev or B200Evaluator(g["spec"], devices=[dist.local_rank])
    app = ev.app_for(doc)
    res = resident_steps(ev, doc, pat, max(3, args.steps // 5), 3)
    e2e = e2e_calls(ev, doc, pat, max(3, args.e2e_steps))
    # the loop kernels' launch sequence replayed on resident data (block
    # library calls are not replayable launches: their kernels are timed on
    # resident buffers by ops_arm)
    rep = app.bench_replay(pat, warmup=3, steps=10) if kernel_loop is not None else {"ms_per_step": None,
                                                                                       "kernel_ms": {}}
    kms = rep["kernel_ms"].get(kernel_loop) if kernel_loop is not None else None
    ms = dist.max(res["ms_per_step"])
    e2e_s = dist.max(e2e["s"])
    scale = 1e9 if unit.startswith("G") else 1e12
    out = {"workload": name, "genome": genome, "unit": unit, "value": round(dist.world * work / (ms * 1e-3) / scale, 3),
           "ms_per_step": round(ms, 4), "gpu_launches_per_step": int(res["launches_per_step"]),
           "e2e": e2e_obj(dist.world * work / e2e_s / scale, unit, e2e),
           "gpu_launch_sequence_ms": round(rep["ms_per_step"], 4) if rep["ms_per_step"] else None,
           "kernels_us": {f"b2o_k{k}": round(v * 1e3, 2) for k, v in rep["kernel_ms"].items()}}
    if kms:
        kscale = 1e9 if kernel_bound == "hbm" else 1e12
        achieved = kernel_work / (kms * 1e-3) / kscale
        out["roofline"] = {"bound": kernel_bound, "kernel": kernel_name, "achieved": round(achieved, 2),
                           "peak": kernel_peak, "unit": "GB/s" if kernel_bound == "hbm" else "TFLOP/s",
                           "frac": round(achieved / kernel_peak, 4), "kernel_us": round(kms * 1e3, 2),
                           "peak_source": peak_source}
    if dist.world == 1 and dist.rank == 0:
        c = cpu or ref_cpu(g, genome, runs=cpu_runs, warm=2, doc=doc)
        out["cpu_baseline"] = cpu_line(work / c["median_s"] / scale, unit, c, cpu_sample)
        out["speedup_vs_cpu"] = {"e2e": round(c["median_s"] / e2e_s, 2), "value": round(c["median_s"] / (ms * 1e-3), 2)}
        if cpu1_runs and cpu is None:
            c1 = ref_cpu(g, None, runs=cpu1_runs, warm=0, doc=doc)
            out["cpu_baseline_1core"] = cpu_line(work / c1["median_s"] / scale, unit, c1, cpu_sample)
    return out


def apps_arm(args, dist: Dist) -> dict:
    pk = peaks()
    cp = compute_peaks()
    out = {}
    # config 1: Python matmul 1024 loop nest (python_like IR), i-root pattern:
    # the register-tiled k-reduction kernel, bit-exact (no FMA contraction)
    g = golden("matmul_1024")
    n = 1024
    out["config1_matmul_1024"] = _app_entry(
        "matmul 1024^3 fp32 loop nest (python_like IR), genome 10 (i-nest on the GPU)", g, "10", "GFLOP/s",
        2 * n ** 3, args, dist, kernel_loop=g["genome_loops"][0], kernel_work=2 * n ** 3, kernel_bound="fp32",
        kernel_peak=cp["fp32_no_fma_tflops"], peak_source="measured FP32 FMUL+FADD rate (profiles/r02/compute_peaks.json;"
        " the loop's C semantics forbid FMA contraction)", kernel_name="k-tile kernel (register-tiled k-reduction)",
        cpu_sample="one full matmul 1024 app run")
    # config 4: NAS-MG resid + correction 258^3 (java_like IR), genome 100100
    g = golden("nasmg_258")
    n = 258
    nit = decl_init(g["doc"], "nit")
    pts = (n - 2) ** 3
    out["config4_nasmg_258"] = _app_entry(
        f"NAS-MG resid + correction 258^3 fp32 (java_like IR), nit={nit}, genome 100100", g, "100100", "GB/s",
        24 * pts * nit, args, dist, kernel_loop=g["genome_loops"][0], kernel_work=12 * pts, kernel_bound="hbm",
        kernel_peak=pk["hbm_gbs"], peak_source=pk.get("source"),
        kernel_name="plane-marching quad kernel (resid nest; 12 B/point: u, v read, r written)",
        cpu_sample=f"one full NAS-MG app run ({nit} iterations; 24 B/point/iteration: resid 12 + correction 12)")
    # config 3: GEMM 4096^3 + FFT 4096^2 through the block replacements
    out["config3_blocks_4096"] = blocks_entry(args, dist, pk, cp)
    return out


def blocks_entry(args, dist: Dist, pk: dict, cp: dict) -> dict:
    import numpy as np

    from oracle.externals import fft2d, gemm
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.evaluator import B200Evaluator
    from paper_2011_03602_b200.ir import Program

    g = golden("blocks_4096")
    n = 4096
    v0 = g["variants"][0]
    both = next(v for v in g["variants"] if len(v["subset"]) == 2)
    prog = Program(v0["doc"])
    st = appspec.initial_state(prog, g["spec"])
    ids = {k: prog.var_by_name[k].id for k in ("ma", "mb", "x")}
    ref = {"mc": gemm(st[ids["ma"]], st[ids["mb"]], n, n, n, np.float32),
           "y": fft2d(st[ids["x"]], n, np.float32)}
    ev = B200Evaluator(g["spec"], devices=[dist.local_rank], reference_outputs=ref)
    import math

    work = 2 * n ** 3 + 5 * n * n * math.log2(n * n)
    # CPU baseline: the same two operations as host library calls (numpy:
    # OpenBLAS sgemm on every core + pocketfft fft2 on complex64)
    cpu = None
    if dist.world == 1 and dist.rank == 0:
        a = st[ids["ma"]].reshape(n, n)
        b = st[ids["mb"]].reshape(n, n)
        xc = st[ids["x"]].reshape(n, n, 2)
        xc = (xc[..., 0] + 1j * xc[..., 1]).astype(np.complex64)
        times = []
        for i in range(3):
            t0 = time.perf_counter()
            a @ b
            np.fft.fft2(xc)
            if i:
                times.append(time.perf_counter() - t0)
        cpu = {"median_s": statistics.median(times), "min_s": min(times), "runs": len(times), "warm": 1,
               "cores": len(os.sched_getaffinity(0)), "kind": "port",
               "what": "numpy float32 matmul (OpenBLAS, all cores) + numpy.fft.fft2 complex64 -- the opaque calls' "
                       "CPU library equivalent (the reference has no CPU implementation of gemm/fft)"}
    out = _app_entry("gemm 4096^3 + fft 4096^2 (sample_db name matches), both replaced: cublas_gemm -> tcgen05 "
                     "3xTF32, cufft_exec -> cluster FFT", g, "blocks", "GFLOP/s", work, args, dist,
                     kernel_loop=None, kernel_work=0, kernel_bound="tensor", kernel_peak=1.0, peak_source="",
                     kernel_name="", cpu_sample="GEMM 4096^3 + FFT 4096^2 on the host", doc=both["doc"],
                     pat=both["pattern"], ev=ev, cpu=cpu)
    # dominant kernels of the step: the MMA kernel (tensor) and the FFT (HBM)
    ops = ops_arm(dist)
    out["roofline"] = dict(ops["gemm_roofline"])
    out["fft_roofline"] = ops["fft_roofline"]
    out["max_rel_err_elementwise_mc"] = e2e_last_err(ev, both)
    return out


def e2e_last_err(ev, variant) -> float:
    r = ev.measure_payloads(variant["doc"], [variant["pattern"]])[0]
    return r["max_rel_err"]


def reductions_arm(args, dist: Dist) -> dict:
    """Opt-in reduction screen (reductions.py): the same Himeno M app with
    the gosa nest offloaded too (genome 100100100: no per-sweep gs download,
    no host gosa nest).  Not the headline (the genome differs from the
    reference screen's); reported beside it, same bytes metric."""
    from paper_2011_03602_b200.evaluator import B200Evaluator

    g = golden("himeno_M_red")
    nn = sweeps_of(g["doc"])
    bytes_per_step = BYTES_PER_POINT * interior(SIZE) * nn
    ev = B200Evaluator(g["spec"], devices=[dist.local_rank])
    pat = g["patterns"]["100100100"]
    res = resident_steps(ev, g["doc"], pat, max(3, args.e2e_steps), 2)
    e2e = e2e_calls(ev, g["doc"], pat, max(3, args.e2e_steps))
    e2e_s = dist.max(e2e["s"])
    ms = dist.max(res["ms_per_step"])
    return {"genome": "100100100", "value_GBps": round(bytes_per_step / (ms * 1e-3) / 1e9, 3),
            "e2e_GBps": round(bytes_per_step / e2e_s / 1e9, 3), "ms_per_call": round(e2e_s * 1e3, 3),
            "app_run_ms": round(e2e["last"]["time_s"] * 1e3, 3), "h2d_bytes": int(e2e["last"]["h2d_bytes"]),
            "d2h_bytes": int(e2e["last"]["d2h_bytes"]),
            "note": "gosa summed on the GPU in loop order, bit-identical to the sequential CPU loop (b2o_exact_sum_f32)"}


def ga_arm(args, dist: Dist) -> dict | None:
    """BASELINE config 5: the reference GA (pop 64 x 20 generations) on Himeno
    L, each generation's uncached genomes measured in one batch; under
    torchrun the batch is sharded LPT over the ranks (one B200 each) and the
    results are all-gathered (search.ShardedEvaluator).  patterns/sec =
    evaluations_performed / GA wall time (max over ranks).  Beside it: the
    reference's own GA driving its CostModelEvaluator (no program executed),
    1 core -- the reference's fitness path as it ships."""
    try:
        from gpuoffload.evaluators import CostModelEvaluator
        from gpuoffload.ga import GAParams, run_search
        from gpuoffload.irdoc import load_ir_document
        from gpuoffload.screen import screen_model
    except ImportError as exc:
        return {"skipped": f"reference package not importable: {exc}"}
    from paper_2011_03602_b200.evaluator import B200Evaluator
    from paper_2011_03602_b200.search import ShardedEvaluator, run_search_batched

    g = golden(args.ga_workload)
    model = load_ir_document(json.dumps(g["doc"]))
    ev = B200Evaluator(g["spec"], devices=[dist.local_rank], timeout_seconds=args.ga_timeout,
                       dedupe=bool(args.ga_dedupe))
    ev.app_for(g["doc"])  # compile + load + all-CPU reference run, untimed
    evaluator = ShardedEvaluator(ev) if dist.world > 1 else ev
    params = GAParams(population_size=args.ga_pop, generations=args.ga_gens, seed=args.ga_seed)
    dist.barrier()
    t0 = time.perf_counter()
    stats: dict = {}
    res = run_search_batched(model, screen_model(model), evaluator, params, stats=stats)
    wall = dist.max(time.perf_counter() - t0)
    valid = sum(1 for r in ev.log if r.get("validity") == "valid")
    local = dist.sum(float(len(ev.log)))
    fit_sum = dist.sum(float(sum(r.get("time_s") or 0.0 for r in ev.log)))
    programs = dist.sum(float(ev.programs_executed))
    out = {"workload": f"{args.ga_workload} inline nn={sweeps_of(g['doc'])}, pop {args.ga_pop} x {args.ga_gens} gens",
           "patterns_per_s": round(res.evaluations_performed / wall, 3), "evaluations": res.evaluations_performed,
           "cache_hits": res.cache_hits, "wall_s": round(wall, 3), "best_genome": "".join(map(str, res.best_genome)),
           "best_time_s": res.best_time, "measured_by_all_ranks": int(local), "valid_on_rank0": valid,
           "speculated": stats.get("speculated", 0), "speculated_unused": stats.get("speculated_unused", 0),
           "sum_fitness_s_all_ranks": round(fit_sum, 3),
           "programs_executed_all_ranks": int(programs),
           "dedupe": ("genomes whose GPU roots and transfer plan coincide share one program run "
                      "(B200Evaluator.run_key, SURVEY.md §8e)") if args.ga_dedupe else "off",
           "history_evals": [h.evaluations for h in res.history][:6]}
    if dist.world == 1 and args.ga_workers > 1:
        out["overlapped"] = _guarded(ga_overlapped, args, g, model, params, out["best_genome"])
    if dist.rank == 0:
        t0 = time.perf_counter()
        ref = run_search(model, screen_model(model), CostModelEvaluator(), params)
        ref_wall = time.perf_counter() - t0
        out["reference_ga_cost_model"] = {
            "patterns_per_s": round(ref.evaluations_performed / ref_wall, 1), "wall_s": round(ref_wall, 3),
            "evaluations": ref.evaluations_performed, "best_genome": "".join(map(str, ref.best_genome)),
            "cores": 1, "what": "reference run_search + CostModelEvaluator (synthetic cost, no program executed), "
                                "same model/params; the fitness the reference ships with"}
    return out


def ga_overlapped(args, g: dict, model, params, best_solo: str) -> dict:
    """The same GA with W workers sharing the one B200 (host loops of one
    pattern overlap the GPU work of another; the runtime in a child process,
    isolated.IsolatedEvaluator), and the k fastest genomes re-measured alone
    at the end (run_search_batched confirm_top) because concurrent patterns
    drift (tools/ga_drift.py).  Not the headline GA: a throughput option."""
    from gpuoffload.screen import screen_model

    from paper_2011_03602_b200.isolated import IsolatedEvaluator
    from paper_2011_03602_b200.search import run_search_batched

    W = int(args.ga_workers)
    ev = IsolatedEvaluator(g["spec"], devices=[0] * W, timeout_seconds=args.ga_timeout, dedupe=bool(args.ga_dedupe))
    try:
        first = sorted(g["patterns"])[0]
        ev.measure_payloads(g["doc"], [g["patterns"][first]])  # child up, program loaded, reference run (untimed)
        stats: dict = {}
        t0 = time.perf_counter()
        res = run_search_batched(model, screen_model(model), ev, params, stats=stats, confirm_top=3, confirm_repeats=2)
        wall = time.perf_counter() - t0
    finally:
        ev.close()
    best = "".join(map(str, res.best_genome))
    return {"workers_per_gpu": W, "patterns_per_s": round(res.evaluations_performed / wall, 3),
            "evaluations": res.evaluations_performed, "wall_s": round(wall, 3), "best_genome": best,
            "best_time_s": res.best_time, "one_worker_best_genome": best_solo,
            "same_program_as_one_worker": IsolatedEvaluator.run_key("", g["patterns"][best])
            == IsolatedEvaluator.run_key("", g["patterns"][best_solo]),
            "noise_note": "Himeno L's two fastest programs (100100, 100010) are ~1 % apart: single measurements "
                          "(the reference GA's one per genome) swap them from run to run; the confirmation times "
                          "the top 3 alone, best of 2",
            "confirmed_top3": stats.get("confirmed"), "programs_executed": ev.programs_executed,
            "note": "wall includes the solo re-measurement of the 3 fastest genomes"}


def ops_arm(dist: Dist) -> dict:
    """BASELINE config 3 kernels on resident data: the tcgen05 3xTF32 GEMM
    (cublas_gemm replacement) at 4096^3 and the radix-16 FFT (cufft_exec
    replacement) at 4096^2, CUDA events on the launching stream."""
    import ctypes as ct

    import numpy as np

    from paper_2011_03602_b200.runtime import lib

    try:
        import torch
    except ImportError:
        return {"skipped": "torch unavailable for device buffers"}
    dev = torch.device("cuda", dist.local_rank)
    torch.cuda.set_device(dev)
    L = lib()
    st = torch.cuda.current_stream().cuda_stream
    n = 4096
    a, b = torch.rand(n, n, device=dev), torch.rand(n, n, device=dev)
    c = torch.empty(n, n, device=dev)
    x = torch.rand(2 * n * n, device=dev) * 2 - 1
    y = torch.empty_like(x)

    def timed(fn, iters=10):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    gemm_ms = timed(lambda: L.b2o_gemm_f32(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, st))
    prep, mma = [], []
    for _ in range(10):
        p_ms, m_ms = ct.c_double(), ct.c_double()
        L.b2o_gemm_f32_phases(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, st, ct.byref(p_ms), ct.byref(m_ms))
        prep.append(p_ms.value)
        mma.append(m_ms.value)
    mma_ms = statistics.median(mma)
    prep_ms = statistics.median(prep)
    cd = c[:256].double().cpu().numpy()
    rd = (a[:256].double() @ b.double()).cpu().numpy()
    err = float(np.linalg.norm(cd - rd) / np.linalg.norm(rd))
    elem = float(np.max(np.abs(cd - rd) / np.abs(rd)))
    fft_ms = timed(lambda: L.b2o_fft2d_c64(x.data_ptr(), y.data_ptr(), n, st))
    nh = 1 << 26  # 256 MB of int32 (> L2)
    hd = torch.randint(0, 256, (nh,), dtype=torch.int32, device=dev)
    hh = torch.zeros(256, dtype=torch.int32, device=dev)
    hist_ms = timed(lambda: L.b2o_histogram(hd.data_ptr(), nh, hh.data_ptr(), 256, 0, st))
    pk = peaks()
    cp = compute_peaks()
    tf32_peak = cp["tf32_nominal_dense_tflops"]
    tf32_issued = 3 * 2 * n ** 3 / (gemm_ms * 1e-3) / 1e12
    tf32_kernel = 3 * 2 * n ** 3 / (mma_ms * 1e-3) / 1e12
    fft_gbs = 2 * 2 * 8 * n * n / (fft_ms * 1e-3) / 1e9
    return {"gemm_4096_ms": round(gemm_ms, 4), "gemm_tflops_fp32_equiv": round(2 * n ** 3 / (gemm_ms * 1e-3) / 1e12, 1),
            "gemm_tf32_tflops_issued": round(tf32_issued, 1),
            "gemm_roofline": {"bound": "tensor", "kernel": "gemm_tc_pair_kernel (cta_group::2, persistent)",
                              "achieved": round(tf32_kernel, 1), "peak": round(tf32_peak, 1),
                              "unit": "TFLOP/s", "frac": round(tf32_kernel / tf32_peak, 3),
                              "kernel_ms": round(mma_ms, 4), "prep_ms": round(prep_ms, 4),
                              "op_frac_incl_prep": round(tf32_issued / tf32_peak, 3),
                              "vs_cublas_tf32_measured": round(tf32_kernel / cp["tf32_cublas_tflops"], 3),
                              "peak_source": "nominal dense TF32 1.1 PFLOP/s (cuBLAS's own TF32 GEMM measures "
                                             f"{cp['tf32_cublas_tflops']} TFLOP/s here, below this kernel; "
                                             "profiles/r02/compute_peaks.json); 3 TF32 passes counted"},
            "gemm_err_rows0_255": {"normwise": err, "elementwise_max_rel": elem},
            "fft_4096_ms": round(fft_ms, 4),
            "fft_roofline": {"bound": "hbm", "achieved": round(fft_gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                             "frac": round(fft_gbs / pk["hbm_gbs"], 3), "bytes": "2 passes x read+write complex64"},
            "histogram_64M_256bins_ms": round(hist_ms, 4),
            "histogram_roofline": {"bound": "hbm", "achieved": round(4 * nh / (hist_ms * 1e-3) / 1e9, 1),
                                   "peak": pk["hbm_gbs"], "unit": "GB/s",
                                   "frac": round(4 * nh / (hist_ms * 1e-3) / 1e9 / pk["hbm_gbs"], 3),
                                   "bytes": "4 B read per element"}}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--apps", type=int, default=1, help="also measure BASELINE configs 1, 3, 4")
    ap.add_argument("--ga", type=int, default=1, help="also measure GA patterns/sec (config 5)")
    ap.add_argument("--ops", type=int, default=1, help="also time the GEMM/FFT/histogram block kernels (config 3)")
    ap.add_argument("--reductions", type=int, default=1, help="also time the opt-in reduction pattern")
    ap.add_argument("--ga-workload", default="himeno_L")
    ap.add_argument("--ga-pop", type=int, default=64)
    ap.add_argument("--ga-gens", type=int, default=20)
    ap.add_argument("--ga-seed", type=int, default=20201106)
    ap.add_argument("--ga-timeout", type=float, default=120.0)
    ap.add_argument("--ga-dedupe", type=int, default=1, help="run identical programs (same GPU roots + plan) once")
    ap.add_argument("--ga-workers", type=int, default=4,
                    help="also run the GA with this many workers sharing the B200 (N=1 only; 1 = skip)")
    args = ap.parse_args()
    dist = Dist()
    try:
        if args.impl == "reference":
            reference_arm(args, dist)
        else:
            b200_arm(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
