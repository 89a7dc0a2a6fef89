#!/usr/bin/env python
"""Benchmark of the fitness-evaluation hot path on B200 (BASELINE.json config 2).

Workload: Himeno size M (129x129x257), inline form, nn = 20 sweeps, executed
under the all-GPU offload pattern (genome 100100: Jacobi i-nest and copy
i-nest on the GPU, gosa reduction on the host) with the reference's hoisted
transfer plan (tests/golden/himeno_M.json, produced by the reference).

* ``value`` (GB/s): one step = the pattern's whole GPU launch sequence for one
  app run (20 Jacobi + 20 copy launches), replayed on data already resident in
  HBM, timed with CUDA events on the worker stream; algorithmic bytes =
  (60 + 8) B per interior point per sweep.  The 239 MB working
  set exceeds the 126 MB L2.
* ``e2e``: the same metric through the public plugin call
  (``B200Evaluator.measure_payloads``: host buffers, the plan's H2D/D2H, the
  host gosa nest, output comparison), wall clock per call.
* ``--impl reference``: the reference CPU implementation of the path (the C
  restatement in oracle/, all-CPU genome, OpenMP on every host core).

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


def sweeps_of(doc: dict) -> int:
    for v in doc["variables"]:
        if v["name"] == "nn":
            nn_id = v["id"]
    for r in doc["regions"]:
        for s in r["statements"]:
            if s.get("decl") == nn_id and "init" in s:
                return int(s["init"]["num"])
    raise ValueError("nn not found")


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

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

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
        return dict(json.loads(f.read_text()), source="measured")
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(kernel: str) -> float | None:
    """dram bytes (read + write) per launch from the committed ncu capture."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if not f.exists():
        return None
    data = json.loads(f.read_text())
    k = data.get("kernels", {}).get(kernel)
    return None if k is None else k.get("dram_bytes")


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_run(doc: dict, spec: dict, openmp: bool, runs: int) -> tuple[float, int]:
    from oracle.cgen import CProgram
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.ir import Program

    state = appspec.initial_state(Program(doc), spec)
    prog = CProgram(doc, spec.get("precision", "fp32"), openmp=openmp, opt="-O3")
    best = float("inf")
    for _ in range(runs):
        t0 = time.perf_counter()
        prog.run(state)
        best = min(best, time.perf_counter() - t0)
    cores = len(os.sched_getaffinity(0)) if openmp else 1
    return best, cores


def reference_arm(args, dist: Dist) -> None:
    if dist.rank != 0:
        return
    g = golden(WORKLOAD)
    nn = sweeps_of(g["doc"])
    bytes_per_step = BYTES_PER_POINT * interior(SIZE) * nn
    from oracle.cgen import CProgram
    from paper_2011_03602_b200 import appspec
    from paper_2011_03602_b200.ir import Program

    state = appspec.initial_state(Program(g["doc"]), g["spec"])
    prog = CProgram(g["doc"], "fp32", openmp=True, opt="-O3")
    for _ in range(max(args.warmup, 0)):
        prog.run(state)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        prog.run(state)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    cores = len(os.sched_getaffinity(0))
    value = bytes_per_step / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (Himeno initmt)",
        "config": {"workload": f"{WORKLOAD} inline nn={nn}, all-CPU genome 000000", "size": list(SIZE),
                   "sweeps": nn},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"one full Himeno M app run ({nn} sweeps) per step, C restatement (oracle/cgen.py) "
                                   f"gcc -O3 OpenMP", "cpu_model": cpu_model()},
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
    # correctness of the benchmarked pattern first
    check = ev.measure_payloads(g["doc"], [pat])[0]
    if check["validity"] != "valid":
        raise SystemExit(f"pattern {GENOME} invalid: {check}")
    dist.barrier()
    with Clocks(dist.local_rank) as clk:
        rep = app.bench_replay(pat, warmup=max(args.warmup, 3), steps=args.steps)
        dist.barrier()
        e2e = []
        for _ in range(max(1, args.warmup // 2)):
            ev.measure_payloads(g["doc"], [pat])
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            r = ev.measure_payloads(g["doc"], [pat])[0]
            e2e.append((time.perf_counter() - t0, r))
        dist.barrier()
    # the side measurements never cost the headline line: a failure is
    # reported in its own field
    red = _guarded(reductions_arm, args, dist) if args.reductions else None
    ga = _guarded(ga_arm, args, dist) if args.ga else None
    ops = _guarded(ops_arm, dist) if args.ops else None
    ms = dist.max(rep["ms_per_step"])
    e2e_s = dist.max(statistics.median(t for t, _ in e2e))
    last = e2e[-1][1]
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
    cpu_s, cores = cpu_run(g["doc"], g["spec"], openmp=True, runs=1) if dist.world == 1 else (None, None)
    # the faithful sequential semantics too (both reported)
    cpu1_s, _ = cpu_run(g["doc"], g["spec"], openmp=False, runs=1) if dist.world == 1 else (None, None)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": dist.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (Himeno initmt)",
        "config": {"workload": f"{WORKLOAD} inline nn={nn}, genome {GENOME} (Jacobi+copy nests on GPU, "
                               "reference hoisted plan)", "size": list(SIZE), "sweeps": nn,
                   "l2": "inputs larger than L2 (239 MB working set > 126 MB)", "parallelism": f"replicas{dist.world}"},
        "gpu_launches": int(rep["launches_per_step"] * args.steps),
        "e2e": {"value": round(e2e_value, 3), "unit": "GB/s", "h2d_bytes_per_step": int(last["h2d_bytes"]),
                "d2h_bytes_per_step": int(last["d2h_bytes"]), "ms_per_call": round(e2e_s * 1e3, 3),
                "app_run_ms": round(last["time_s"] * 1e3, 3), "call": "B200Evaluator.measure_payloads"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                     "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4) if achieved else None,
                     "traffic": ncu_traffic(f"b2o_k{jac_loop}"), "kernel": f"b2o_k{jac_loop} (Himeno Jacobi nest)",
                     "kernel_us": round(kms * 1e3, 2) if kms else None, "bytes_per_launch": 60 * pts,
                     "peak_source": pk.get("source")},
        "kernels_us": {f"b2o_k{k}": round(v * 1e3, 2) for k, v in rep["kernel_ms"].items()},
        "cpu_baseline": {"value": round(bytes_per_step / cpu_s / 1e9, 3), "unit": "GB/s", "cores": cores,
                         "kind": "port", "sample": f"one full Himeno M app run ({nn} sweeps), C restatement "
                                                   "(oracle/cgen.py), gcc -O3 OpenMP, all-CPU genome",
                         "cpu_model": cpu_model()}
        if cpu_s else None,
        "cpu_baseline_1core": {"value": round(bytes_per_step / cpu1_s / 1e9, 3), "unit": "GB/s", "cores": 1,
                               "kind": "port", "sample": "the same app run, single-threaded (sequential C semantics)",
                               "cpu_model": cpu_model()} if cpu1_s else None,
        "app_speedup_vs_cpu": round(cpu_s / e2e_s, 2) if cpu_s else None,
        "app_speedup_vs_cpu_1core": round(cpu1_s / e2e_s, 2) if cpu1_s else None,
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
    ev.measure_payloads(g["doc"], [pat])
    times, last = [], None
    for _ in range(max(3, args.e2e_steps)):
        t0 = time.perf_counter()
        last = ev.measure_payloads(g["doc"], [pat])[0]
        times.append(time.perf_counter() - t0)
    e2e_s = dist.max(statistics.median(times))
    return {"genome": "100100100", "validity": last["validity"], "e2e_GBps": round(bytes_per_step / e2e_s / 1e9, 3),
            "ms_per_call": round(e2e_s * 1e3, 3), "app_run_ms": round(last["time_s"] * 1e3, 3),
            "h2d_bytes": int(last["h2d_bytes"]), "d2h_bytes": int(last["d2h_bytes"]),
            "note": "gosa summed on the GPU in loop order, bit-identical to the sequential CPU loop (b2o_exact_sum_f32)"}


def ga_arm(args, dist: Dist) -> dict | None:
    """BASELINE config 5: the reference GA (pop 64 x 20 generations) on Himeno
    L, each generation's uncached genomes measured in one batch; under
    torchrun the batch is sharded LPT over the ranks (one B200 each) and the
    results are all-gathered (search.ShardedEvaluator).  patterns/sec =
    evaluations_performed / GA wall time (max over ranks)."""
    try:
        from gpuoffload.ga import GAParams
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
    return {"workload": f"{args.ga_workload} inline nn={sweeps_of(g['doc'])}, pop {args.ga_pop} x {args.ga_gens} gens",
            "patterns_per_s": round(res.evaluations_performed / wall, 3), "evaluations": res.evaluations_performed,
            "cache_hits": res.cache_hits, "wall_s": round(wall, 3), "best_genome": "".join(map(str, res.best_genome)),
            "best_time_s": res.best_time, "measured_by_all_ranks": int(local), "valid_on_rank0": valid,
            "speculated": stats.get("speculated", 0), "speculated_unused": stats.get("speculated_unused", 0),
            "sum_fitness_s_all_ranks": round(fit_sum, 3),
            "programs_executed_all_ranks": int(programs),
            "dedupe": ("genomes whose GPU roots and transfer plan coincide share one program run "
                       "(B200Evaluator.run_key, SURVEY.md §8e)") if args.ga_dedupe else "off",
            "history_evals": [h.evaluations for h in res.history][:6]}


def ops_arm(dist: Dist) -> dict:
    """BASELINE config 3 kernels on resident data: the tcgen05 3xTF32 GEMM
    (cublas_gemm replacement) at 4096^3 and the radix-16 FFT (cufft_exec
    replacement) at 4096^2, CUDA events on the launching stream."""
    import ctypes

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
    import ctypes as ct

    prep, mma = [], []
    for _ in range(10):
        p_ms, m_ms = ct.c_double(), ct.c_double()
        L.b2o_gemm_f32_phases(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, st, ct.byref(p_ms), ct.byref(m_ms))
        prep.append(p_ms.value)
        mma.append(m_ms.value)
    mma_ms = statistics.median(mma)
    prep_ms = statistics.median(prep)
    err = float(np.linalg.norm(c[:256].double().cpu().numpy() - (a[:256].double() @ b.double()).cpu().numpy())
                / np.linalg.norm((a[:256].double() @ b.double()).cpu().numpy()))
    fft_ms = timed(lambda: L.b2o_fft2d_c64(x.data_ptr(), y.data_ptr(), n, st))
    nh = 1 << 26  # 256 MB of int32 (> L2)
    hd = torch.randint(0, 256, (nh,), dtype=torch.int32, device=dev)
    hh = torch.zeros(256, dtype=torch.int32, device=dev)
    hist_ms = timed(lambda: L.b2o_histogram(hd.data_ptr(), nh, hh.data_ptr(), 256, 0, st))
    pk = peaks()
    # dense TF32 ceiling: the nominal 1.1 PFLOP/s (B200_PROFILING.md).  The
    # measured-cuBLAS-bf16 / 2 figure cannot be the ceiling: the MMA kernel
    # alone issues TF32 faster than that (ncu: tensor pipe 89 % of elapsed)
    tf32_peak = max(1100.0, pk["bf16_tflops"] / 2)
    tf32_issued = 3 * 2 * n ** 3 / (gemm_ms * 1e-3) / 1e12
    tf32_kernel = 3 * 2 * n ** 3 / (mma_ms * 1e-3) / 1e12
    fft_gbs = 2 * 2 * 8 * n * n / (fft_ms * 1e-3) / 1e9
    del ctypes
    return {"gemm_4096_ms": round(gemm_ms, 4), "gemm_tflops_fp32_equiv": round(2 * n ** 3 / (gemm_ms * 1e-3) / 1e12, 1),
            "gemm_tf32_tflops_issued": round(tf32_issued, 1),
            "gemm_roofline": {"bound": "tensor", "kernel": "gemm_tc_pair_kernel (cta_group::2, persistent)",
                              "achieved": round(tf32_kernel, 1), "peak": round(tf32_peak, 1),
                              "unit": "TFLOP/s", "frac": round(tf32_kernel / tf32_peak, 3),
                              "kernel_ms": round(mma_ms, 4), "prep_ms": round(prep_ms, 4),
                              "op_frac_incl_prep": round(tf32_issued / tf32_peak, 3),
                              "peak_source": "nominal dense TF32 1.1 PFLOP/s (B200_PROFILING.md); 3 TF32 passes counted"},
            "gemm_normwise_err_rows0_255": err,
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
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--ga", type=int, default=1, help="also measure GA patterns/sec (config 5)")
    ap.add_argument("--ops", type=int, default=1, help="also time the GEMM/FFT/histogram block kernels (config 3)")
    ap.add_argument("--reductions", type=int, default=1, help="also time the opt-in reduction pattern")
    ap.add_argument("--ga-workload", default="himeno_L")
    ap.add_argument("--ga-pop", type=int, default=64)
    ap.add_argument("--ga-gens", type=int, default=20)
    ap.add_argument("--ga-seed", type=int, default=20201106)
    ap.add_argument("--ga-timeout", type=float, default=120.0)
    ap.add_argument("--ga-dedupe", type=int, default=1, help="run identical programs (same GPU roots + plan) once")
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
