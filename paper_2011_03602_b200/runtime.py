"""ctypes binding of ``libb2o.so`` (declared in include/b2o.h).

There is no fallback: if the native library or a GPU is missing, every entry
point raises :class:`B2OError`.  The product path never executes programs on
the CPU in Python.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("B2O_LIB", PKG / "libb2o.so"))

VALIDITY = ("valid", "numeric_mismatch", "compile_error", "runtime_error", "timeout")
MODE = {"coherent": 0, "literal": 1}
DIRECTION = {"host_to_device": 0, "device_to_host": 1, "h2d": 0, "d2h": 1}
SIDE = {"before": 0, "after": 1}


class B2OError(RuntimeError):
    pass


class Directive(ctypes.Structure):
    _fields_ = [("var_id", ctypes.c_int32), ("dir", ctypes.c_int32), ("anchor_loop", ctypes.c_int32),
                ("side", ctypes.c_int32), ("multiplicity", ctypes.c_uint64), ("batch_id", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class Pattern(ctypes.Structure):
    _fields_ = [("gpu_root", ctypes.POINTER(ctypes.c_uint8)), ("n_loops", ctypes.c_int32),
                ("n_directives", ctypes.c_int32), ("directives", ctypes.POINTER(Directive)),
                ("priority", ctypes.c_double), ("timeout_s", ctypes.c_double), ("device", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("repeats", ctypes.c_int32), ("flags", ctypes.c_int32)]


class Result(ctypes.Structure):
    _fields_ = [("time_s", ctypes.c_double), ("validity", ctypes.c_int32), ("worker", ctypes.c_int32),
                ("max_rel_err", ctypes.c_double), ("mismatches", ctypes.c_uint64),
                ("planned_bytes", ctypes.c_uint64), ("elided_bytes", ctypes.c_uint64),
                ("unplanned_bytes", ctypes.c_uint64), ("block_bytes", ctypes.c_uint64),
                ("epilogue_bytes", ctypes.c_uint64), ("directive_execs", ctypes.c_uint64),
                ("launches", ctypes.c_uint64), ("stale_reads", ctypes.c_uint64), ("h2d_bytes", ctypes.c_uint64),
                ("d2h_bytes", ctypes.c_uint64), ("diag", ctypes.c_char * 256)]

    def to_dict(self) -> dict:
        return {
            "time_s": self.time_s if self.validity == 0 else None,
            "validity": VALIDITY[self.validity],
            "worker": self.worker,
            "max_rel_err": self.max_rel_err,
            "mismatches": self.mismatches,
            "planned_bytes": self.planned_bytes,
            "elided_bytes": self.elided_bytes,
            "unplanned_bytes": self.unplanned_bytes,
            "block_bytes": self.block_bytes,
            "epilogue_bytes": self.epilogue_bytes,
            "directive_execs": self.directive_execs,
            "launches": self.launches,
            "stale_reads": self.stale_reads,
            "h2d_bytes": self.h2d_bytes,
            "d2h_bytes": self.d2h_bytes,
            "diag": self.diag.decode(errors="replace"),
        }


_lib = None
_lib_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise B2OError(f"native library {LIB_PATH} is missing: run __graft_entry__.build()")
        L = ctypes.CDLL(str(LIB_PATH))
        u64p = ctypes.POINTER(ctypes.c_uint64)
        sig = {
            "b2o_init": ([ctypes.POINTER(ctypes.c_int32), ctypes.c_int32], ctypes.c_int),
            "b2o_shutdown": ([], ctypes.c_int),
            "b2o_last_error": ([], ctypes.c_char_p),
            "b2o_num_workers": ([], ctypes.c_int),
            "b2o_debug_inject_fault": ([ctypes.c_int32], ctypes.c_int),
            "b2o_worker_recoveries": ([ctypes.c_int32], ctypes.c_int64),
            "b2o_abi_version": ([], ctypes.c_int),
            "b2o_app_create": ([ctypes.c_char_p, ctypes.c_char_p, u64p], ctypes.c_int),
            "b2o_app_load": ([ctypes.c_char_p, ctypes.c_char_p, u64p], ctypes.c_int),
            "b2o_app_num_loops": ([ctypes.c_uint64], ctypes.c_int),
            "b2o_app_var_id": ([ctypes.c_uint64, ctypes.c_char_p], ctypes.c_int),
            "b2o_app_set_initial": ([ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_uint64], ctypes.c_int),
            "b2o_app_set_reference": ([ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_uint64],
                                      ctypes.c_int),
            "b2o_app_finalize": ([ctypes.c_uint64], ctypes.c_int),
            "b2o_app_get_reference": ([ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_uint64],
                                      ctypes.c_int),
            "b2o_app_read": ([ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_uint64],
                             ctypes.c_int),
            "b2o_app_reference_time": ([ctypes.c_uint64], ctypes.c_double),
            "b2o_app_destroy": ([ctypes.c_uint64], ctypes.c_int),
            "b2o_submit": ([ctypes.c_uint64, ctypes.POINTER(Pattern), ctypes.c_int32, u64p], ctypes.c_int),
            "b2o_wait": ([ctypes.c_uint64, ctypes.POINTER(Result), ctypes.c_int32, ctypes.c_double], ctypes.c_int),
            "b2o_gemm_f32": ([ctypes.c_void_p] * 3 + [ctypes.c_int64] * 3 + [ctypes.c_void_p], ctypes.c_int),
            "b2o_fft2d_c64": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p], ctypes.c_int),
            "b2o_gemm_f32_phases": ([ctypes.c_void_p] * 3 + [ctypes.c_int64] * 3 + [ctypes.c_void_p] * 3,
                                    ctypes.c_int),
            "b2o_histogram": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                               ctypes.c_void_p], ctypes.c_int),
            "b2o_gemm_impl": ([], ctypes.c_int),
            "b2o_exact_sum_f32": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_void_p],
                                  ctypes.c_int),
            "b2o_exact_sum_workspace": ([ctypes.c_int64], ctypes.c_size_t),
            "b2o_exact_sum_f64": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p],
                                  ctypes.c_int),
            "b2o_exact_sum_f64_ws": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
            "b2o_exact_sum_f32_ws": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
            "b2o_bench_replay": ([ctypes.c_uint64, ctypes.c_int32, ctypes.POINTER(Pattern), ctypes.c_int32,
                                  ctypes.c_int32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                  ctypes.c_int32, u64p], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().b2o_last_error().decode(errors="replace")
        raise B2OError(f"{what}: {msg}")


class Runtime:
    """Process-wide worker pool (one worker thread + stream per device)."""

    _instance: "Runtime | None" = None
    _ilock = threading.Lock()

    def __init__(self, devices: list[int] | None):
        L = lib()
        if devices:
            arr = (ctypes.c_int32 * len(devices))(*devices)
            check(L.b2o_init(arr, len(devices)), "b2o_init")
        else:
            check(L.b2o_init(None, 0), "b2o_init")
        self.devices = devices
        self.n_workers = L.b2o_num_workers()

    @classmethod
    def get(cls, devices: list[int] | None = None) -> "Runtime":
        with cls._ilock:
            if cls._instance is None:
                cls._instance = Runtime(devices)
            elif devices is not None and list(devices) != cls._current_devices():
                # one worker pool per process: a different device set would
                # silently run on the wrong GPUs
                raise B2OError(f"runtime already initialised on devices {cls._current_devices()}, "
                               f"requested {list(devices)}")
            return cls._instance

    @classmethod
    def _current_devices(cls) -> list[int]:
        inst = cls._instance
        return list(inst.devices) if inst.devices else list(range(inst.n_workers))

    @classmethod
    def shutdown(cls) -> None:
        with cls._ilock:
            if cls._instance is not None:
                lib().b2o_shutdown()
                cls._instance = None


FLAG_INPUTS_RESIDENT = 2  # include/b2o.h B2O_FLAG_INPUTS_RESIDENT


class NativeApp:
    """One compiled program loaded on every worker."""

    def __init__(self, compiled, initial: dict[int, np.ndarray], reference: dict[int, np.ndarray] | None = None):
        self.rt = Runtime.get()
        L = lib()
        h = ctypes.c_uint64()
        check(L.b2o_app_create(str(compiled.host_so).encode(), str(compiled.cubin).encode(), ctypes.byref(h)),
              "b2o_app_create")
        self.handle = h.value
        self.compiled = compiled
        self.n_loops = compiled.n_loops
        self.dtypes = {k: v.dtype for k, v in initial.items()}
        self.sizes = {k: v.shape[0] for k, v in initial.items()}
        for vid, arr in initial.items():
            a = np.ascontiguousarray(arr)
            check(L.b2o_app_set_initial(self.handle, vid, a.ctypes.data, a.nbytes), f"set_initial({vid})")
        for vid, arr in (reference or {}).items():
            a = np.ascontiguousarray(arr)
            check(L.b2o_app_set_reference(self.handle, vid, a.ctypes.data, a.nbytes), f"set_reference({vid})")
        check(L.b2o_app_finalize(self.handle), "b2o_app_finalize")

    @property
    def reference_time(self) -> float:
        return lib().b2o_app_reference_time(self.handle)

    def reference(self, vid: int) -> np.ndarray:
        out = np.empty(self.sizes[vid], dtype=self.dtypes[vid])
        check(lib().b2o_app_get_reference(self.handle, vid, out.ctypes.data, out.nbytes), "get_reference")
        return out

    def read(self, vid: int, worker: int = 0) -> np.ndarray:
        out = np.empty(self.sizes[vid], dtype=self.dtypes[vid])
        check(lib().b2o_app_read(self.handle, worker, vid, out.ctypes.data, out.nbytes), "b2o_app_read")
        return out

    def _patterns(self, patterns: list[dict]):
        n = len(patterns)
        keep = []
        arr = (Pattern * max(n, 1))()
        for i, p in enumerate(patterns):
            roots = (ctypes.c_uint8 * max(self.n_loops, 1))()
            for r in p.get("gpu_roots", ()):
                if not 0 <= r < self.n_loops:
                    raise B2OError(f"gpu root {r} out of range")
                roots[r] = 1
            dirs = p.get("directives", ())
            darr = (Directive * max(len(dirs), 1))()
            for k, d in enumerate(dirs):
                darr[k] = Directive(d["var"], DIRECTION[d["dir"]], d["anchor_loop"], SIDE[d["side"]],
                                    int(d.get("multiplicity", 1)), int(d.get("batch", 0)), 0)
            keep.extend([roots, darr])
            arr[i] = Pattern(ctypes.cast(roots, ctypes.POINTER(ctypes.c_uint8)), self.n_loops, len(dirs),
                             ctypes.cast(darr, ctypes.POINTER(Directive)), float(p.get("priority", 0.0)),
                             float(p.get("timeout_s", 0.0) or 0.0), int(p.get("device", -1)),
                             MODE[p.get("mode", "coherent")], int(p.get("repeats", 1)),
                             FLAG_INPUTS_RESIDENT if p.get("inputs_resident") else 0)
        return arr, keep

    def run(self, patterns: list[dict]) -> list[dict]:
        """Execute pattern dicts {gpu_roots, directives, mode, repeats,
        timeout_s, priority, device}; returns result dicts in order."""
        n = len(patterns)
        arr, _keep = self._patterns(patterns)
        L = lib()
        b = ctypes.c_uint64()
        check(L.b2o_submit(self.handle, arr, n, ctypes.byref(b)), "b2o_submit")
        res = (Result * max(n, 1))()
        check(L.b2o_wait(b.value, res, n, 0.0), "b2o_wait")
        return [res[i].to_dict() for i in range(n)]

    def bench_replay(self, pattern: dict, warmup: int, steps: int, worker: int = 0) -> dict:
        """Device-resident replay of the pattern's kernel launches (see
        b2o_bench_replay in include/b2o.h)."""
        arr, _keep = self._patterns([pattern])
        ms = ctypes.c_double()
        kms = (ctypes.c_double * max(self.n_loops, 1))()
        nl = ctypes.c_uint64()
        check(lib().b2o_bench_replay(self.handle, worker, arr, warmup, steps, ctypes.byref(ms), kms, self.n_loops,
                                     ctypes.byref(nl)), "b2o_bench_replay")
        return {"ms_per_step": ms.value, "kernel_ms": {i: kms[i] for i in range(self.n_loops) if kms[i] > 0},
                "launches_per_step": nl.value}

    def close(self) -> None:
        if self.handle:
            lib().b2o_app_destroy(self.handle)
            self.handle = 0
