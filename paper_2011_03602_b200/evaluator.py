"""B200Evaluator — the drop-in measurement plugin.

Implements the reference's duck-typed evaluator protocol exactly as its
callers use it:

* ``evaluator_id`` / ``concurrency_safe`` / ``needs_code`` attributes
  (``src/evaluators.py:113-115``, read at ``src/ga.py:103`` and
  ``src/blocks.py:616``);
* ``measure(EvaluationRequest) -> MeasurementResult`` (``src/evaluators.py:120``),
  called from ``GenomeEvaluator.evaluate`` (``src/ga.py:125``) and from
  ``_measure_subset`` (``src/blocks.py:630``);
* failures never raise: they come back as ``MeasurementResult(None, validity)``
  with the reference's validity vocabulary (``src/evaluators.py:23-27``),
  honouring the invariant *time iff valid* (``src/evaluators.py:61-62``).

Beyond the protocol, ``measure_batch`` evaluates many patterns at once across
all visible B200s (one worker per device, LPT order by the reference's own
cost model, ``src/evaluators.py:74-109``); results come back in request order.

Each program is serialised once (the reference's ``irdoc.model_to_document``),
compiled once (``compiler.compile_program``, cached by content hash) and
loaded once per device.  A pattern is then just: GPU roots + the transfer plan
+ a timed run of the compiled program.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from . import appspec
from .compiler import CompileError, build_key, compile_program
from .ir import Program, document_digest, document_of
from .runtime import B2OError, NativeApp, Runtime

EVALUATOR_ID = "b200"


@dataclass(frozen=True)
class _LocalMeasurementResult:
    """Stand-in with the reference's fields when gpuoffload is not importable
    (e.g. replaying golden requests on a box without the reference)."""

    time_seconds: float | None
    validity: str
    evaluator_id: str
    diagnostics: str = ""

    @property
    def feasible(self) -> bool:
        return self.validity == "valid"

    def __post_init__(self):
        assert (self.time_seconds is not None) == (self.validity == "valid")


def _result_cls():
    try:
        from gpuoffload.evaluators import MeasurementResult

        return MeasurementResult
    except ImportError:
        return _LocalMeasurementResult


def payload_from_request(request) -> dict:
    """Pattern + plan of an ``EvaluationRequest`` as plain data (what crosses
    the C ABI): ``pattern.gpu_roots`` (src/patterns.py:83-88) and every
    ``TransferDirective`` (src/transfers.py:45-53)."""
    directives = []
    for d in request.transfer_plan.directives:
        directives.append({
            "var": d.var_id,
            "dir": "h2d" if d.direction == "host_to_device" else "d2h",
            "anchor_loop": d.placement.anchor_loop,
            "side": d.placement.side,
            "multiplicity": d.multiplicity,
            "batch": d.batch_id,
        })
    payload = {"genome": request.pattern.genome_text, "gpu_roots": list(request.pattern.gpu_roots),
               "directives": directives}
    try:
        from gpuoffload.evaluators import CostModelParams, cost_model_time

        cm = cost_model_time(request, CostModelParams())
        payload["cost_model_time"] = cm.time_seconds or 0.0
    except ImportError:
        pass
    return payload


def _family(prog: Program, spec: dict) -> str:
    """Programs that differ only by replaced blocks share variables (ids and
    names are preserved by apply_replacements, src/blocks.py:480-563) and
    therefore share reference outputs."""
    sig = [(v.name, v.base_type, v.is_array, v.length) for v in prog.vars]
    return json.dumps([sig, spec.get("inputs"), spec.get("precision")], sort_keys=True)


class B200Evaluator:
    evaluator_id = EVALUATOR_ID
    concurrency_safe = True   # results are merged in request order
    needs_code = False        # the pattern runs from the compiled program, no emission

    def __init__(self, app_spec: dict, devices: list[int] | None = None, mode: str = "coherent",
                 timeout_seconds: float = 300.0, repeats: int = 1, reference_outputs: dict | None = None,
                 cache_dir=None, dedupe: bool = True):
        if mode not in ("coherent", "literal"):
            raise ValueError(f"unknown mode {mode!r}")
        self.spec = dict(app_spec)
        self.mode = mode
        self.timeout_seconds = timeout_seconds
        self.repeats = repeats
        self.cache_dir = cache_dir
        self.user_reference = reference_outputs or {}
        self.runtime = Runtime.get(devices)
        self._apps: dict[str, NativeApp | Exception] = {}
        self._families: dict[str, dict[str, np.ndarray]] = {}
        self._docs: dict[int, tuple[object, dict]] = {}
        self._keys: dict[int, tuple[dict, str]] = {}
        self.log: list[dict] = []
        # program-level dedupe: genomes whose GPU roots and
        # transfer plan coincide run the identical program, so it is executed
        # once and its measurement shared (reported: programs_executed vs
        # dedupe_hits; dedupe=False measures every request)
        self.dedupe = dedupe
        self._runs: dict = {}
        self.programs_executed = 0
        self.dedupe_hits = 0

    @property
    def parallel_width(self) -> int:
        """Patterns measured concurrently (one per B200 worker): the batch
        drivers pad generations to a multiple of this (search.py)."""
        return max(1, int(self.runtime.n_workers))

    # -- program management -------------------------------------------------

    def _doc(self, model) -> dict:
        if isinstance(model, dict):
            return model
        hit = self._docs.get(id(model))
        if hit is not None and hit[0] is model:
            return hit[1]
        doc = document_of(model)
        self._docs[id(model)] = (model, doc)
        return doc

    def _key(self, doc: dict) -> str:
        """build_key (a sha256 over the whole document) memoised per document
        object: the GA and the bench hand the same dict over and over."""
        hit = self._keys.get(id(doc))
        if hit is not None and hit[0] is doc:
            return hit[1]
        key = build_key(doc, self.spec)
        self._keys[id(doc)] = (doc, key)
        return key

    def app_for(self, doc: dict) -> NativeApp:
        """Compile + load (cached). Raises CompileError / B2OError."""
        key = self._key(doc)
        got = self._apps.get(key)
        if isinstance(got, Exception):
            raise got
        if got is not None:
            return got
        try:
            prog = Program(doc)
            compiled = compile_program(doc, self.spec, self.cache_dir)
            initial = appspec.initial_state(prog, self.spec)
            fam = _family(prog, self.spec)
            ref = {}
            for name, arr in self.user_reference.items():
                if name in prog.var_by_name:
                    ref[prog.var_by_name[name].id] = np.asarray(arr, dtype=initial[prog.var_by_name[name].id].dtype)
            if fam in self._families:
                for name, arr in self._families[fam].items():
                    ref.setdefault(prog.var_by_name[name].id, arr)
            app = NativeApp(compiled, initial, ref)
            has_blocks = any(st.kind == "replaced" for st in prog.stmts)
            if fam not in self._families and not has_blocks:
                self._families[fam] = {prog.vars[vid].name: app.reference(vid)
                                       for vid, _, _ in appspec.outputs_of(prog, self.spec)}
        except (CompileError, B2OError, ValueError) as exc:
            self._apps[key] = exc
            raise
        except OSError as exc:  # compiler missing, cache disk full: not cached, may be transient
            raise B2OError(f"I/O failure while building the program: {exc}") from exc
        self._apps[key] = app
        return app

    # -- measurement ------------------------------------------------------------

    def _result(self, validity: str, time_s: float | None, diag: dict | str):
        cls = _result_cls()
        text = diag if isinstance(diag, str) else json.dumps(diag, sort_keys=True)
        return cls(time_s if validity == "valid" else None, validity, EVALUATOR_ID, text)

    def measure_payloads(self, doc: dict, payloads: list[dict]) -> list[dict]:
        """Run raw pattern payloads against one program; returns result dicts
        (the C ABI's b2o_result) in order.  Build failures map to
        compile_error / runtime_error for every payload."""
        try:
            app = self.app_for(doc)
        except CompileError as exc:
            return [{"validity": "compile_error", "time_s": None, "diag": str(exc)[-250:]} for _ in payloads]
        except (B2OError, ValueError) as exc:
            return [{"validity": "runtime_error", "time_s": None, "diag": str(exc)[-250:]} for _ in payloads]
        pats = []
        for p in payloads:
            q = dict(p)
            q.setdefault("mode", self.mode)
            q.setdefault("repeats", self.repeats)
            q.setdefault("timeout_s", self.timeout_seconds)
            q.setdefault("priority", float(p.get("cost_model_time", 0.0) or 0.0))
            pats.append(q)
        try:
            return app.run(pats)
        except B2OError as exc:
            return [{"validity": "runtime_error", "time_s": None, "diag": str(exc)[-250:]} for _ in payloads]

    @staticmethod
    def run_key(doc_key: str, payload: dict) -> str:
        """What the runtime executes for a payload: the program, its GPU
        roots and every directive (the genome text and the cost-model
        priority do not change the run)."""
        dirs = sorted(json.dumps(d, sort_keys=True) for d in payload["directives"])
        return json.dumps([doc_key, sorted(payload["gpu_roots"]), dirs], sort_keys=True)

    def measure_batch(self, requests) -> list:
        groups: dict[str, list[int]] = {}
        docs: dict[str, dict] = {}
        payloads = []
        keys = []
        for i, req in enumerate(requests):
            doc = self._doc(req.model)
            key = document_digest(doc)
            docs[key] = doc
            payloads.append(payload_from_request(req))
            keys.append(self.run_key(key, payloads[i]))
            if self.dedupe and (keys[i] in self._runs or keys[i] in keys[:i]):
                continue  # the identical program is (being) measured already
            groups.setdefault(key, []).append(i)
        out: list = [None] * len(requests)
        for key, idxs in groups.items():
            results = self.measure_payloads(docs[key], [payloads[i] for i in idxs])
            self.programs_executed += len(idxs)
            for i, r in zip(idxs, results):
                r = dict(r)
                r["genome"] = payloads[i]["genome"]
                if self.dedupe:
                    self._runs[keys[i]] = r
                self.log.append(r)
                out[i] = self._result(r["validity"], r.get("time_s"), r)
        for i in range(len(requests)):
            if out[i] is None:
                r = dict(self._runs[keys[i]])
                r["dedupe_of"] = r.pop("genome")
                r["genome"] = payloads[i]["genome"]
                self.dedupe_hits += 1
                out[i] = self._result(r["validity"], r.get("time_s"), r)
        return out

    def measure(self, request):
        return self.measure_batch([request])[0]

    def inject_fault(self, worker: int = 0) -> int:
        """Tests only: the worker's next job traps on the device (a sticky
        CUDA error; see isolated.py for what recovers from it)."""
        from .runtime import lib

        return lib().b2o_debug_inject_fault(int(worker))

    def measure_solo(self, request, repeats: int = 3):
        """One request alone on the worker pool (nothing else in flight),
        best of ``repeats`` runs, bypassing the program-level dedupe cache:
        the contention-free fitness a final selection should rest on when the
        search measured patterns concurrently (``run_search_batched(...,
        confirm_top=k)``; tools/ga_drift.py measures the drift)."""
        doc = self._doc(request.model)
        p = payload_from_request(request)
        p["repeats"] = max(1, int(repeats))
        r = dict(self.measure_payloads(doc, [p])[0])
        r["genome"] = p["genome"]
        r["solo"] = True
        self.log.append(r)
        return self._result(r["validity"], r.get("time_s"), r)

    def close(self) -> None:
        for app in self._apps.values():
            if isinstance(app, NativeApp):
                app.close()
        self._apps.clear()
