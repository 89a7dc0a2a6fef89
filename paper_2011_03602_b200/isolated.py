"""IsolatedEvaluator — the B200 plugin with the runtime in a child process.

A sticky CUDA error (an illegal address or a trap in one pattern's kernel)
kills the CUDA context of the process that raised it: after it every CUDA
call in that process fails, ``cudaDeviceReset`` included (measured on the
B200 box: ``profiles/r02/reset_probe.log`` -- after the reset, context
creation reports "device busy or unavailable").  An in-process runtime can
therefore only report ``runtime_error`` for every later pattern on that
device (``b2o_runtime.cu`` marks the worker broken).  The reference's own
harness is immune because every measurement is a fresh process
(``ExternalCommandEvaluator``, src/evaluators.py:268-293); this wrapper gets the
same isolation without paying a process per pattern:

* the runtime (``B200Evaluator``) lives in one spawned child process that
  measures batch after batch (programs stay compiled and resident);
* when a batch comes back with a lost device (``device lost`` diagnostics:
  the sticky-error path) or the child dies or exceeds the batch deadline (a
  hung kernel cannot be stopped from the host), the child is killed and a
  fresh one started; the pattern that faulted keeps its ``runtime_error`` /
  ``timeout``, the patterns that never ran because the device was gone are
  measured again on the fresh child (once);
* everything else -- plugin attributes, ``measure`` / ``measure_batch`` /
  ``measure_payloads`` / ``measure_solo``, program-level dedupe, results in
  request order -- is ``B200Evaluator``'s (src/evaluators.py:113-120 protocol).

``restarts`` counts replaced children.
"""

from __future__ import annotations

import multiprocessing as mp

from .evaluator import EVALUATOR_ID, B200Evaluator, _result_cls, payload_from_request
from .ir import document_digest, document_of

_LOST = "device lost"


def _serve(conn, spec: dict, kwargs: dict, factory: str) -> None:
    """Child main loop: one B200Evaluator (``factory``, "module:name"; tests
    substitute a double), requests over a pipe."""
    import importlib

    mod, name = factory.split(":")
    ev = getattr(importlib.import_module(mod), name)(spec, **kwargs)
    while True:
        try:
            msg = conn.recv()
        except EOFError:
            return
        op = msg[0]
        try:
            if op == "payloads":
                conn.send(("ok", ev.measure_payloads(msg[1], msg[2])))
            elif op == "width":
                conn.send(("ok", ev.parallel_width))
            elif op == "inject":  # tests: the worker's next job traps on the device
                conn.send(("ok", ev.inject_fault(int(msg[1]))))
            elif op == "stop":
                conn.send(("ok", None))
                return
            else:
                conn.send(("err", f"unknown request {op!r}"))
        except Exception as exc:  # never leave the parent waiting
            conn.send(("err", f"{type(exc).__name__}: {exc}"))


class IsolatedEvaluator:
    evaluator_id = EVALUATOR_ID
    concurrency_safe = True
    needs_code = False
    run_key = staticmethod(B200Evaluator.run_key)

    def __init__(self, app_spec: dict, devices: list[int] | None = None, mode: str = "coherent",
                 timeout_seconds: float = 300.0, repeats: int = 1, reference_outputs: dict | None = None,
                 dedupe: bool = True, start_timeout: float = 600.0,
                 factory: str = "paper_2011_03602_b200.evaluator:B200Evaluator"):
        self.spec = dict(app_spec)
        self.timeout_seconds = timeout_seconds
        self.repeats = repeats
        self.start_timeout = start_timeout
        self._kwargs = {"devices": devices, "mode": mode, "timeout_seconds": timeout_seconds, "repeats": repeats,
                        "reference_outputs": reference_outputs, "dedupe": False}
        self._factory = factory
        self._ctx = mp.get_context("spawn")  # a forked child would inherit the parent's CUDA state
        self._proc = None
        self._conn = None
        self.restarts = 0
        self.dedupe = dedupe
        self._runs: dict = {}
        self.programs_executed = 0
        self.dedupe_hits = 0
        self.log: list[dict] = []
        self._width = None

    # -- child management ---------------------------------------------------------

    def _start(self) -> None:
        parent, child = self._ctx.Pipe()
        self._proc = self._ctx.Process(target=_serve, args=(child, self.spec, self._kwargs, self._factory),
                                      daemon=True)
        self._proc.start()
        child.close()
        self._conn = parent

    def _kill(self) -> None:
        if self._proc is not None:
            self._proc.kill()
            self._proc.join(10)
        if self._conn is not None:
            self._conn.close()
        self._proc = self._conn = None

    def _call(self, msg, deadline_s: float):
        """(status, value); status "dead" when the child died or missed the
        deadline (it is killed then)."""
        if self._proc is None:
            self._start()
        try:
            self._conn.send(msg)
            if not self._conn.poll(deadline_s):
                self._kill()
                return "dead", "deadline exceeded"
            return self._conn.recv()
        except (EOFError, BrokenPipeError, ConnectionResetError, OSError) as exc:
            self._kill()
            return "dead", f"runtime process died: {exc}"

    def restart(self) -> None:
        self._kill()
        self.restarts += 1
        self._start()

    def close(self) -> None:
        if self._proc is not None and self._proc.is_alive():
            try:
                self._conn.send(("stop",))
                self._conn.poll(30)
            except (BrokenPipeError, OSError):
                pass
        self._kill()

    def __del__(self):
        try:
            self._kill()
        except Exception:
            pass

    # -- measurement --------------------------------------------------------------------

    @property
    def parallel_width(self) -> int:
        if self._width is None:
            st, v = self._call(("width",), self.start_timeout)
            self._width = int(v) if st == "ok" else 1
        return self._width

    def inject_fault(self, worker: int = 0) -> None:
        """Tests: make the child's worker trap on its next job."""
        self._call(("inject", worker), self.start_timeout)

    def _deadline(self, payloads: list[dict]) -> float:
        per = sum(max(1, int(p.get("repeats", self.repeats))) * float(p.get("timeout_s", self.timeout_seconds))
                  for p in payloads)
        return self.start_timeout + per

    def measure_payloads(self, doc: dict, payloads: list[dict]) -> list[dict]:
        st, res = self._call(("payloads", doc, payloads), self._deadline(payloads))
        if st == "err":
            return [{"validity": "runtime_error", "time_s": None, "diag": str(res)[-250:]} for _ in payloads]
        if st == "dead":
            # nothing came back: which pattern hung or crashed is unknown, so
            # each is measured alone on a fresh child; the culprit keeps
            # timing out or crashing (and is reported so), the others succeed
            self.restarts += 1
            if len(payloads) == 1:
                v = "timeout" if res == "deadline exceeded" else "runtime_error"
                return [{"validity": v, "time_s": None, "diag": f"{res} (runtime restarted)"}]
            return [self.measure_payloads(doc, [p])[0] for p in payloads]
        lost = [i for i, r in enumerate(res) if r.get("validity") != "valid" and _LOST in str(r.get("diag", ""))]
        if lost:
            # the context is dead: replace the child; the jobs the dead
            # device refused are measured again on the fresh one (the job
            # that faulted ran and keeps its result)
            self.restart()
            again = [i for i in lost if str(res[i].get("diag", "")).startswith(_LOST)]
            if again:
                st2, res2 = self._call(("payloads", doc, [payloads[i] for i in again]),
                                       self._deadline([payloads[i] for i in again]))
                if st2 == "ok":
                    for i, r in zip(again, res2):
                        res[i] = r
        return res

    def _result(self, r: dict):
        import json

        cls = _result_cls()
        v = r["validity"]
        return cls(r.get("time_s") if v == "valid" else None, v, EVALUATOR_ID, json.dumps(r, sort_keys=True,
                                                                                         default=str))

    def measure_batch(self, requests) -> list:
        groups: dict[str, list[int]] = {}
        docs: dict[str, dict] = {}
        payloads, keys = [], []
        for i, req in enumerate(requests):
            doc = document_of(req.model) if not isinstance(req.model, dict) else req.model
            dk = document_digest(doc)
            docs[dk] = doc
            payloads.append(payload_from_request(req))
            keys.append(B200Evaluator.run_key(dk, payloads[i]))
            if self.dedupe and (keys[i] in self._runs or keys[i] in keys[:i]):
                continue
            groups.setdefault(dk, []).append(i)
        out: list = [None] * len(requests)
        for dk, idxs in groups.items():
            results = self.measure_payloads(docs[dk], [payloads[i] for i in idxs])
            self.programs_executed += len(idxs)
            for i, r in zip(idxs, results):
                r = dict(r)
                r["genome"] = payloads[i]["genome"]
                if self.dedupe:
                    self._runs[keys[i]] = r
                self.log.append(r)
                out[i] = self._result(r)
        for i in range(len(requests)):
            if out[i] is None:
                r = dict(self._runs[keys[i]])
                r["dedupe_of"] = r.pop("genome")
                r["genome"] = payloads[i]["genome"]
                self.dedupe_hits += 1
                out[i] = self._result(r)
        return out

    def measure(self, request):
        return self.measure_batch([request])[0]

    def measure_solo(self, request, repeats: int = 3):
        doc = document_of(request.model) if not isinstance(request.model, dict) else request.model
        p = payload_from_request(request)
        p["repeats"] = max(1, int(repeats))
        r = dict(self.measure_payloads(doc, [p])[0])
        r["genome"] = p["genome"]
        r["solo"] = True
        self.log.append(r)
        return self._result(r)
