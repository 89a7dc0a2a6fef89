"""Test double for IsolatedEvaluator's child (tests/test_isolated.py): behaves
like B200Evaluator after a sticky CUDA error -- the faulting job returns
runtime_error, every later job in the same process "device lost" -- and can
crash or hang its process on request (genome "crash" / "hang")."""

import os
import time


class FakeB200:
    def __init__(self, spec, **kwargs):
        self.spec = spec
        self.parallel_width = 1
        self.armed = False
        self.dead = False
        self.pid = os.getpid()

    def inject_fault(self, worker):
        self.armed = True
        return 0

    def measure_payloads(self, doc, payloads):
        out = []
        for p in payloads:
            g = p.get("genome", "")
            if g == "crash":
                os._exit(3)
            if g == "hang":
                time.sleep(3600)
            if self.dead:
                out.append({"validity": "runtime_error", "time_s": None,
                            "diag": "device lost: device reset after a sticky error failed: stream re-creation failed"})
            elif self.armed:
                self.armed, self.dead = False, True
                out.append({"validity": "runtime_error", "time_s": None, "diag": "stream sync: unspecified launch failure"})
            else:
                out.append({"validity": "valid", "time_s": 0.001, "diag": "", "pid": self.pid})
        return out
