"""Exact-sum statistics on Himeno M's real gosa terms (gs after one sweep of
the opt-in reduction pattern): B2O_XSUM_STATS=1 prints the walk counters."""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03602_b200.evaluator import B200Evaluator  # noqa: E402
from paper_2011_03602_b200.ir import Program  # noqa: E402
from paper_2011_03602_b200.runtime import lib  # noqa: E402

root = Path(__file__).resolve().parent.parent
g = json.loads((root / "tests" / "golden" / "himeno_M.json").read_text())
ev = B200Evaluator(g["spec"], devices=[0])
app = ev.app_for(g["doc"])
r = ev.measure_payloads(g["doc"], [g["patterns"]["100100"]])[0]
gs = app.read(Program(g["doc"]).var_by_name["gs"].id, worker=r["worker"]).reshape(129, 129, 257)
x = np.ascontiguousarray(gs[1:-1, 1:-1, 1:-1].reshape(-1))
print("distinct values", len(np.unique(x)), "zeros", int((x == 0).sum()), flush=True)
dx = torch.from_numpy(x).cuda()
out = torch.empty(1, device="cuda")
st = torch.cuda.current_stream().cuda_stream
L = lib()
for _ in range(2):
    L.b2o_exact_sum_f32(dx.data_ptr(), dx.numel(), 0.0, out.data_ptr(), st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    L.b2o_exact_sum_f32(dx.data_ptr(), dx.numel(), 0.0, out.data_ptr(), st)
e1.record()
torch.cuda.synchronize()
want = np.add.accumulate(x, dtype=np.float32)[-1]
print(json.dumps({"us": round(e0.elapsed_time(e1) / 10 * 1e3, 1), "exact": bool(out.cpu().numpy()[0] == want)}))
