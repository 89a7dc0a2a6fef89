"""Time the exact sequential fp32 sum (b2o_exact_sum_f32) at Himeno M's
interior size on data shaped like the gosa terms, CUDA events."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03602_b200.runtime import lib  # noqa: E402

L = lib()
st = torch.cuda.current_stream().cuda_stream
for name, n, gen in (("uniform", 4_112_895, lambda r, n: r.random(n, dtype=np.float32)),
                     ("squares", 4_112_895, lambda r, n: (r.standard_normal(n, dtype=np.float32) * 1e-3) ** 2),
                     ("mixed_sign", 4_112_895, lambda r, n: r.standard_normal(n, dtype=np.float32)),
                     ("dyadic", 4_112_895, lambda r, n: (r.integers(0, 64, n) * np.float32(2.0 ** -10)).astype(np.float32)),
                     ("constant", 4_112_895, lambda r, n: np.full(n, np.float32(0.1)))):
    x = torch.from_numpy(gen(np.random.default_rng(5), n)).cuda()
    out = torch.empty(1, device="cuda")
    for _ in range(3):
        L.b2o_exact_sum_f32(x.data_ptr(), n, 0.0, out.data_ptr(), st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        L.b2o_exact_sum_f32(x.data_ptr(), n, 0.0, out.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    want = np.add.accumulate(x.cpu().numpy(), dtype=np.float32)[-1]
    print(json.dumps({"data": name, "n": n, "us": round(e0.elapsed_time(e1) / 20 * 1e3, 1),
                      "exact": bool(out.cpu().numpy()[0] == want)}), flush=True)
