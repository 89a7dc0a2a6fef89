"""Time the 4096^2 FFT (cufft_exec replacement) under the current B2O_FFT_*
environment and check it against torch.fft.fft2 (norm-wise)."""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2011_03602_b200.runtime import lib  # noqa: E402

L = lib()
st = torch.cuda.current_stream().cuda_stream
n = 4096
x = torch.rand(2 * n * n, device="cuda") * 2 - 1
y = torch.empty_like(x)
for _ in range(3):
    assert L.b2o_fft2d_c64(x.data_ptr(), y.data_ptr(), n, st) == 0
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
s.record()
for _ in range(20):
    L.b2o_fft2d_c64(x.data_ptr(), y.data_ptr(), n, st)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
ref = torch.fft.fft2(torch.view_as_complex(x.view(n, n, 2)).to(torch.complex128))
got = torch.view_as_complex(y.view(n, n, 2)).to(torch.complex128)
err = float((got - ref).abs().norm() / ref.abs().norm())
env = {k: v for k, v in os.environ.items() if k.startswith("B2O_FFT")}
print(json.dumps({"env": env, "ms": round(ms, 4), "gbs_two_pass": round(4 * 8 * n * n / ms / 1e6, 1),
                  "normwise_err": err}), flush=True)
