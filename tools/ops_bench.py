"""Time the block kernels (GEMM 4096^3, FFT 4096^2) with CUDA events on the
launching stream; prints one JSON line per op."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2011_03602_b200.runtime import lib  # noqa: E402


def timed(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


L = lib()
L.b2o_histogram.argtypes  # bound in runtime.lib()
st = torch.cuda.current_stream().cuda_stream
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
a = torch.rand(n, n, device="cuda")
b = torch.rand(n, n, device="cuda")
c = torch.empty(n, n, device="cuda")
ms = timed(lambda: L.b2o_gemm_f32(a.data_ptr(), b.data_ptr(), c.data_ptr(), n, n, n, st))
print(json.dumps({"op": "gemm_3xtf32", "n": n, "ms": round(ms, 4), "tflops_fp32_equiv": round(2 * n**3 / ms / 1e9, 1),
                  "tflops_tf32_issued": round(3 * 2 * n**3 / ms / 1e9, 1)}))
ms_tf = timed(lambda: torch.matmul(a, b))
torch.backends.cuda.matmul.allow_tf32 = True
ms_tf32 = timed(lambda: torch.matmul(a, b))
print(json.dumps({"op": "cublas_fp32_sgemm", "ms": round(ms_tf, 4), "tflops": round(2 * n**3 / ms_tf / 1e9, 1),
                  "cublas_tf32_ms": round(ms_tf32, 4), "cublas_tf32_tflops": round(2 * n**3 / ms_tf32 / 1e9, 1)}))
x = torch.rand(2 * n * n, device="cuda")
y = torch.empty_like(x)
ms = timed(lambda: L.b2o_fft2d_c64(x.data_ptr(), y.data_ptr(), n, st))
bytes_ = 2 * 2 * 8 * n * n
print(json.dumps({"op": "fft2d", "n": n, "ms": round(ms, 4), "gbs_two_pass": round(bytes_ / ms / 1e6, 1)}))
xc = torch.view_as_complex(x.view(n, n, 2))
ms_cufft = timed(lambda: torch.fft.fft2(xc))
print(json.dumps({"op": "cufft_c2c_2d", "ms": round(ms_cufft, 4)}))
nh = 1 << 26  # 64M int32 = 256 MB > L2
d = torch.randint(0, 256, (nh,), dtype=torch.int32, device="cuda")
h = torch.zeros(256, dtype=torch.int32, device="cuda")
ms = timed(lambda: L.b2o_histogram(d.data_ptr(), nh, h.data_ptr(), 256, 0, st))
print(json.dumps({"op": "histogram", "n": nh, "bins": 256, "ms": round(ms, 4), "gbs": round(4 * nh / ms / 1e6, 1)}))
ms_t = timed(lambda: torch.bincount(d, minlength=256))
print(json.dumps({"op": "torch_bincount", "ms": round(ms_t, 4)}))
