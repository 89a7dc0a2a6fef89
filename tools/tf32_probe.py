"""Probe what tcgen05.mma kind::tf32 does with the low 13 mantissa bits of
fp32 operands (truncate or round), through the GEMM entry point with the
split disabled (B2O_GEMM_SPLIT=1: hi = raw fp32, lo = 0) and B = identity,
so C = tf32_hw(A) exactly.  Prints which rule matches."""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("B2O_GEMM_SPLIT", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2011_03602_b200.runtime import lib  # noqa: E402

n = 256
rng = np.random.default_rng(0)
a = (rng.random((n, n)) * 2 - 1).astype(np.float32)
b = np.eye(n, dtype=np.float32)
da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
dc = torch.empty(n, n, device="cuda")
assert lib().b2o_gemm_f32(da.data_ptr(), db.data_ptr(), dc.data_ptr(), n, n, n, 0) == 0
torch.cuda.synchronize()
c = dc.cpu().numpy()
bits = a.view(np.uint32)
trunc = (bits & np.uint32(0xFFFFE000)).view(np.float32)
# round to nearest, ties away (cvt.rna): add half ulp of tf32 then truncate
rna = ((bits + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)
print(json.dumps({"matches_truncation": float(np.mean(c == trunc)), "matches_rna": float(np.mean(c == rna)),
                  "matches_raw_fp32": float(np.mean(c == a))}))
