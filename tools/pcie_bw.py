"""Host<->device copy bandwidth from pinned memory at the sizes the Himeno M
plan moves (15 arrays of 17.1 MB), CUDA events."""

import json

import torch

n = 129 * 129 * 257
bufs = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(15)]
dev = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(15)]
s = torch.cuda.Stream()
for direction in ("h2d", "d2h"):
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            for h, d in zip(bufs, dev):
                if direction == "h2d":
                    d.copy_(h, non_blocking=True)
                else:
                    h.copy_(d, non_blocking=True)
            e1.record()
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"dir": direction, "MB": round(15 * n * 4 / 1e6, 1), "ms": round(ms, 3),
                      "GBps": round(15 * n * 4 / ms / 1e6, 1)}))
