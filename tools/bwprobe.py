#!/usr/bin/env python
"""HBM probe: achievable read-only, write-only and copy bandwidth with torch kernels (context for
the roofline denominators; MEASURED_PEAKS.json's hbm_gbs is a copy)."""
import json
import torch


def t(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e-3


res = {}
for mb in (188, 1024):
    n = mb * 2**20 // 4
    x = torch.randn(n, device="cuda")
    y = torch.empty_like(x)
    s = torch.empty((), device="cuda")
    res[f"read_{mb}MB_GBps"] = n * 4 / t(lambda: torch.sum(x)) / 1e9
    res[f"write_{mb}MB_GBps"] = n * 4 / t(lambda: y.fill_(1.0)) / 1e9
    res[f"copy_{mb}MB_GBps"] = 2 * n * 4 / t(lambda: y.copy_(x)) / 1e9
print(json.dumps(res))
