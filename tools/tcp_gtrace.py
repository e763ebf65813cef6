#!/usr/bin/env python
"""Developer: which arrival completes the CTA-pair kernel's full barrier last?  %globaltimer stamps
(ns, comparable across SMs) of pair 0: the leader MMA warp's full-wait completion vs each CTA's
producer warps 0/7 arrival and LUT-loader issue, per ring slot (ITLUMM_TC_TRACE=1)."""
import ctypes
import os
import sys

os.environ["ITLUMM_TC_TRACE"] = "1"
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2207_05808_b200 import Plan, fit_layer, _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cfg = synth.CONFIGS[name]
w = synth.workload(name)
bf16 = cfg["dtype"] == "bf16"
p = fit_layer(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=bf16)
plan = Plan(p, algo="tc")
plan.set_onehot("dense")
A = torch.from_numpy(w["A"].view(np.int16) if bf16 else w["A"]).cuda()
if bf16:
    A = A.view(torch.bfloat16)
codes = plan.encode(A)
out = torch.empty((cfg["N"], cfg["M"]), device="cuda")
for _ in range(3):
    plan.lut_accumulate(codes, out=out, relu=cfg["relu"])
torch.cuda.synchronize()
lib = _lib.load()
lib.itlumm_dbg_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
buf = np.zeros(16 * 4 * 512 + 2048, np.uint64)
assert lib.itlumm_dbg_trace_copy(plan._h, buf.ctypes.data_as(ctypes.c_void_p), buf.size) == 0
W, S = 64, 24
t = buf[:2 * S * W].reshape(2, S, W).astype(np.int64)
mw = t[0, 16]
ok = mw > 0
print(f"{name}: per slot, ns relative to the leader's full-wait completion (negative = earlier)")
print(" slot  dt_mma | p0_cta0 p7_cta0 ld_cta0 | p0_cta1 p7_cta1 ld_cta1")
rows = []
for i in range(W):
    if not ok[i]:
        continue
    r = [t[0, 17, i], t[0, 19, i], t[0, 18, i], t[1, 17, i], t[1, 19, i], t[1, 18, i]]
    r = [x - mw[i] if x > 0 else 0 for x in r]
    rows.append(r)
    print(f"{96 + i:5d} {mw[i] - mw[ok][0]:7d} | " + " ".join(f"{x:7d}" for x in r))
rows = np.array(rows)
print("median:", " ".join(f"{x:.0f}" for x in np.median(rows, axis=0)), "| cadence", np.median(np.diff(mw[ok])))
