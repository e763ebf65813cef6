#!/usr/bin/env python
"""Developer timeline of the CTA-pair kernel k_tcp (ITLUMM_TC_TRACE=1): per-stage globaltimer stamps of
CTAs 0..3 (two pairs) of the last lut_accumulate launch.  Prints, for pair 0, per ring stage the
loader's LUT-half issue (both CTAs), producer warp 0's arrival (both CTAs) and the MMA issue, relative
to the MMA issue, plus the median cadence of each role (ns).  Usage: tcp_trace.py cfg5 [tc|tc_dense]"""
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
algo = sys.argv[2] if len(sys.argv) > 2 else "tc"
cfg = synth.CONFIGS[name]
w = synth.workload(name)
bf16 = cfg["dtype"] == "bf16"
p = fit_layer(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=bf16)
plan = Plan(p, algo="tc")
plan.set_onehot("dense" if algo.endswith("dense") else "auto")
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
KE = 512
buf = np.zeros(16 * 4 * KE, np.uint64)
assert lib.itlumm_dbg_trace_copy(plan._h, buf.ctypes.data_as(ctypes.c_void_p), buf.size) == 0
W = 64
t = buf[:2 * 24 * W].reshape(2, 24, W)[:, :16].astype(np.int64)   # [CTA][slot][stage - 96]
t0 = t[0][t[0] > 0].min()
S = lambda c, slot: np.where(t[c, slot] > 0, t[c, slot] - t0, -1)  # noqa: E731
mw, mi, l0, l1 = S(0, 0), S(0, 1), S(0, 2), S(1, 3)
prod = np.stack([S(0, 4 + p) for p in range(8)])
print(f"{name} {algo} dbg={os.environ.get('ITLUMM_TCP_DBG', '0')}: stages 96..159 of pair 0 (SM cycles of CTA 0, relative to the MMA issue; loader1 is CTA 1's clock, not comparable)")
print("stage  wait_done   issued | loader0 | producers' arrival (CTA 0, roles 0-7)")
for i in range(W):
    if mi[i] < 0:
        continue
    print(f"{96 + i:5d} {mw[i]-mi[i]:8d} {mi[i] - mi[0]:9d} | {l0[i]-mi[i]:7d} | "
          + " ".join(f"{int(prod[w, i]-mi[i]):6d}" for w in range(8)))
d = np.diff(mi[mi >= 0])
print(f"median MMA issue cadence {np.median(d):.0f} cycles; median issue - wait_done {np.median((mi - mw)[mi >= 0]):.0f} cycles")
