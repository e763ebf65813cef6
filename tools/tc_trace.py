#!/usr/bin/env python
"""Developer timeline of the TC kernel (ITLUMM_TC_TRACE=1): per-role event stamps of CTAs 0..7 of
the last launch.  Prints per-tile MMA start / epilogue start-end and K-block cadence (ns)."""
import ctypes
import json
import os
import sys

os.environ["ITLUMM_TC_TRACE"] = "1"
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2207_05808_b200 import Plan, fit_layer, _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
mode = sys.argv[2] if len(sys.argv) > 2 else "acc"      # acc: lut_accumulate; sp: fused TC_SP amm
if name.startswith("shape:"):                           # shape:N,D,M,C (synthetic small_case)
    N_, D_, M_, C_ = (int(x) for x in name[6:].split(","))
    w = synth.small_case(77, N=N_, D=D_, M=M_, C=C_, n_train=2000)
    cfg = dict(N=N_, M=M_, relu=True, dtype="f32")
else:
    cfg = synth.CONFIGS[name]
    w = synth.workload(name, n_rows=cfg["N"])
bf16 = cfg["dtype"] == "bf16"
p = fit_layer(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=bf16)
if mode == "fusedpk":                                    # fused TC on split-packed rows
    from paper_2207_05808_b200 import split_packed
    p, cols = split_packed(p)
    w["A"] = np.ascontiguousarray(w["A"][:, cols])
plan = Plan(p, algo="tc" if mode in ("acc", "fusedpk") else "tc_pipe")
A = torch.from_numpy(w["A"].view(np.int16) if bf16 else w["A"]).cuda()
if bf16:
    A = A.view(torch.bfloat16)
codes = plan.encode(A)
out = torch.empty((cfg["N"], cfg["M"]), device="cuda")
for _ in range(5):
    if mode == "acc":
        plan.lut_accumulate(codes, out=out, relu=cfg["relu"])
    else:
        plan.amm(A, out=out, relu=cfg["relu"])
torch.cuda.synchronize()
lib = _lib.load()
lib.itlumm_dbg_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
KE = 512
buf = np.zeros(16 * 4 * KE, np.uint64)
assert lib.itlumm_dbg_trace_copy(plan._h, buf.ctypes.data_as(ctypes.c_void_p), buf.size) == 0
t = buf.reshape(16, 4, KE).astype(np.int64)
t0 = t[t > 0].min()
res = {}
for cta in range(4):
    ev = {}
    for role, nm in enumerate(["producer_kb", "mma", "epi", "loader"]):
        x = t[cta, role]
        x = x[x > 0] - t0
        ev[nm] = x.tolist()
    res[cta] = ev
    pk, mm, ep, ld = (np.array(ev[k]) for k in ("producer_kb", "mma", "epi", "loader"))
    print(f"CTA {cta}: producer K-blocks {len(pk)}, mma events {len(mm)}, epi events {len(ep)}, loads {len(ld)}")
    print("  loader   ", ld[:10].tolist())
    print("  producer ", pk[:24].tolist())
    print("  mma      ", mm[:30].tolist())
    print("  epi s/e  ", ep.tolist())
    print("  end      ", max(pk.max(initial=0), mm.max(initial=0), ep.max(initial=0)))
if len(sys.argv) > 3 and sys.argv[3] == "cadence":
    # streamed LUT: per K-block, loader B-issue (role 3, after the item's codes stamp), producer
    # arrive (role 0) and MMA issue (role 1, after the item stamp) of CTA 0
    x = lambda r: (t[0, r][t[0, r] > 0] - t0)
    ld, pk, mm = x(3), x(0), x(1)
    print("loader stamps (codes+B):", np.diff(ld[:40]).tolist())
    print("producer K-block deltas:", np.diff(pk[:40]).tolist())
    print("mma stamp deltas:       ", np.diff(mm[:40]).tolist())
    n = min(len(pk), 300)
    print("median producer cadence (ns):", float(np.median(np.diff(pk[50:n]))))
    print("median mma cadence (ns):", float(np.median(np.diff(mm[50:min(len(mm), 300)]))))
for cta in range(8, 10):
    pi, cd, pu = (t[cta, r][t[cta, r] > 0] - t0 for r in range(3))
    print(f"encoder CTA {cta - 8}: issues {len(pi)}, consumed {len(cd)}, published {len(pu)}")
    print("  issue    ", pi[:24].tolist())
    print("  consumed ", cd[:24].tolist())
    print("  publish  ", pu[:24].tolist())
json.dump(res, open(os.path.join("gpurun_out", f"tc_trace_{name.replace(':', '_').replace(',', '_')}_{mode}.json"), "w"))
