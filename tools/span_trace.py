#!/usr/bin/env python
"""Developer: per-CTA start/end spans of the encoder and TC kernels of one itlumm_amm (TC_PIPE)
call (ITLUMM_TC_TRACE=1), relative to the first encoder CTA start (us)."""
import ctypes
import os
import sys

os.environ["ITLUMM_TC_TRACE"] = "1"
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2207_05808_b200 import Plan, fit_layer, _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
packed = name.endswith("_packed")
base = name[:-7] if packed else name
cfg = synth.CONFIGS[base]
w = synth.workload(base, n_rows=cfg["N"])
bf16 = cfg["dtype"] == "bf16"
p = fit_layer(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=bf16)
if packed:
    from paper_2207_05808_b200 import split_packed
    p, cols = split_packed(p)
    w["A"] = np.ascontiguousarray(w["A"][:, cols])
plan = Plan(p, algo="tc_pipe")
A = torch.from_numpy(w["A"].view(np.int16) if bf16 else w["A"]).cuda()
if bf16:
    A = A.view(torch.bfloat16)
out = torch.empty((cfg["N"], cfg["M"]), device="cuda")
for _ in range(6):
    plan.amm(A, out=out, relu=cfg["relu"])
torch.cuda.synchronize()
lib = _lib.load()
lib.itlumm_dbg_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
n = 16 * 4 * 512 + 4 * 512
buf = np.zeros(n, np.uint64)
assert lib.itlumm_dbg_trace_copy(plan._h, buf.ctypes.data_as(ctypes.c_void_p), n) == 0
sp = buf[16 * 4 * 512:].astype(np.int64).reshape(2, 512, 2)
enc, tc = sp[0], sp[1]
enc = enc[enc[:, 0] > 0]
tc = tc[tc[:, 0] > 0]
t0 = enc[:, 0].min()
f = lambda x: np.round((x - t0) / 1000.0, 2)  # noqa: E731
print(f"encoder CTAs {len(enc)}: start {f(enc[:, 0].min())}..{f(enc[:, 0].max())} us, end {f(enc[:, 1].min())}..{f(enc[:, 1].max())} us")
print(f"TC CTAs {len(tc)}: start {f(tc[:, 0].min())}..{f(tc[:, 0].max())} us, end {f(tc[:, 1].min())}..{f(tc[:, 1].max())} us")
print("encoder end percentiles (us):", f(np.percentile(enc[:, 1], [0, 10, 50, 90, 100])))
print("TC start percentiles (us):", f(np.percentile(tc[:, 0], [0, 10, 50, 90, 100])))
print("TC end percentiles (us):", f(np.percentile(tc[:, 1], [0, 10, 50, 90, 100])))
if len(sys.argv) > 2 and sys.argv[2] == "detail":
    # per TC CTA: start, end, duration; CTAs with a leftover column part (static schedule:
    # worker = cta // G < rem * parts) vs without
    tcs = sp[1]
    idx = np.nonzero(tcs[:, 0] > 0)[0]
    G = int(os.environ.get("TC_G", "2"))
    ntiles = (cfg["N"] + 127) // 128
    ngroups = len(idx) // G
    full, rem = ntiles // ngroups, ntiles % ngroups
    parts = max(1, min(cfg["M"] // G // 32, ngroups // rem)) if rem else 1
    lead = (idx // G) < rem * parts
    st, en = tcs[idx, 0], tcs[idx, 1]
    print(f"G={G} ngroups={ngroups} full={full} rem={rem} parts={parts}")
    for nm, m in (("with part", lead), ("without", ~lead)):
        print(f"  {nm:10s}: n={m.sum():3d} start {f(st[m].mean())} end {f(en[m].mean())} (max {f(en[m].max())}) "
              f"dur {np.round((en[m] - st[m]).mean() / 1000.0, 2)} us")
    order = np.argsort(en)
    print("  latest 10 CTAs (cta, start, end):", [(int(idx[i]), float(f(st[i])), float(f(en[i]))) for i in order[-10:]])
    print("  corr(start, end):", float(np.corrcoef(st, en)[0, 1]))
