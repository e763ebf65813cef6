#!/usr/bin/env python
"""Developer: SM clock / power / throttle reasons while the cfg5 accumulate (or the fused call) runs
back to back for a few seconds (nvidia-smi sampled every 50 ms), and the per-call time meanwhile."""
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2207_05808_b200 import Plan, fit_layer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
what = sys.argv[2] if len(sys.argv) > 2 else "acc"
cfg = synth.CONFIGS[name]
w = synth.workload(name)
bf16 = cfg["dtype"] == "bf16"
p = fit_layer(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=bf16)
plan = Plan(p)
A = torch.from_numpy(w["A"].view(np.int16) if bf16 else w["A"]).cuda()
if bf16:
    A = A.view(torch.bfloat16)
codes = plan.encode(A)
out = torch.empty((cfg["N"], cfg["M"]), device="cuda")
fn = (lambda: plan.lut_accumulate(codes, out=out, relu=cfg["relu"])) if what == "acc" else (lambda: plan.amm(A, out=out, relu=cfg["relu"]))
for _ in range(5):
    fn()
torch.cuda.synchronize()
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(50):
            fn()
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "50"],
                       stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
reps = 0
a.record()
while time.time() - t0 < 3.0:
    g.replay()
    reps += 1
    if reps % 4 == 0:
        torch.cuda.synchronize()
b.record()
torch.cuda.synchronize()
smi.terminate()
lines = smi.communicate()[0].strip().splitlines()
ms = a.elapsed_time(b) / (reps * 50)
clk = [float(x.split(",")[0]) for x in lines if x.strip()]
pw = [float(x.split(",")[1]) for x in lines if x.strip()]
rs = sorted({x.split(",")[2].strip() for x in lines if x.strip()})
print(f"{name} {what}: {ms:.3f} ms per call over {reps * 50} calls; SM MHz median {np.median(clk):.0f} min {min(clk):.0f} max {max(clk):.0f}; "
      f"power W median {np.median(pw):.0f} max {max(pw):.0f}; reasons {rs}; samples {len(clk)}")
