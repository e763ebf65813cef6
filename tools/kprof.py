#!/usr/bin/env python
"""Developer: per-kernel device time of a whole-MLP forward (cfg4_c*) or a single-layer amm (cfg*)
from the CUDA activity trace (torch.profiler / CUPTI; kernels not serialised, caches not flushed).

    python tools/kprof.py cfg4_c256 [--root DIR] [--iters 3]

--root imports the package (and synth) from another checkout (e.g. an archived older build)."""
import argparse
import collections
import json
import os
import sys

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--root", default=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--rows", type=int, default=None)
args = ap.parse_args()
sys.path.insert(0, os.path.abspath(args.root))

import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import synth  # noqa: E402
import paper_2207_05808_b200 as pkg  # noqa: E402

dev = torch.device("cuda", 0)
if args.workload.startswith("cfg4_c"):
    C = int(args.workload.split("_c")[1])
    n = args.rows or synth.MLP_CFG["N"]
    w = synth.mlp_workload(C, 0)
    params = pkg.fit_mlp(w["A_train"], w["Bs"], w["Cs"], w["perms"], w["biases"], w["relus"], device=0)
    mlp = pkg.Mlp(params, w["relus"], device=0)
    rng = np.random.default_rng(0)
    A = torch.from_numpy(rng.standard_normal((n, synth.MLP_LAYERS[0][0]), dtype=np.float32)).to(dev)
    out = torch.empty((n, synth.MLP_LAYERS[-1][1]), device=dev)

    def call():
        mlp.forward(A, out=out)
else:
    cfg = synth.CONFIGS[args.workload]
    n = args.rows or cfg["N"]
    w = synth.workload(args.workload, n_rows=n)
    bf16 = cfg["dtype"] == "bf16"
    plan = pkg.Plan(pkg.fit_layer(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=bf16))
    A = torch.from_numpy(w["A"].view(np.int16) if bf16 else w["A"]).to(dev)
    if bf16:
        A = A.view(torch.bfloat16)
    out = torch.empty((n, cfg["M"]), device=dev)

    def call():
        plan.amm(A, out=out, relu=cfg["relu"])

for _ in range(2):
    call()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(args.iters):
        call()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
per = len(evs) // args.iters
last = evs[-per:]
seq = [(e.name[:48], round(e.time_range.end - e.time_range.start, 1)) for e in last]
span = last[-1].time_range.end - last[0].time_range.start
print(json.dumps({"workload": args.workload, "root": args.root, "launches_per_call": per,
                  "span_us": round(span, 1), "sequence": seq}))
