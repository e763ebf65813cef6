#!/usr/bin/env python
"""Small parity run for compute-sanitizer: every algo on a few ragged shapes (incl. a streamed LUT),
the encode/accumulate entry points and a 3-layer MLP.  Exits non-zero on any mismatch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from oracle import fit as ofit  # noqa: E402
from paper_2207_05808_b200 import Mlp, Plan  # noqa: E402
from paper_2207_05808_b200._lib import ItlummError  # noqa: E402

bad = 0
for seed, N, D, M, C, dt in [(2, 333, 97, 33, 10, "f32"), (3, 300, 96, 40, 12, "bf16"),
                             (10, 260, 512, 300, 130, "f32"), (5, 130, 784, 512, 32, "f32")]:
    w = synth.small_case(seed, N=N, D=D, M=M, C=C, dtype=dt, n_train=400)
    p = ofit.fit(w["A_train"], w["B"], C, w["perm"], w["bias"], a_is_bf16=dt == "bf16")
    ref = oracle.amm(p, w["A"], relu=True, dtype=dt)["y"]
    A = torch.from_numpy(w["A"].view(np.int16) if dt == "bf16" else w["A"]).cuda()
    if dt == "bf16":
        A = A.view(torch.bfloat16)
    for algo in ("simt", "tc", "tc_pipe"):
        plan = Plan(p, algo=algo)
        try:
            y = plan.amm(A, relu=True).cpu().numpy()
        except ItlummError as e:
            if e.status == 3:
                continue
            raise
        ok = np.array_equal(y.view(np.uint32), ref.view(np.uint32))
        bad += not ok
        print(seed, algo, "ok" if ok else "MISMATCH", flush=True)
        plan.close()
layers = [(96, 64, True), (64, 48, True), (48, 10, False)]
w = synth.mlp_workload(8, 500, n_train=400, layers=layers)
ps = oracle.fit_mlp(w["A_train"], w["Bs"], w["Cs"], w["perms"], w["biases"], w["relus"])
y = Mlp(ps, w["relus"]).forward(torch.from_numpy(w["A"]).cuda()).cpu().numpy()
ok = np.array_equal(y.view(np.uint32), oracle.mlp_forward(ps, w["relus"], w["A"]).view(np.uint32))
bad += not ok
print("mlp", "ok" if ok else "MISMATCH")
sys.exit(1 if bad else 0)
