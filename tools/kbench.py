#!/usr/bin/env python
"""Per-kernel timing probe (CUDA events): encode, lut_accumulate, fused amm for one workload and
algo.  Diagnostic only (bench.py is the contract); prints one JSON dict per line."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2207_05808_b200 import Plan, fit_layer  # noqa: E402


GRAPH = True


def timeit(fn, iters, warm=5):
    """Mean device time per call: the calls are captured into one CUDA graph and replayed, so
    host-side (ctypes/Python) overhead does not leak into the number."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if GRAPH:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(iters):
                    fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a.record()
        g.replay()
        b.record()
    else:
        a.record()
        for _ in range(iters):
            fn()
        b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--algos", default="simt,tc")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--only", default="encode,acc,fused")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--summation", default="exact")
    ap.add_argument("--packed", action="store_true", help="split-packed input (the layer re-parameterised)")
    args = ap.parse_args()
    global GRAPH
    GRAPH = not args.no_graph
    if args.workload.startswith("shape:"):          # shape:N,D,M,C (synthetic small_case, f32, ReLU)
        N_, D_, M_, C_ = (int(x) for x in args.workload[6:].split(","))
        cfg = dict(N=N_, M=M_, C=C_, relu=True, dtype="f32")
        n = N_
        bf16 = False
        w = synth.small_case(77, N=N_, D=D_, M=M_, C=C_, n_train=2000)
    else:
        cfg = synth.CONFIGS[args.workload]
        n = cfg["N"] if args.rows is None else args.rows
        bf16 = cfg["dtype"] == "bf16"
        w = synth.workload(args.workload, n_rows=n)
    params = fit_layer(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=bf16)
    if args.packed:
        from paper_2207_05808_b200 import split_packed
        params, cols = split_packed(params)
        w["A"] = np.ascontiguousarray(w["A"][:, cols])
    plan = Plan(params)
    if args.summation != "exact":
        plan.set_summation(args.summation)
    A = torch.from_numpy(w["A"].view(np.int16) if bf16 else w["A"]).cuda()
    if bf16:
        A = A.view(torch.bfloat16)
    out = torch.empty((n, cfg["M"]), device="cuda")
    codes = plan.encode(A)
    s_a = 2 if bf16 else 4
    res = {"workload": args.workload, "rows": n}
    only = args.only.split(",")
    if "encode" in only:
        res["encode_ms"] = timeit(lambda: plan.encode(A, codes=codes), args.iters)
    for algo in args.algos.split(","):
        try:
            base, onehot = algo, "auto"
            for suffix, oh in (("_sp24", "sparse24"), ("_dense", "dense")):
                if algo.endswith(suffix):
                    base, onehot = algo[: -len(suffix)], oh
            plan.set_algo(base)
            plan.set_onehot(onehot)
            if "acc" in only:
                res[f"{algo}_accumulate_ms"] = timeit(lambda: plan.lut_accumulate(codes, out=out, relu=cfg["relu"]), args.iters)
            if "fused" not in only:
                continue
            res[f"{algo}_fused_ms"] = timeit(lambda: plan.amm(A, out=out, relu=cfg["relu"]), args.iters)
            ab = n * (4 * cfg["C"] * s_a + 4 * cfg["M"]) + 16 * cfg["C"] * cfg["M"]
            res[f"{algo}_fused_GBps_alg"] = ab / (res[f"{algo}_fused_ms"] * 1e-3) / 1e9
        except Exception as e:  # report, keep going
            res[f"{algo}_error"] = str(e)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
