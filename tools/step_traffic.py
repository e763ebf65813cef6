#!/usr/bin/env python
"""DRAM traffic of one bench step (one itlumm_amm call) in steady state.

    python tools/step_traffic.py run cfg5             # the exact bench step, 6 calls, rotating 2 buffer sets
    ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --csv --log-file launches.csv python tools/step_traffic.py run cfg5
    python tools/step_traffic.py parse launches.csv cfg5 [--out profiles/r02/ncu_traffic.json]

With --cache-control none the L2 is not flushed between launches, so the output a kernel leaves
dirty in L2 is counted where it is written back (the next kernel): summing the launches of one
middle call counts the call's own traffic in steady state."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CALLS = 6


def run(workload):
    import numpy as np
    import torch
    import synth
    from bench import base_workload, _split_packed, gen_rows
    from paper_2207_05808_b200 import Plan, fit_layer
    base, packed = base_workload(workload)
    cfg = synth.CONFIGS[base]
    bf16 = cfg["dtype"] == "bf16"
    w0 = synth.workload(base, n_rows=0)
    params = fit_layer(w0["A_train"], w0["B"], w0["C"], w0["perm"], w0["bias"], a_is_bf16=bf16)
    cols = None
    if packed:
        params, cols = _split_packed(params)
    A = gen_rows(cfg["dist"], cfg["cfg"], 0, 0, cfg["N"], cfg["D"])
    if packed:
        A = np.ascontiguousarray(A[:, cols])
    At = torch.from_numpy(A.view(np.int16) if bf16 else A).cuda()
    As = [At, At.clone()]
    if bf16:
        As = [a.view(torch.bfloat16) for a in As]
    outs = [torch.empty((cfg["N"], cfg["M"]), device="cuda") for _ in range(2)]
    plan = Plan(params)
    for i in range(CALLS):
        plan.amm(As[i % 2], out=outs[i % 2], relu=cfg["relu"])
    torch.cuda.synchronize()
    print(json.dumps({"workload": workload, "rows": cfg["N"], "launches_per_call": plan.last_launch_count}))


def parse(path, workload, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    iid, iname, imet, ival = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = {}
    for r in rows[1:]:
        k = per.setdefault(int(r[iid]), {"name": r[iname]})
        k[r[imet]] = float(r[ival].replace(",", ""))
    ids = sorted(per)
    # only the library's kernels (the harness's own copies/clones are excluded)
    ids = [i for i in ids if any(s in per[i]["name"] for s in ("k_encode", "k_tc", "k_lut"))]
    lpc = len(ids) // CALLS
    call = ids[3 * lpc: 4 * lpc]                       # the 4th of 6 calls: steady state
    unit = lambda k: 1.0  # noqa: E731  (ncu --csv reports bytes when asked for .sum in bytes)
    tot = sum(per[i]["dram__bytes_read.sum"] + per[i]["dram__bytes_write.sum"] for i in call)
    rec = {"bytes": int(tot), "source": os.path.relpath(path, ROOT) + " (ncu --cache-control none, call 4 of 6)",
           "kernels": [{"name": per[i]["name"][:60], "read": int(per[i]["dram__bytes_read.sum"]),
                        "write": int(per[i]["dram__bytes_write.sum"]),
                        "ms": per[i]["gpu__time_duration.sum"] / 1e6} for i in call]}
    print(json.dumps(rec, indent=1))
    if out:
        import synth
        from bench import base_workload
        n = synth.CONFIGS[base_workload(workload)[0]]["N"]
        d = json.load(open(out)) if os.path.exists(out) else {"_doc": __doc__.split("\n\n")[-1]}
        d[f"{workload}:auto:rows={n}"] = rec
        json.dump(d, open(out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        parse(sys.argv[2], sys.argv[3], sys.argv[5] if len(sys.argv) > 5 and sys.argv[4] == "--out" else None)
