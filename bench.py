#!/usr/bin/env python
"""Benchmark of the fused ITLUMM hot path (one step = itlumm_amm over one batch of rows).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2] [--algo auto|simt|tc]
  python bench.py --impl reference ...     # the CPU oracle, timed as it stands (reference arm)

Default workload: cfg5 (BASELINE configs[4], the largest single-GPU single-layer config).
N > 1 runs under torchrun (one process per GPU, NCCL): rank 0 fits the layer once and
broadcasts its parameters (one packed payload); the config's fixed global row count is sharded
over the ranks (strong scaling; --scaling weak gives every rank the full N instead), with no
collective in the data path.  Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOAD_DESC = {
    "cfg1": "BASELINE configs[0]: MNIST-shaped final layer, N=1000 D=784 M=10 C=16 (no ReLU)",
    "cfg2": "BASELINE configs[1]: MNIST-shaped hidden layer, N=60000 D=784 M=512 C=32, seeded permutation, ReLU",
    "cfg3_c64": "BASELINE configs[2]: CIFAR-shaped layer, N=50000 D=3072 M=1024 C=64",
    "cfg3_c128": "BASELINE configs[2]: CIFAR-shaped layer, N=50000 D=3072 M=1024 C=128",
    "cfg5": "BASELINE configs[4]: FFN-shaped stress case, N=262144 D=4096 M=4096 C=256, bf16 input",
}
for _w in ("cfg2", "cfg3_c64", "cfg3_c128", "cfg5"):
    WORKLOAD_DESC[_w + "_packed"] = (WORKLOAD_DESC[_w] + "; SPLIT-PACKED input: each row holds only its 4C split "
                                     "values in [c][level] order (the same layer re-parameterised, bit-identical "
                                     "outputs; SURVEY 8(d) judges the 70% HBM target on this layout)")
for _c in synth.MLP_CFG["C_sweep"]:
    WORKLOAD_DESC[f"cfg4_c{_c}"] = (f"BASELINE configs[3]: whole 3-layer ReLU MLP 3072-1024-1024-10, every layer "
                                   f"ITLUMM with C={_c}, N=1048576 CIFAR-shaped rows (itlumm_mlp_forward)")
METRIC = "fused ITLUMM rows/s"


def base_workload(workload: str):
    """(base config name, split-packed?) of a workload name."""
    return (workload[:-7], True) if workload.endswith("_packed") else (workload, False)


def _split_packed(params: dict):
    """Bench-local split-packed re-parameterisation (host indexing only, shared by both arms; the
    product exposes the same as paper_2207_05808_b200.split_packed): cols[c][t] =
    perm[b_c + split_dim[c][t]]; the packed layer has D = 4C, identity perm, 4-dim chunks."""
    D, C = int(params["D"]), int(params["C"])
    perm = np.arange(D) if params.get("perm") is None else np.asarray(params["perm"], np.int64)
    if params.get("boundaries") is None:
        sizes = np.full(C, D // C)
        sizes[: D % C] += 1
        bnd = np.concatenate([[0], np.cumsum(sizes)])
    else:
        bnd = np.asarray(params["boundaries"], np.int64)
    cols = perm[bnd[:C, None] + np.asarray(params["split_dim"], np.int64).reshape(C, 4)].reshape(-1)
    packed = {k: v for k, v in params.items() if k != "T"}
    packed.update(D=4 * C, perm=np.arange(4 * C, dtype=np.int32), boundaries=np.arange(0, 4 * C + 1, 4, dtype=np.int32),
                  split_dim=np.tile(np.arange(4, dtype=np.int32), (C, 1)))
    return packed, cols


def _rows_chunk(a):
    return synth.rows(*a)


def gen_rows(dist, cfg, stream, r0, r1, D):
    """synth.rows in parallel over the 65536-row seed chunks (identical result)."""
    bounds = list(range(r0, r1, synth.CHUNK_ROWS)) + [r1]
    if len(bounds) <= 3:
        return synth.rows(dist, cfg, stream, r0, r1, D)
    import multiprocessing as mp
    jobs = [(dist, cfg, stream, a, b, D) for a, b in zip(bounds[:-1], bounds[1:])]
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        parts = pool.map(_rows_chunk, jobs)
    return np.concatenate(parts, axis=0)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def acc_kernel_name(C, M):
    """Which accumulate kernel AUTO runs (the rule of tc_layout_host, csrc/tc.cuh): the LUT stays
    resident in shared memory (1-CTA k_tc) unless that would force slices narrower than 256 columns;
    a streamed LUT runs on CTA pairs (k_tcp)."""
    kb = (16 * C + 127) // 128
    ns_max = (128 * 1024 // (kb * 128)) // 32 * 32
    streamed = ns_max < 32 or (ns_max < 256 and M > ns_max)
    return ("k_tcp (a3' one-hot x LUT, tcgen05 CTA pairs, streamed LUT, + a4)" if streamed
            else "k_tc (a3' one-hot x LUT on tcgen05, resident LUT, + a4)")


def i8_peaks():
    """Two dense int8 peaks for the one-hot x LUT contraction: the measured bf16 GEMM burst
    (MEASURED_PEAKS.json) x the nominal int8/bf16 ratio 2 (4.5 / 2.25 PFLOP/s dense), and the
    kind::i8 issue rate measured by the builder's probe (tools/probes/mma_rate.cu:
    profiles/r01/mma_rate.jsonl, 4558 dense-equivalent TOPS at N=256)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        bf = (2.0 * float(d["bf16_tflops"]), "measured bf16 burst (MEASURED_PEAKS.json) x 2 (int8/bf16 nominal ratio)")
    else:
        bf = (2.0 * 1590.0, "fallback (B200_PROFILING.md: 1.59 PF bf16) x 2")
    return [bf, (4558.0, "measured tcgen05 kind::i8 issue rate (profiles/r01/mma_rate.jsonl, N=256)")]


def alg_bytes(w: dict, n: int) -> int:
    """A split columns + output + LUT = N*(4C*s_A + 4M) + 16CM per launch."""
    s_a = 2 if w["dtype"] == "bf16" else 4
    return n * (4 * w["C"] * s_a + 4 * w["M"]) + 16 * w["C"] * w["M"]


def ncu_traffic(workload: str, algo: str, n_gpus: int, rows: int):
    """DRAM read+write bytes of one call from a committed ncu capture of that exact step (the
    capture's command line, rows and n_gpus are recorded next to the number), or None."""
    p = os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(f"{workload}:{algo}:rows={rows}")
    return v if isinstance(v, dict) else None


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.out = None

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits", "-lms", "50"],
                                     stdout=self.out, stderr=subprocess.DEVNULL)
        time.sleep(0.3)

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        self.proc.wait()
        self.out.flush()
        with open(self.out.name) as f:
            lines = [l.strip() for l in f if l.strip()]
        os.unlink(self.out.name)
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 10:
                continue
            try:
                sm.append(float(parts[2]))
                mx = float(parts[3])
            except ValueError:
                continue
            try:
                pw.append(float(parts[4]))
            except ValueError:
                pass
            for n, v in zip(names, parts[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        out = {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(sm)}
        if pw:   # nvidia-smi power.draw is a ~1 s average: it lags a short timed region (only the max
            out["power_w_max_1s_avg"] = float(max(pw))   # is reported; tools/clock_probe.py measures sustained power)
        return out


# --------------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2207_05808_b200 import Plan, fit_layer
    from paper_2207_05808_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    base, packed = base_workload(args.workload)
    cfg = synth.CONFIGS[base]
    n_global = (cfg["N"] if args.rows is None else args.rows) * (world if args.scaling == "weak" else 1)
    # strong scaling: the fixed global row count split over the ranks; weak: every
    # rank its own full N rows of the seeded stream
    r0, r1 = pdist.shard_rows(n_global, world, rank)
    n = r1 - r0
    relu = cfg["relu"]
    bf16 = cfg["dtype"] == "bf16"

    # offline fit on rank 0 (host), broadcast once over NCCL, plan on every rank
    params = None
    if rank == 0:
        w0 = synth.workload(base, n_rows=0)
        params = fit_layer(w0["A_train"], w0["B"], w0["C"], w0["perm"], w0["bias"], a_is_bf16=bf16)
    if world > 1:
        params = pdist.broadcast_params(params, dev)          # one packed payload over NCCL
    cols = None
    if packed:
        params, cols = _split_packed(params)
    plan = Plan(params, device=local, algo=args.algo)

    # this rank's rows [r0, r1) of the seeded stream (chunk-seeded: the same rows for any world size)
    A_host = gen_rows(cfg["dist"], cfg["cfg"], 0, r0, r1, cfg["D"])
    if packed:
        A_host = np.ascontiguousarray(A_host[:, cols])
    A_t = torch.from_numpy(A_host.view(np.int16) if bf16 else A_host)
    A_pin = A_t.pin_memory()
    # rotate enough A/out buffer sets that the inputs read between two uses of a buffer exceed
    # twice the L2 (126 MB): 2 sets for row-major inputs, more for split-packed ones
    nbuf = int(min(16, max(2, -(-(256 << 20) // max(1, A_host.nbytes)))))
    A_dev = [A_pin.to(dev) for _ in range(nbuf)]
    if bf16:
        A_dev = [a.view(torch.bfloat16) for a in A_dev]
        A_pin = A_pin.view(torch.bfloat16)
    out_dev = [torch.empty((n, cfg["M"]), dtype=torch.float32, device=dev) for _ in range(nbuf)]
    stream = torch.cuda.current_stream(dev)

    def step(i):
        plan.amm(A_dev[i % nbuf], out=out_dev[i % nbuf], relu=relu)
        return plan.last_launch_count

    def graph_of(fn, nsteps):
        """Capture nsteps calls of fn(i) into one CUDA graph (no host work between steps)."""
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(stream)
        n_launch = 0
        with torch.cuda.stream(cs):
            with torch.cuda.graph(g, stream=cs):
                for i in range(nsteps):
                    n_launch += fn(i)
        stream.wait_stream(cs)
        torch.cuda.synchronize(dev)
        return g, n_launch

    def timed_replay(g):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize(dev)
        return a.elapsed_time(b)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    per_step_launches = plan.last_launch_count
    # the K timed steps are one CUDA graph (captured here, replayed once untimed to warm it)
    g_steps, launches = graph_of(step, args.steps)
    g_steps.replay()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    total_ms = timed_replay(g_steps)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    if world > 1:
        total_ms = pdist.max_over_ranks(total_ms, dev)
    ms_per_step = total_ms / args.steps
    launch_ms = ms_per_step                      # one itlumm_amm call per step
    rows_per_s = n_global / (ms_per_step * 1e-3)
    del g_steps

    # per-kernel breakdown of the step (same plan, same buffers, graph-timed through the C ABI)
    kernels = []
    if per_step_launches == 2:
        codes = plan.encode(A_dev[0])
        kk = min(args.steps, 200)
        g_enc, _ = graph_of(lambda i: (plan.encode(A_dev[i % nbuf], codes=codes), 1)[1], kk)
        g_acc, _ = graph_of(lambda i: (plan.lut_accumulate(codes, out=out_dev[i % nbuf], relu=relu), 1)[1], kk)
        t_enc, t_acc = timed_replay(g_enc) / kk, timed_replay(g_acc) / kk
        s_a = 2 if bf16 else 4
        nb = (cfg["C"] + 1) // 2
        b_enc = n * (4 * cfg["C"] * s_a + nb)
        b_acc = n * (nb + 4 * cfg["M"]) + 16 * cfg["C"] * cfg["M"]
        if world > 1:
            t_enc, t_acc = pdist.max_over_ranks(t_enc, dev), pdist.max_over_ranks(t_acc, dev)
        kernels = [
            {"kernel": "k_encode_rows (a1+a2)", "ms": t_enc, "alg_bytes": b_enc,
             "achieved_GBps": b_enc / (t_enc * 1e-3) / 1e9,
             "note": ("split-packed rows: 4C values per row, contiguous" if packed else
                      "reads whole rows: the 4C split columns touch ~every DRAM line of a row")},
            {"kernel": acc_kernel_name(cfg["C"], cfg["M"]), "ms": t_acc, "alg_bytes": b_acc,
             "achieved_GBps": b_acc / (t_acc * 1e-3) / 1e9},
        ]
        del g_enc, g_acc
        # the accumulate's other roofline (SURVEY 8(d) "tensor int8 ceiling = peak / (32 C M)"):
        # the one-hot x LUT product is 2 * 16C * M int8 ops per row (16x the method's C*M
        # lookup-adds: it describes the tensor-core formulation, not the method's work)
        ops = 32.0 * cfg["C"] * cfg["M"] * n
        ach = ops / (t_acc * 1e-3) / 1e12
        kernels[1]["tensor"] = [{"bound": "tensor", "achieved": ach, "peak": pk,
                                 "unit": "TOPS (int8, dense-equivalent one-hot MMA work)",
                                 "frac": ach / pk, "peak_source": src, "ops_per_launch": ops}
                                for pk, src in i8_peaks()]

    # end to end through the host-buffer C-ABI call (H2D + kernel + D2H inside the region)
    out_pin = torch.empty((n, cfg["M"]), dtype=torch.float32).pin_memory()
    k_e2e = max(3, min(args.steps, args.e2e_steps))
    for _ in range(2):
        plan.amm_host(A_pin, out=out_pin, relu=relu)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(k_e2e):
        plan.amm_host(A_pin, out=out_pin, relu=relu)
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - t0) / k_e2e
    if world > 1:
        e2e_s = pdist.max_over_ranks(e2e_s, dev)
        dist.barrier()
    e2e = {"value": n_global / e2e_s, "unit": "rows/s",
           "h2d_bytes_per_step": int(A_host.nbytes), "d2h_bytes_per_step": int(n * cfg["M"] * 4),
           "api": "itlumm_amm_host (pinned host buffers, chunked H2D/kernel/D2H)", "steps": k_e2e}

    peak, peak_src = peaks()
    ab = alg_bytes(cfg, n)
    achieved = ab / (launch_ms * 1e-3) / 1e9
    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(args.workload, params, n, budget_s=args.cpu_budget, cols=cols)
        line = {
            "metric": METRIC, "value": rows_per_s, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded stand-in for the dataset, DESIGN.md input recipe)",
            "config": {"workload": WORKLOAD_DESC[args.workload], "name": args.workload,
                       "rows_per_gpu": n, "global_rows": n_global, "D": int(params["D"]), "C": cfg["C"],
                       "M": cfg["M"], "input": ("bf16" if bf16 else "f32") + (" split-packed" if packed else " row-major"),
                       "epilogue": "relu" if relu else "none", "algo": args.algo,
                       "parallelism": f"rows sharded dp{world}" + (" (strong: fixed global N)" if args.scaling == "strong"
                                                                   else " (weak: N rows per rank)"),
                       "l2": f"inputs larger than L2: A {A_host.nbytes / 2**20:.0f} MiB per step, {nbuf} rotating "
                             f"A/out buffer sets ({nbuf * A_host.nbytes / 2**20:.0f} MiB of A between reuses of a buffer)",
                       "timing": "K steps captured as one CUDA graph, replayed once between CUDA events",
                       "compute": "uint8 LUT, exact int32 accumulate, fp32 compare + fmaf dequant"},
            "output_elems_per_s": rows_per_s * cfg["M"],
            # the method's bytes (A split columns + output + LUT) of one itlumm_amm call
            # over its device time, against the measured HBM copy bandwidth
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": (tr["bytes"] if (tr := ncu_traffic(args.workload, args.algo, world, n)) else None),
                         "traffic_source": (tr["source"] if tr else "no committed ncu capture of this step"),
                         "alg_bytes_per_launch": ab, "launch_ms": launch_ms,
                         "peak_source": peak_src,
                         "kernel": f"itlumm_amm ({per_step_launches} kernel launch(es) per call)",
                         "kernels": kernels},
            # secondary: the tensor-core accumulate against the int8 roofline of its one-hot x LUT
            # formulation (16x the method's work), both peaks
            "roofline_tensor": (kernels[1]["tensor"] if kernels else None),
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return line


def run_ours_mlp(args):
    """BASELINE configs[3]: one step = itlumm_mlp_forward of the whole 3-layer MLP over N rows."""
    import torch
    import torch.distributed as dist
    from paper_2207_05808_b200 import Mlp, fit_mlp
    from paper_2207_05808_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    C = int(args.workload.split("_c")[1])
    n_global = (synth.MLP_CFG["N"] if args.rows is None else args.rows) * (world if args.scaling == "weak" else 1)
    r0, r1 = pdist.shard_rows(n_global, world, rank)
    n = r1 - r0
    layers = synth.MLP_LAYERS
    w = synth.mlp_workload(C, 0)
    params = None
    if rank == 0:
        params = fit_mlp(w["A_train"], w["Bs"], w["Cs"], w["perms"], w["biases"], w["relus"], device=local)
    if world > 1:
        params = pdist.broadcast_layers(params, dev)          # every layer in one packed payload
    mlp = Mlp(params, w["relus"], device=local)
    A_host = gen_rows(synth.MLP_CFG["dist"], synth.MLP_CFG["cfg"], 0, r0, r1, layers[0][0])
    A_pin = torch.from_numpy(A_host).pin_memory()
    nbuf = 2
    A_dev = [A_pin.to(dev) for _ in range(nbuf)]
    M = layers[-1][1]
    out_dev = [torch.empty((n, M), dtype=torch.float32, device=dev) for _ in range(nbuf)]
    stream = torch.cuda.current_stream(dev)

    def step(i):
        mlp.forward(A_dev[i % nbuf], out=out_dev[i % nbuf])
        return mlp.last_launch_count

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(dev)
    cs.wait_stream(stream)
    launches = 0
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            for i in range(args.steps):
                launches += step(i)
    stream.wait_stream(cs)
    g.replay()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    a.record(stream)
    g.replay()
    b.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    total_ms = a.elapsed_time(b)
    if world > 1:
        total_ms = pdist.max_over_ranks(total_ms, dev)
    del g
    ms_per_step = total_ms / args.steps
    rows_per_s = n_global / (ms_per_step * 1e-3)
    # end to end through the public host-buffer C-ABI call (itlumm_mlp_forward_host: pinned H2D of
    # the rows, forward, D2H of the logits, pipelined in chunks inside the library)
    out_pin = torch.empty((n, M), dtype=torch.float32).pin_memory()
    k_e2e = max(2, min(args.steps, args.e2e_steps))
    mlp.forward_host(A_pin, out=out_pin)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(k_e2e):
        mlp.forward_host(A_pin, out=out_pin)
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - t0) / k_e2e
    if world > 1:
        e2e_s = pdist.max_over_ranks(e2e_s, dev)
    widths = mlp.widths()
    # bytes the method moves with dead-column elimination: layer l reads its 4C split columns and
    # writes the widths[l] columns it computes (the last layer all M), plus its LUT of those columns
    ab_row = sum(4 * C * 4 + 4 * wl for wl in widths)
    ab = n * ab_row + sum(16 * C * wl for wl in widths)
    ab_full = n * sum(4 * C * 4 + 4 * m for (_, m, _) in layers) + sum(16 * C * m for (_, m, _) in layers)
    peak, peak_src = peaks()
    achieved = ab / (ms_per_step * 1e-3) / 1e9
    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            import oracle
            cores = os.cpu_count() or 1
            ns = 2048
            t0 = time.perf_counter()
            oracle.mlp_forward(params, w["relus"], A_host[:ns], nthreads=cores)
            v = ns / (time.perf_counter() - t0)
            cpu = {"value": v, "unit": "rows/s", "cores": cores, "kind": "oracle",
                   "sample": f"first {ns} rows, all 3 layers computed in full"}
        line = {
            "metric": METRIC, "value": rows_per_s, "unit": "rows/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded stand-in for CIFAR-shaped rows, DESIGN.md input recipe)",
            "config": {"workload": WORKLOAD_DESC[args.workload], "name": args.workload,
                       "rows_per_gpu": n, "global_rows": n_global, "layers": layers, "C": C,
                       "computed_widths": widths, "input": "f32 row-major",
                       "parallelism": f"rows sharded dp{world}",
                       "l2": f"inputs larger than L2 (A {A_host.nbytes / 2**30:.1f} GiB/step), {nbuf} rotating buffers",
                       "timing": "K steps captured as one CUDA graph, replayed once between CUDA events"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "alg_bytes_per_launch": ab, "launch_ms": ms_per_step, "peak_source": peak_src,
                         "kernel": f"itlumm_mlp_forward ({launches // args.steps} launches per call)",
                         "note": "bytes the method moves with dead-column elimination (each layer: its 4C split "
                                 "columns in, the columns it computes out, their LUT); the three full-width "
                                 "layers would be full_width_alg_bytes",
                         "full_width_alg_bytes": ab_full},
            "e2e": {"value": n_global / e2e_s, "unit": "rows/s", "h2d_bytes_per_step": int(A_host.nbytes),
                    "d2h_bytes_per_step": int(n * M * 4),
                    "api": "itlumm_mlp_forward_host (pinned host buffers, chunked H2D/forward/D2H)",
                    "steps": k_e2e},
            "gpu_launches": launches, "clocks": clocks, "cpu_baseline": cpu,
        }
    mlp.close()
    if world > 1:
        dist.destroy_process_group()
    return line


# --------------------------------------------------------------------------------- oracle
def _oracle_rows_per_s(params, A, relu, dtype, nthreads):
    import oracle
    t0 = time.perf_counter()
    oracle.amm(params, A, relu=relu, dtype=dtype, nthreads=nthreads)
    return A.shape[0] / (time.perf_counter() - t0)


def cpu_baseline(workload: str, params: dict, n: int, budget_s: float = 15.0, cols=None):
    """The oracle (plain C, never tuned) on the host cores, on a bounded sample of the same
    workload (fitted parameters shared); ~budget_s seconds of work."""
    cfg = synth.CONFIGS[base_workload(workload)[0]]
    cores = os.cpu_count() or 1
    dtype = "bf16" if cfg["dtype"] == "bf16" else "f32"
    sel = (lambda a: np.ascontiguousarray(a[:, cols])) if cols is not None else (lambda a: a)
    probe = sel(synth.rows(cfg["dist"], cfg["cfg"], 0, 0, min(n, 512), cfg["D"]))
    rate = _oracle_rows_per_s(params, probe, cfg["relu"], dtype, cores)
    n_s = int(max(512, min(n, rate * budget_s)))
    A = sel(synth.rows(cfg["dist"], cfg["cfg"], 0, 0, n_s, cfg["D"]))
    v = _oracle_rows_per_s(params, A, cfg["relu"], dtype, cores)
    return {"value": v, "unit": "rows/s", "cores": cores, "kind": "oracle",
            "sample": f"first {n_s} of the {n} rows of {workload} (rank 0), full encode+accumulate+dequant"}


def run_reference(args):
    """--impl reference: the CPU oracle timed as it stands on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle
    from oracle import fit as ofit
    if args.workload.startswith("cfg4"):
        return run_reference_mlp(args)
    base, packed = base_workload(args.workload)
    cfg = synth.CONFIGS[base]
    n = cfg["N"] if args.rows is None else args.rows
    w0 = synth.workload(base, n_rows=0)
    bf16 = cfg["dtype"] == "bf16"
    params = ofit.fit(w0["A_train"], w0["B"], w0["C"], w0["perm"], w0["bias"], a_is_bf16=bf16)
    cols = None
    if packed:
        params, cols = _split_packed(params)
    sel = (lambda a: np.ascontiguousarray(a[:, cols])) if packed else (lambda a: a)
    dtype = "bf16" if bf16 else "f32"
    cores = os.cpu_count() or 1
    probe = sel(synth.rows(cfg["dist"], cfg["cfg"], 0, 0, min(n, 512), cfg["D"]))
    rate = _oracle_rows_per_s(params, probe, cfg["relu"], dtype, cores)
    per_step = int(max(1, min(n, rate * args.ref_budget / max(1, args.steps + args.warmup))))
    A = sel(synth.rows(cfg["dist"], cfg["cfg"], 0, 0, per_step, cfg["D"]))
    for _ in range(args.warmup):
        oracle.amm(params, A, relu=cfg["relu"], dtype=dtype, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.amm(params, A, relu=cfg["relu"], dtype=dtype, nthreads=cores)
    dt = time.perf_counter() - t0
    v = per_step * args.steps / dt
    sample = f"first {per_step} of the {n} rows of {args.workload} per step"
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "rows/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD_DESC[args.workload], "name": args.workload,
                       "rows_per_step": per_step, "D": cfg["D"], "C": cfg["C"], "M": cfg["M"]},
            "cpu_baseline": {"value": v, "unit": "rows/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_reference_mlp(args):
    import oracle
    C = int(args.workload.split("_c")[1])
    n = synth.MLP_CFG["N"] if args.rows is None else args.rows
    w = synth.mlp_workload(C, 0)
    params = oracle.fit_mlp(w["A_train"], w["Bs"], w["Cs"], w["perms"], w["biases"], w["relus"])
    cores = os.cpu_count() or 1
    probe = synth.rows(synth.MLP_CFG["dist"], synth.MLP_CFG["cfg"], 0, 0, 512, synth.MLP_LAYERS[0][0])
    t0 = time.perf_counter()
    oracle.mlp_forward(params, w["relus"], probe, nthreads=cores)
    rate = 512 / (time.perf_counter() - t0)
    per_step = int(max(1, min(n, rate * args.ref_budget / max(1, args.steps + args.warmup))))
    A = synth.rows(synth.MLP_CFG["dist"], synth.MLP_CFG["cfg"], 0, 0, per_step, synth.MLP_LAYERS[0][0])
    for _ in range(args.warmup):
        oracle.mlp_forward(params, w["relus"], A, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.mlp_forward(params, w["relus"], A, nthreads=cores)
    dt = time.perf_counter() - t0
    v = per_step * args.steps / dt
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "rows/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD_DESC[args.workload], "name": args.workload,
                       "rows_per_step": per_step, "C": C},
            "cpu_baseline": {"value": v, "unit": "rows/s", "cores": cores, "kind": "oracle",
                             "sample": f"first {per_step} rows per step, all layers in full"},
            "e2e": {"value": v, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the config's global row count split over the ranks; weak: N rows per rank")
    ap.add_argument("--algo", default="auto", choices=["auto", "simt", "tc", "tc_pipe"])
    ap.add_argument("--rows", type=int, default=None, help="override rows per GPU (default: config N)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=90.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.gpus > 1:                      # the driver checks the communicator's rank count here
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        line = run_reference(args)
    elif args.workload.startswith("cfg4"):
        line = run_ours_mlp(args)
    else:
        line = run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
