"""Multi-GPU plumbing: one process per GPU (torchrun), rows sharded over ranks.

The hot path has no exchange step (rows are independent), so the only
collectives are a one-time broadcast of the fitted parameters from rank 0 (NCCL over
NVLink/NVSwitch on the GPU box; gloo in the CPU tests) and a post-loop max of per-rank
timings.  Nothing here touches the data path."""
from __future__ import annotations

import numpy as np

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = dist = None

# order and dtypes of the broadcast payload
PARAM_FIELDS = [("perm", np.int32), ("boundaries", np.int32), ("split_dim", np.int32),
                ("thresholds", np.float32), ("lut", np.uint8), ("scale", np.float32),
                ("offset", np.float32), ("bias", np.float32)]


def shard_rows(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range of `rank` when n_total rows are split over `world` ranks; lower
    ranks take the remainder."""
    if world < 1 or not (0 <= rank < world) or n_total < 0:
        raise ValueError("bad shard arguments")
    q, r = divmod(n_total, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def weak_rows(n_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank processes its own n_per_rank rows of the seeded row stream."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


def broadcast_params(params: dict | None, device, src: int = 0, group=None) -> dict:
    """Broadcast a fitted parameter dict from `src` to every rank (one collective per field,
    once per plan, outside any timed region).  Non-src ranks pass params=None."""
    rank = dist.get_rank(group)
    hdr = torch.zeros(3, dtype=torch.int64, device=device)
    if rank == src:
        hdr[:] = torch.tensor([params["D"], params["C"], params["M"]], dtype=torch.int64)
    dist.broadcast(hdr, src, group=group)
    D, C, M = (int(x) for x in hdr.cpu().tolist())
    shapes = {"perm": (D,), "boundaries": (C + 1,), "split_dim": (C, 4), "thresholds": (C, 15),
              "lut": (C, 16, M), "scale": (M,), "offset": (M,), "bias": (M,)}
    out = dict(D=D, C=C, M=M)
    for name, dt in PARAM_FIELDS:
        if rank == src:
            arr = np.ascontiguousarray(params[name], dtype=dt)
            if arr.shape != shapes[name]:
                raise ValueError(f"{name} has shape {arr.shape}, expected {shapes[name]}")
            t = torch.from_numpy(arr.copy()).to(device)
        else:
            t = torch.empty(shapes[name], dtype=torch.from_numpy(np.zeros(0, dt)).dtype, device=device)
        dist.broadcast(t, src, group=group)
        out[name] = t.cpu().numpy()
    return out


def max_over_ranks(x: float, device, group=None) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
