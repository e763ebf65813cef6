"""Multi-GPU plumbing: one process per GPU (torchrun), rows sharded over ranks.

The hot path has no exchange step (rows are independent), so the only
collectives are a one-time broadcast of the fitted parameters from rank 0 (NCCL over
NVLink/NVSwitch on the GPU box; gloo in the CPU tests: a 512-byte header and ONE packed
payload) and a post-loop max of per-rank timings.  Nothing here touches the data path.
bench.py shards a fixed global row count over the ranks (strong scaling, shard_rows)."""
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


def _shapes(D: int, C: int, M: int) -> dict:
    return {"perm": (D,), "boundaries": (C + 1,), "split_dim": (C, 4), "thresholds": (C, 15),
            "lut": (C, 16, M), "scale": (M,), "offset": (M,), "bias": (M,)}


def pack_params(layers: list) -> tuple[np.ndarray, np.ndarray]:
    """Fitted layer dicts -> (header int64 [1 + 3L]: L, then D, C, M per layer; payload uint8: every
    field of PARAM_FIELDS of every layer, in order, 4-byte aligned)."""
    hdr = [len(layers)]
    parts = []
    for p in layers:
        D, C, M = int(p["D"]), int(p["C"]), int(p["M"])
        hdr += [D, C, M]
        shp = _shapes(D, C, M)
        for name, dt in PARAM_FIELDS:
            arr = np.ascontiguousarray(p[name] if p.get(name) is not None else np.zeros(shp[name]), dtype=dt)
            if arr.shape != shp[name]:
                raise ValueError(f"{name} has shape {arr.shape}, expected {shp[name]}")
            b = arr.view(np.uint8).reshape(-1)
            parts.append(b)
            if b.size % 4:
                parts.append(np.zeros(4 - b.size % 4, np.uint8))
    return np.array(hdr, np.int64), (np.concatenate(parts) if parts else np.zeros(0, np.uint8))


def unpack_params(hdr: np.ndarray, payload: np.ndarray) -> list:
    out, o = [], 0
    L = int(hdr[0])
    for l in range(L):
        D, C, M = (int(x) for x in hdr[1 + 3 * l: 4 + 3 * l])
        shp = _shapes(D, C, M)
        p = dict(D=D, C=C, M=M)
        for name, dt in PARAM_FIELDS:
            nbytes = int(np.prod(shp[name])) * np.dtype(dt).itemsize
            p[name] = payload[o:o + nbytes].view(dt).reshape(shp[name]).copy()
            o += nbytes + (-nbytes) % 4
        out.append(p)
    return out


def broadcast_layers(layers: list | None, device, src: int = 0, group=None) -> list:
    """Broadcast fitted layers from `src` to every rank, once per plan, outside any timed region:
    ONE payload collective (every field of every layer packed into one uint8 buffer) after a
    header collective that carries the sizes.  Non-src ranks pass layers=None."""
    rank = dist.get_rank(group)
    hbuf = torch.zeros(64, dtype=torch.int64, device=device)       # sizes + per-layer dims (L <= 20)
    if rank == src:
        hdr, payload = pack_params(layers)
        if hdr.size > 62:
            raise ValueError("too many layers for the broadcast header")
        hbuf[0], hbuf[1] = int(hdr.size), int(payload.size)
        hbuf[2:2 + hdr.size] = torch.from_numpy(hdr)
    dist.broadcast(hbuf, src, group=group)
    nh, npay = int(hbuf[0].item()), int(hbuf[1].item())
    hdr = hbuf[2:2 + nh].cpu().numpy()
    if rank == src:
        buf = torch.from_numpy(payload.copy()).to(device)
    else:
        buf = torch.empty(npay, dtype=torch.uint8, device=device)
    dist.broadcast(buf, src, group=group)
    return unpack_params(hdr, buf.cpu().numpy())


def broadcast_params(params: dict | None, device, src: int = 0, group=None) -> dict:
    """One layer: broadcast_layers([params])[0]."""
    return broadcast_layers([params] if params is not None else None, device, src, group)[0]


def max_over_ranks(x: float, device, group=None) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
