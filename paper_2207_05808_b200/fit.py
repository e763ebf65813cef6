"""Offline fit of an ITLUMM layer on the host (fit-time, NOT the hot path).

The paper's contributions are all fit-time; the inference path (the CUDA library)
consumes what this module produces: gather permutation + partition, depth-4 trees, and the
uint8 LUT with per-output scale/offset.  The rules follow the same readings as the oracle
(R3-R6, R12) but this is an independent, vectorised implementation; the test
suite checks that both produce bit-identical parameters.

Reductions are defined so that results are reproducible bit for bit: node means and node sums
of squares are numpy reductions over the node's rows in ascending row order; the LUT is
accumulated over subspace dims in ascending order (product rounded, then added).
"""
from __future__ import annotations

import numpy as np

N_LEVELS = 4
N_PROTO = 16


def chunk_bounds(D: int, C: int) -> np.ndarray:
    """C contiguous chunks of the permuted dims, sizes differing by <= 1, larger first (R12)."""
    if C < 1 or C > D:
        raise ValueError(f"need 1 <= C <= D, got C={C}, D={D}")
    sizes = np.full(C, D // C, dtype=np.int64)
    sizes[: D % C] += 1
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)


def _segments(leaf: np.ndarray, n_nodes: int):
    order = np.argsort(leaf, kind="stable")
    cnt = np.bincount(leaf, minlength=n_nodes)
    starts = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    return order, cnt, starts


def _fit_subspace(X: np.ndarray):
    """One tree (R3/R4) + leaf-mean prototypes (R5) for one subspace X (n x d, fp64)."""
    n, d = X.shape
    leaf = np.zeros(n, dtype=np.int64)
    split = np.zeros(N_LEVELS, dtype=np.int32)
    thr = np.zeros(2 ** N_LEVELS - 1, dtype=np.float64)
    level_means = []
    for t in range(N_LEVELS + 1):
        nn = 2 ** t
        order, cnt, starts = _segments(leaf, nn)
        means = np.zeros((nn, d))
        sse = np.zeros(d)
        for node in range(nn):
            if cnt[node]:
                Xn = X[order[starts[node]:starts[node] + cnt[node]]]
                means[node] = Xn.mean(axis=0)
                if t < N_LEVELS:
                    sse += ((Xn - means[node]) ** 2).sum(axis=0)
        level_means.append((means, cnt))
        if t == N_LEVELS:
            break
        j = int(np.argmax(sse))
        split[t] = j
        # lower median per node: sort rows by (node, value), take index (cnt-1)//2 of each segment
        key = np.lexsort((X[:, j], leaf))
        base = 2 ** t - 1
        for node in range(nn):
            h = base + node
            if cnt[node]:
                thr[h] = X[key[starts[node] + (cnt[node] - 1) // 2], j]
            else:
                thr[h] = thr[(h - 1) // 2]
        leaf = 2 * leaf + (X[:, j] > thr[base + leaf]).astype(np.int64)
    # prototypes: leaf mean, or the nearest non-empty ancestor's mean for an empty leaf
    P = np.zeros((N_PROTO, d))
    for k in range(N_PROTO):
        for t in range(N_LEVELS, -1, -1):
            means, cnt = level_means[t]
            node = k >> (N_LEVELS - t)
            if cnt[node]:
                P[k] = means[node]
                break
    return split, thr, P


def fit_trees_gpu(Xall: np.ndarray, bnd: np.ndarray, device: int = 0):
    """Depth-4 trees of all C subspaces at once on the GPU (readings R3/R4; SURVEY f4 "tree fitting at
    BASELINE scale"), fp64 torch ops batched over codebooks: per level the pooled within-node sum of
    squares of every dim (segment sums by scatter_add), its argmax (first maximum = smallest dim on
    ties), and each node's lower median on the chosen dim (a stable sort of the node's values).
    Returns split [C][4], thresholds [C][15] (fp64 data values) and the leaf of every row [n][C].
    The leaf assignment decides the prototypes, which the caller averages on the host exactly as the
    oracle does, so the LUT is bit-identical whenever the split dims agree (their SSE sums differ from
    numpy's only in rounding order)."""
    import torch
    dev = torch.device("cuda", device)
    n = Xall.shape[0]
    C = len(bnd) - 1
    dmax = int(np.max(np.diff(bnd)))
    # [C][n][dmax] fp64, padded dims hold 0 (their SSE is 0: never chosen unless every dim is constant,
    # where the first dim wins in both implementations)
    Xc = np.zeros((C, n, dmax))
    for c in range(C):
        Xc[c, :, : bnd[c + 1] - bnd[c]] = Xall[:, bnd[c]:bnd[c + 1]]
    X = torch.from_numpy(Xc).to(dev)
    leaf = torch.zeros((C, n), dtype=torch.int64, device=dev)
    split = torch.zeros((C, N_LEVELS), dtype=torch.int64, device=dev)
    thr = torch.zeros((C, 2 ** N_LEVELS - 1), dtype=torch.float64, device=dev)
    crange = torch.arange(C, device=dev)
    for t in range(N_LEVELS):
        nn = 2 ** t
        seg = (crange[:, None] * nn + leaf).reshape(-1)                     # (c, node) segment of each row
        cnt = torch.bincount(seg, minlength=C * nn).to(torch.float64)
        sums = torch.zeros((C * nn, dmax), dtype=torch.float64, device=dev).index_add_(0, seg, X.reshape(-1, dmax))
        means = sums / cnt.clamp(min=1)[:, None]
        dev2 = (X.reshape(-1, dmax) - means[seg]) ** 2
        sse = torch.zeros((C * nn, dmax), dtype=torch.float64, device=dev).index_add_(0, seg, dev2)
        j = torch.argmax(sse.reshape(C, nn, dmax).sum(dim=1), dim=1)    # [C]; first maximum on ties
        split[:, t] = j
        v = X[crange, :, j]                                                 # [C][n] values on the split dim
        # lower median per node: stable sort by value, then stable by node -> node segments in value order
        o1 = torch.argsort(v, dim=1, stable=True)
        o2 = torch.argsort(torch.gather(leaf, 1, o1), dim=1, stable=True)
        order = torch.gather(o1, 1, o2)
        sv = torch.gather(v, 1, order)
        cnt_n = cnt.reshape(C, nn).long()
        starts = torch.cumsum(cnt_n, dim=1) - cnt_n
        mid = (starts + (cnt_n - 1).clamp(min=0) // 2).clamp(max=n - 1)
        med = torch.gather(sv, 1, mid)
        base = 2 ** t - 1
        for node in range(nn):                                              # empty node: parent's threshold
            h = base + node
            parent = thr[:, (h - 1) // 2] if h > 0 else torch.zeros(C, dtype=torch.float64, device=dev)
            thr[:, h] = torch.where(cnt_n[:, node] > 0, med[:, node], parent)
        leaf = 2 * leaf + (v > torch.gather(thr, 1, base + leaf)).long()
    return split.cpu().numpy().astype(np.int32), thr.cpu().numpy(), leaf.t().contiguous().cpu().numpy()


def _prototypes_from_leaves(X: np.ndarray, leaf: np.ndarray) -> np.ndarray:
    """Leaf-mean prototypes (R5) from a leaf assignment, with the oracle's reductions: node mean =
    numpy mean over the node's rows in ascending row order; an empty leaf takes its nearest
    non-empty ancestor's mean."""
    P = np.zeros((N_PROTO, X.shape[1]))
    for k in range(N_PROTO):
        for t in range(N_LEVELS, -1, -1):
            node = k >> (N_LEVELS - t)
            rows = np.nonzero((leaf >> (N_LEVELS - t)) == node)[0]
            if len(rows):
                P[k] = X[rows].mean(axis=0)
                break
    return P


def fit_layer(A_train: np.ndarray, B: np.ndarray, C: int, perm: np.ndarray | None = None,
              bias: np.ndarray | None = None, a_is_bf16: bool = False, device: int | None = None) -> dict:
    """Fit trees and the quantised LUT of one layer approximating A @ B (+ bias).  device=None fits
    the trees on the host; device=k fits them on GPU k (fit_trees_gpu) — same parameters.

    Returns the parameter dict consumed by :class:`paper_2207_05808_b200.Plan`."""
    if device is not None:
        return _fit_layer_gpu_trees(A_train, B, C, perm, bias, a_is_bf16, device)
    A = np.asarray(A_train)
    if a_is_bf16:
        A = (A.astype(np.uint32) << 16).view(np.float32)
    A = A.astype(np.float32)
    D = A.shape[1]
    B = np.asarray(B, dtype=np.float64)
    M = B.shape[1]
    perm = np.arange(D, dtype=np.int32) if perm is None else np.asarray(perm, dtype=np.int32)
    bnd = chunk_bounds(D, C)
    Xall = A[:, perm].astype(np.float64)
    Bp = B[perm]
    split = np.zeros((C, N_LEVELS), np.int32)
    thr = np.zeros((C, 2 ** N_LEVELS - 1), np.float32)
    T = np.zeros((C, N_PROTO, M))
    for c in range(C):
        sd, th, P = _fit_subspace(Xall[:, bnd[c]:bnd[c + 1]])
        split[c], thr[c] = sd, th.astype(np.float32)
        Bc = Bp[bnd[c]:bnd[c + 1]]
        for j in range(P.shape[1]):
            T[c] += P[:, j:j + 1] * Bc[j:j + 1, :]
    q, scale, lo = quantize_table(T)
    return dict(D=D, C=C, M=M, perm=perm, boundaries=bnd, split_dim=split, thresholds=thr,
                lut=q, scale=scale.astype(np.float32), offset=lo.astype(np.float32),
                bias=(np.zeros(M, np.float32) if bias is None else np.asarray(bias, np.float32)), T=T)


def _fit_layer_gpu_trees(A_train, B, C, perm, bias, a_is_bf16, device):
    A = np.asarray(A_train)
    if a_is_bf16:
        A = (A.astype(np.uint32) << 16).view(np.float32)
    A = A.astype(np.float32)
    D = A.shape[1]
    B = np.asarray(B, dtype=np.float64)
    M = B.shape[1]
    perm = np.arange(D, dtype=np.int32) if perm is None else np.asarray(perm, dtype=np.int32)
    bnd = chunk_bounds(D, C)
    Xall = A[:, perm].astype(np.float64)
    Bp = B[perm]
    split, thr64, leaf = fit_trees_gpu(Xall, bnd, device)
    T = np.zeros((C, N_PROTO, M))
    for c in range(C):
        P = _prototypes_from_leaves(Xall[:, bnd[c]:bnd[c + 1]], leaf[:, c])
        Bc = Bp[bnd[c]:bnd[c + 1]]
        for j in range(P.shape[1]):
            T[c] += P[:, j:j + 1] * Bc[j:j + 1, :]
    q, scale, lo = quantize_table(T)
    return dict(D=D, C=C, M=M, perm=perm, boundaries=bnd, split_dim=split, thresholds=thr64.astype(np.float32),
                lut=q, scale=scale.astype(np.float32), offset=lo.astype(np.float32),
                bias=(np.zeros(M, np.float32) if bias is None else np.asarray(bias, np.float32)), T=T)


def split_columns(params: dict) -> np.ndarray:
    """The 4C input columns the encoder reads, in [c][level] order: perm[b_c + split_dim[c][t]]
    (step a1 folded)."""
    D, C = int(params["D"]), int(params["C"])
    perm = np.arange(D) if params.get("perm") is None else np.asarray(params["perm"], np.int64)
    bnd = chunk_bounds(D, C) if params.get("boundaries") is None else np.asarray(params["boundaries"], np.int64)
    sd = np.asarray(params["split_dim"], np.int64).reshape(C, N_LEVELS)
    return perm[bnd[:C, None] + sd].reshape(-1).astype(np.int64)


def split_packed(params: dict):
    """Re-parameterise a fitted layer for SPLIT-PACKED input: an input row that
    holds only the 4C split values in [c][level] order, A_packed = A[:, cols].  The packed layer is
    an ordinary ITLUMM layer (D = 4C, identity permutation, 4-dim chunks, split_dim[c] = 0..3)
    with the same thresholds, LUT and dequant, so it computes bit-identical outputs from 16C
    input bytes per row (fp32) instead of whole rows.  Returns (packed_params, cols)."""
    C = int(params["C"])
    cols = split_columns(params)
    packed = {k: v for k, v in params.items() if k not in ("T",)}
    packed.update(D=4 * C, perm=np.arange(4 * C, dtype=np.int32), boundaries=np.arange(0, 4 * C + 1, 4, dtype=np.int32),
                  split_dim=np.tile(np.arange(N_LEVELS, dtype=np.int32), (C, 1)))
    return packed, cols


def quantize_table(T: np.ndarray):
    """uint8 LUT with per-output-column scale/offset (reading R6): lo = min, scale = (hi-lo)/255
    (1 for a constant column), q = clamp(floor((T-lo)/scale + 0.5), 0, 255), fp64."""
    T = np.asarray(T, np.float64)
    lo = T.min(axis=(0, 1))
    hi = T.max(axis=(0, 1))
    scale = np.where(hi > lo, (hi - lo) / 255.0, 1.0)
    q = np.clip(np.floor((T - lo) / scale + 0.5), 0, 255).astype(np.uint8)
    return q, scale, lo


def fit_mlp(A_train: np.ndarray, Bs: list, Cs: list, perms: list, biases: list, relus: list,
            device: int = 0, a_is_bf16: bool = False) -> list:
    """Fit every layer of an MLP whose linear layers are all replaced by ITLUMM (BASELINE
    configs[3]; P:110-121 incremental replacement).  Layer l+1's trees and LUT are fit on the
    ITLUMM outputs of the training rows through the already-replaced layers 0..l (reading O9 of
    SURVEY §8(c)); those activations come from the GPU path (Plan.amm), which is bit-identical to
    the oracle's inference."""
    import torch
    from .api import Plan

    X = np.asarray(A_train)
    out = []
    for l, (B, C, perm, bias, relu) in enumerate(zip(Bs, Cs, perms, biases, relus)):
        p = fit_layer(X, B, C, perm, bias, a_is_bf16=(a_is_bf16 and l == 0))
        out.append(p)
        if l + 1 < len(Bs):
            plan = Plan(p, device=device)
            if a_is_bf16 and l == 0:
                At = torch.from_numpy(np.ascontiguousarray(X).view(np.int16)).to(f"cuda:{device}").view(torch.bfloat16)
            else:
                At = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(f"cuda:{device}")
            X = plan.amm(At, relu=relu).cpu().numpy()
            plan.close()
    return out


def optimize_lut(params: dict, A_train: np.ndarray, B: np.ndarray, lam: float = 1.0, relu: bool = False,
                 iters: int = 200, lr: float = 1e-2, device: int = 0, a_is_bf16: bool = False,
                 objective: str = "mse") -> dict:
    """ITLUMM model-aware LUT optimisation, Eq. 3, on the GPU:
    argmin_T ||sigma(A B) - sigma(G T)||^2 + lam ||T - P0 B||^2, sigma = + bias (then ReLU when
    `relu`).  G comes from the plan's own encode kernel on the training rows.  Without a
    nonlinearity the bias cancels and T solves the normal equations (G^T G + lam I) T = G^T A B +
    lam P0 B (fp64, cuSOLVER through torch.linalg); with ReLU that solution seeds `iters` Adam steps
    on the ReLU objective.
    objective="kld": sigma = bias then a row-wise softmax, first term sum over rows of
    KL(softmax(a B + b) || softmax(g T + b)) (the objective the paper finds better; SPEC
    S:343), minimised by `iters` steps of plain gradient descent from T = P0 B with the analytic
    gradient G^T (softmax(G T + b) - softmax(A B + b)) + 2 lam (T - P0 B) (reading R23), fp64.
    Returns the parameters with the new table requantised (same trees), so the hot path is unchanged
    (P:131)."""
    import torch
    from .api import Plan

    dev = torch.device("cuda", device)
    C, M = int(params["C"]), int(params["M"])
    plan = Plan(params, device=device)
    X = np.asarray(A_train)
    if a_is_bf16:
        At = torch.from_numpy(np.ascontiguousarray(X).view(np.int16)).to(dev).view(torch.bfloat16)
        Af = torch.from_numpy((X.astype(np.uint32) << 16).view(np.float32)).to(dev).double()
    else:
        At = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(dev)
        Af = At.double()
    packed = plan.encode(At)
    plan.close()
    lo_nib, hi_nib = packed & 15, packed >> 4
    codes = torch.stack([lo_nib, hi_nib], dim=2).reshape(packed.shape[0], -1)[:, :C].long()
    N = codes.shape[0]
    G = torch.zeros((N, 16 * C), dtype=torch.float64, device=dev)
    G.scatter_(1, codes + 16 * torch.arange(C, device=dev), 1.0)
    Y = Af @ torch.from_numpy(np.asarray(B, np.float64)).to(dev)
    T0 = torch.from_numpy(np.asarray(params["T"], np.float64).reshape(16 * C, M)).to(dev)
    if objective == "kld":
        b = torch.from_numpy(np.asarray(params["bias"], np.float64)).to(dev)
        Pt = torch.softmax(Y + b, dim=1)
        T = T0.clone()
        for _ in range(int(iters)):
            T = T - lr * (G.T @ (torch.softmax(G @ T + b, dim=1) - Pt) + 2.0 * lam * (T - T0))
        Tn = T.reshape(C, 16, M).cpu().numpy()
        q, scale, lo = quantize_table(Tn)
        out = dict(params)
        out.update(lut=q, scale=scale.astype(np.float32), offset=lo.astype(np.float32), T=Tn)
        return out
    if objective != "mse":
        raise ValueError(f"objective must be 'mse' or 'kld', got {objective!r}")
    lhs = G.T @ G + lam * torch.eye(16 * C, dtype=torch.float64, device=dev)
    T = torch.linalg.solve(lhs, G.T @ Y + lam * T0)
    if relu:
        b = torch.from_numpy(np.asarray(params["bias"], np.float64)).to(dev)
        target = torch.relu(Y + b)
        Tv = T.clone().requires_grad_(True)
        opt = torch.optim.Adam([Tv], lr=lr)
        for _ in range(int(iters)):
            opt.zero_grad()
            loss = ((target - torch.relu(G @ Tv + b)) ** 2).sum() / N + lam * ((Tv - T0) ** 2).sum() / N
            loss.backward()
            opt.step()
        T = Tv.detach()
    Tn = T.reshape(C, 16, M).cpu().numpy()
    q, scale, lo = quantize_table(Tn)
    out = dict(params)
    out.update(lut=q, scale=scale.astype(np.float32), offset=lo.astype(np.float32), T=Tn)
    return out
