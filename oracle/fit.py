"""ORACLE — offline fit, written out plainly in fp64 (TEST INFRASTRUCTURE; see oracle/__init__.py).

Each function follows PAPER.md (P:line) / SPEC.md (S:line) step by step, in the paper's order,
with the readings R# of DESIGN.md where the sources are silent.  Plain loops over codebooks,
nodes and dims; numpy is used only for elementwise arithmetic, sorting and sums.
"""
from __future__ import annotations

import numpy as np

K = 16        # prototypes per codebook: "runs efficiently ... when K = 16"
LEVELS = 4    # "exactly 4 comparisons"


def boundaries(D: int, C: int) -> np.ndarray:
    """Slice the permuted dims into C contiguous "equally-sized chunks".

    Reading R12: when C does not divide D the first D mod C chunks get one extra
    dim ("larger first").  Returns b[0..C] with chunk c = [b[c], b[c+1])."""
    if not (1 <= C <= D):
        raise ValueError("need 1 <= C <= D")
    q, r = divmod(D, C)
    b = [0]
    for c in range(C):
        b.append(b[-1] + q + (1 if c < r else 0))
    return np.array(b, dtype=np.int32)


def fit_tree(X: np.ndarray):
    """Depth-4 balanced binary regression tree on one subspace.

    Reading R3 (BASELINE.json configs[0]: "per level, split dim = highest-variance dim of the
    training sample in that subspace; thresholds = node medians"): at level t the split dim
    j_t maximises the pooled within-node sum of squares sum_nodes sum_i (x_ij - mean_node_j)^2
    (ties -> smallest j).  Reading R4: threshold of node n = LOWER median x_((n-1)//2) of the
    node's values on j_t; an empty node copies its parent's threshold.  A row goes
    right iff x > threshold.

    Returns (split_dims[4], thresholds[15] heap order, nodes_by_level) where
    nodes_by_level[t] is the list of the 2^t row-index arrays at level t (t = 0..4)."""
    X = np.asarray(X, dtype=np.float64)
    n, d = X.shape
    nodes = [np.arange(n)]
    levels = [nodes]
    split_dims = []
    thr = np.zeros(2 ** LEVELS - 1, dtype=np.float64)
    for t in range(LEVELS):
        sse = np.zeros(d, dtype=np.float64)
        for idx in nodes:
            if len(idx) > 0:
                Xn = X[idx]
                sse += ((Xn - Xn.mean(axis=0)) ** 2).sum(axis=0)
        j = int(np.argmax(sse))          # first maximum = smallest index on ties
        split_dims.append(j)
        children = []
        for node, idx in enumerate(nodes):
            h = (2 ** t - 1) + node      # heap index of (level t, node)
            if len(idx) > 0:
                v = np.sort(X[idx, j])
                thr[h] = v[(len(v) - 1) // 2]
            else:
                thr[h] = thr[(h - 1) // 2]
            go_right = X[idx, j] > thr[h]
            children.append(idx[~go_right])   # child 2*node   (bit 0)
            children.append(idx[go_right])    # child 2*node+1 (bit 1)
        nodes = children
        levels.append(nodes)
    return split_dims, thr, levels


def prototypes(X: np.ndarray, levels) -> np.ndarray:
    """P0 rows = bucket means of the 16 leaves (reading R5: no Eq. 2 refit).

    An empty leaf takes the mean of its nearest non-empty ancestor (leaf k's ancestor at
    level t is node k >> (4 - t))."""
    X = np.asarray(X, dtype=np.float64)
    P = np.zeros((K, X.shape[1]), dtype=np.float64)
    for k in range(K):
        for t in range(LEVELS, -1, -1):
            idx = levels[t][k >> (LEVELS - t)]
            if len(idx) > 0:
                P[k] = X[idx].mean(axis=0)
                break
    return P


def build_lut(P: np.ndarray, Bsub: np.ndarray) -> np.ndarray:
    """T = P B restricted to the chunk: T[k][m] = sum_j P[k][j] B[j][m],
    fp64, j ascending, each product rounded then added (R-order pinned in DESIGN.md)."""
    T = np.zeros((P.shape[0], Bsub.shape[1]), dtype=np.float64)
    for j in range(P.shape[1]):
        T += np.outer(P[:, j], Bsub[j])
    return T


def quantize(T: np.ndarray):
    """8-bit LUT with per-output-column scale/offset ("8-bit block floating point";
    S:350-358; reading R6).  T: [C][16][M] fp64.  Per column m: lo = min, hi = max over (c,k);
    scale = (hi-lo)/255 (1 if hi = lo); q = clamp(floor((T-lo)/scale + 0.5), 0, 255)."""
    C, KK, M = T.shape
    q = np.zeros((C, KK, M), dtype=np.uint8)
    scale = np.zeros(M, dtype=np.float64)
    lo = np.zeros(M, dtype=np.float64)
    for m in range(M):
        col = T[:, :, m]
        lo[m] = col.min()
        hi = col.max()
        scale[m] = (hi - lo[m]) / 255.0 if hi > lo[m] else 1.0
        qm = np.floor((col - lo[m]) / scale[m] + 0.5)
        q[:, :, m] = np.clip(qm, 0, 255).astype(np.uint8)
    return q, scale, lo


def fit(A_train: np.ndarray, B: np.ndarray, C: int, perm: np.ndarray, bias: np.ndarray,
        a_is_bf16: bool = False) -> dict:
    """Fit one ITLUMM layer (MADDNESS inference structure, with ITLUMM's permutation
    applied first).  Returns the hot-path parameters plus fp64 intermediates."""
    A_train = np.asarray(A_train)
    if a_is_bf16:
        A_train = (A_train.astype(np.uint32) << 16).view(np.float32)
    A_train = A_train.astype(np.float32)
    D = A_train.shape[1]
    M = B.shape[1]
    perm = np.asarray(perm, dtype=np.int32)
    b = boundaries(D, C)
    Ap = A_train[:, perm]                       # a'[i] = a[perm[i]]  (reading R11)
    Bp = np.asarray(B, dtype=np.float64)[perm]  # rows of B follow the same permutation
    split_dim = np.zeros((C, LEVELS), dtype=np.int32)
    thresholds = np.zeros((C, 2 ** LEVELS - 1), dtype=np.float32)
    T = np.zeros((C, K, M), dtype=np.float64)
    P_all = []
    leaf_sizes = np.zeros((C, K), dtype=np.int64)
    for c in range(C):
        X = Ap[:, b[c]:b[c + 1]]
        sd, thr, levels = fit_tree(X)
        split_dim[c] = sd
        thresholds[c] = thr.astype(np.float32)   # a data value: exact in fp32 (R4)
        P = prototypes(X, levels)
        P_all.append(P)
        leaf_sizes[c] = [len(ix) for ix in levels[LEVELS]]
        T[c] = build_lut(P, Bp[b[c]:b[c + 1]])
    q, scale, lo = quantize(T)
    scale_f = scale.astype(np.float32)
    lo_f = lo.astype(np.float32)
    return dict(D=D, C=C, M=M, perm=perm, boundaries=b, split_dim=split_dim,
                thresholds=thresholds, lut=q, scale=scale_f, offset=lo_f,
                bias=np.asarray(bias, dtype=np.float32).copy(),
                T=T, scale64=scale, lo64=lo, prototypes=P_all, leaf_sizes=leaf_sizes)


def onehot(codes: np.ndarray) -> np.ndarray:
    """G: the concatenation of C one-hot 16-dimensional vectors per row, N x 16C, fp64."""
    N, C = codes.shape
    G = np.zeros((N, K * C), dtype=np.float64)
    for c in range(C):
        G[np.arange(N), K * c + codes[:, c].astype(np.int64)] = 1.0
    return G


def optimize_lut_linear(A: np.ndarray, B: np.ndarray, codes: np.ndarray, T0: np.ndarray, lam: float) -> np.ndarray:
    """ITLUMM model-aware LUT optimisation, Eq. 3, for sigma = the bias alone (no
    nonlinearity): argmin_T ||A B - G T||^2 + lam ||T - P0 B||^2 (the bias cancels inside the
    norm).  Normal equations (G^T G + lam I) T = G^T (A B) + lam P0 B, solved in fp64.
    A: N x D training rows, B: D x M, codes: N x C, T0 = P0 B as [C][16][M].  Returns [C][16][M]."""
    C = codes.shape[1]
    M = B.shape[1]
    G = onehot(codes)
    Y = np.asarray(A, np.float64) @ np.asarray(B, np.float64)
    T0f = np.asarray(T0, np.float64).reshape(K * C, M)
    lhs = G.T @ G + lam * np.eye(K * C)
    rhs = G.T @ Y + lam * T0f
    return np.linalg.solve(lhs, rhs).reshape(C, K, M)


def eq3_objective(A, B, bias, codes, T, T0, lam, relu: bool) -> float:
    """||sigma(A B) - sigma(G T)||^2 + lam ||T - P0 B||^2 with sigma = (+ bias) then ReLU if relu."""
    G = onehot(codes)
    C = codes.shape[1]
    M = B.shape[1]
    Y = np.asarray(A, np.float64) @ np.asarray(B, np.float64) + np.asarray(bias, np.float64)
    Z = G @ np.asarray(T, np.float64).reshape(K * C, M) + np.asarray(bias, np.float64)
    if relu:
        Y, Z = np.maximum(Y, 0), np.maximum(Z, 0)
    return float(((Y - Z) ** 2).sum() + lam * ((np.asarray(T) - np.asarray(T0)) ** 2).sum())


def softmax_rows(Z: np.ndarray) -> np.ndarray:
    """Row-wise softmax, fp64, max-shifted ("a row-wise nonlinearity ... such as softmax")."""
    Z = np.asarray(Z, np.float64)
    E = np.exp(Z - Z.max(axis=1, keepdims=True))
    return E / E.sum(axis=1, keepdims=True)


def eq3_objective_kld(A, B, bias, codes, T, T0, lam) -> float:
    """Eq. 3 with the KL-divergence first term the paper prefers:
    sum over rows of KL(softmax(a B + bias) || softmax(g T + bias)) + lam ||T - P0 B||^2, fp64.
    KL(p || q) = sum_m p_m (log p_m - log q_m), logs from log-softmax (x - max - log sum exp)."""
    G = onehot(codes)
    C = codes.shape[1]
    M = B.shape[1]
    Y = np.asarray(A, np.float64) @ np.asarray(B, np.float64) + np.asarray(bias, np.float64)
    Z = G @ np.asarray(T, np.float64).reshape(K * C, M) + np.asarray(bias, np.float64)

    def log_softmax(X):
        Xs = X - X.max(axis=1, keepdims=True)
        return Xs - np.log(np.exp(Xs).sum(axis=1, keepdims=True))
    lp, lq = log_softmax(Y), log_softmax(Z)
    kl = float((np.exp(lp) * (lp - lq)).sum())
    return kl + lam * float(((np.asarray(T, np.float64) - np.asarray(T0, np.float64)) ** 2).sum())


def eq3_kld_grad(A, B, bias, codes, T, T0, lam) -> np.ndarray:
    """Analytic gradient of eq3_objective_kld in T: with p = softmax(Y), q = softmax(Z), Z = G T + bias,
    d/dZ KL(p || q) = q - p per row, so dJ/dT = G^T (q - p) + 2 lam (T - T0); [C][16][M]."""
    G = onehot(codes)
    C = codes.shape[1]
    M = B.shape[1]
    Y = np.asarray(A, np.float64) @ np.asarray(B, np.float64) + np.asarray(bias, np.float64)
    Z = G @ np.asarray(T, np.float64).reshape(K * C, M) + np.asarray(bias, np.float64)
    g = G.T @ (softmax_rows(Z) - softmax_rows(Y))
    return g.reshape(C, K, M) + 2.0 * lam * (np.asarray(T, np.float64) - np.asarray(T0, np.float64))


def optimize_lut_kld(A, B, bias, codes, T0, lam, steps: int, lr: float) -> np.ndarray:
    """Eq. 3 with the KLD objective minimised by plain gradient descent from T = P0 B (the paper gives
    no optimiser; reading R23 in DESIGN.md): `steps` updates T <- T - lr * eq3_kld_grad(T), fp64."""
    T = np.asarray(T0, np.float64).copy()
    for _ in range(int(steps)):
        T = T - lr * eq3_kld_grad(A, B, bias, codes, T, T0, lam)
    return T


def requantize(params: dict, T: np.ndarray) -> dict:
    """Same trees, LUT from table T through the same uint8 quantiser (reading R6)."""
    q, scale, lo = quantize(np.asarray(T, np.float64))
    out = dict(params)
    out.update(lut=q, scale=scale.astype(np.float32), offset=lo.astype(np.float32), T=np.asarray(T, np.float64),
               scale64=scale, lo64=lo)
    return out
