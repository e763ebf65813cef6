"""Seeded synthetic workloads for the ITLUMM hot path (SURVEY.md §8(d) "Synthetic inputs").

This module is shared by the oracle (``oracle/``), the tests and ``bench.py``.  It holds
NO arithmetic of the method: no partitioning rule, no tree fit, no LUT, no quantisation,
no encode/accumulate/dequant.  It only draws the raw inputs a deployment would hand to the
method: activations A (test rows and a training sample), the fixed weight matrix B, the
stand-in permutation of D (the paper learns it, P:62/P:76/P:83; here it is a seeded
random bijection, reading R21 in DESIGN.md), and the bias.

Stand-ins (no dataset is in the container):
  * "mnist": U[0,1) pixels, each entry zeroed with p = 0.2          (BASELINE.json configs[0], [1])
  * "cifar": clip(0.47 + 0.25 z, 0, 1), z ~ N(0,1), all planes alike (configs[2], [3])
  * "ffn":   z ~ N(0,1), 1% of the columns (41 of 4096) scaled x8, rounded to bf16 (RNE)
             (configs[4])
Seeds: numpy ``default_rng([220705808, cfg, stream, chunk])``; stream 0 = A_test,
1 = A_train, 2 = B (+10*layer), 3 = perm (+10*layer), 4 = bias, 5 = outlier columns;
chunk = 65536-row block index, so a row shard generates its rows independently of the
number of ranks.
"""
from __future__ import annotations

import numpy as np

SEED = 220705808
CHUNK_ROWS = 65536


def rng(cfg: int, stream: int, chunk: int = 0) -> np.random.Generator:
    return np.random.default_rng([SEED, int(cfg), int(stream), int(chunk)])


# ----------------------------------------------------------------------------- configs
# Shapes from BASELINE.json "configs"; the `name` keys are what bench/tests pass around.
CONFIGS = {
    # configs[0]: MNIST-shaped final layer
    "cfg1": dict(cfg=1, N=1000, D=784, M=10, C=16, dist="mnist", n_train=5000,
                 perm="identity", relu=False, b_var=1.0 / 784, dtype="f32"),
    # configs[1]: MNIST-shaped hidden layer with the permutation of D, ReLU fused
    "cfg2": dict(cfg=2, N=60000, D=784, M=512, C=32, dist="mnist", n_train=5000,
                 perm="seeded", relu=True, b_var=2.0 / 784, dtype="f32"),
    # configs[2]: CIFAR-shaped layer, C = 64 and C = 128
    "cfg3_c64": dict(cfg=3, N=50000, D=3072, M=1024, C=64, dist="cifar", n_train=10000,
                     perm="seeded", relu=False, b_var=2.0 / 3072, dtype="f32"),
    "cfg3_c128": dict(cfg=3, N=50000, D=3072, M=1024, C=128, dist="cifar", n_train=10000,
                      perm="seeded", relu=False, b_var=2.0 / 3072, dtype="f32"),
    # configs[4]: transformer-FFN-shaped stress case, bf16 input
    "cfg5": dict(cfg=5, N=262144, D=4096, M=4096, C=256, dist="ffn", n_train=16384,
                 perm="seeded", relu=False, b_var=1.0 / 4096, dtype="bf16"),
}

# configs[3]: 3-layer ReLU MLP 3072-1024-1024-10, every layer replaced (C swept).
MLP_LAYERS = [(3072, 1024, True), (1024, 1024, True), (1024, 10, False)]
MLP_CFG = dict(cfg=4, N=1048576, dist="cifar", n_train=16384, C_sweep=(16, 32, 64, 128, 256))


# ----------------------------------------------------------------------------- rows
def _f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns (data recipe)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return b.astype(np.uint16)


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns to fp32 (used to look at bf16 data on the host)."""
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def outlier_columns(cfg: int, D: int) -> np.ndarray:
    n_out = max(1, int(round(0.01 * D)))
    return np.sort(rng(cfg, 5).choice(D, n_out, replace=False))


SUB_ROWS = 1024  # rows are drawn in fixed sub-blocks so that any prefix of a chunk is stable


def _draw(dist: str, cfg: int, g: np.random.Generator, n: int, D: int) -> np.ndarray:
    """n rows from generator g, drawn SUB_ROWS at a time (prefix-stable in n)."""
    out = [_draw_block(dist, cfg, g, SUB_ROWS, D) for _ in range(0, n, SUB_ROWS)]
    dt = np.uint16 if dist == "ffn" else np.float32
    return np.concatenate(out, axis=0)[:n] if out else np.zeros((0, D), dtype=dt)


def _draw_block(dist: str, cfg: int, g: np.random.Generator, n: int, D: int) -> np.ndarray:
    if dist == "mnist":
        x = g.random((n, D), dtype=np.float32)
        x[g.random((n, D), dtype=np.float32) < 0.2] = 0.0
        return x
    if dist == "cifar":
        z = g.standard_normal((n, D), dtype=np.float32)
        return np.clip(np.float32(0.47) + np.float32(0.25) * z, 0.0, 1.0).astype(np.float32)
    if dist == "ffn":
        z = g.standard_normal((n, D), dtype=np.float32)
        z[:, outlier_columns(cfg, D)] *= np.float32(8.0)
        return _f32_to_bf16_bits(z)
    raise ValueError(f"unknown dist {dist!r}")


def rows(dist: str, cfg: int, stream: int, r0: int, r1: int, D: int) -> np.ndarray:
    """Rows [r0, r1) of the (cfg, stream) row sequence, generated chunk by chunk.

    fp32 for "mnist"/"cifar", uint16 bf16 bit patterns for "ffn"."""
    if r1 <= r0:
        dt = np.uint16 if dist == "ffn" else np.float32
        return np.zeros((0, D), dtype=dt)
    parts = []
    for ch in range(r0 // CHUNK_ROWS, (r1 - 1) // CHUNK_ROWS + 1):
        lo, hi = ch * CHUNK_ROWS, (ch + 1) * CHUNK_ROWS
        a, b = max(lo, r0), min(hi, r1)
        n_need = b - lo  # generate the chunk prefix up to b (prefix-stable per chunk)
        blk = _draw(dist, cfg, rng(cfg, stream, ch), n_need, D)
        parts.append(blk[a - lo:b - lo])
    return np.ascontiguousarray(np.concatenate(parts, axis=0))


def weights(cfg: int, D: int, M: int, var: float, layer: int = 0) -> np.ndarray:
    """B: D x M, N(0, var) in fp64 (kept fp64 for the offline LUT build)."""
    return rng(cfg, 2 + 10 * layer).normal(0.0, np.sqrt(var), size=(D, M))


def permutation(cfg: int, D: int, kind: str, layer: int = 0) -> np.ndarray:
    """Stand-in for the learned permutation of the D input dims (gather: a'[i] = a[perm[i]])."""
    if kind == "identity":
        return np.arange(D, dtype=np.int32)
    return rng(cfg, 3 + 10 * layer).permutation(D).astype(np.int32)


def bias(cfg: int, M: int, kind: str = "zero", layer: int = 0) -> np.ndarray:
    """Benchmark configs use bias = 0; parity suites use N(0, 0.1^2) (reading R15)."""
    if kind == "zero":
        return np.zeros(M, dtype=np.float32)
    return rng(cfg, 4 + 10 * layer).normal(0.0, 0.1, size=M).astype(np.float32)


def workload(name: str, n_rows: int | None = None, row0: int = 0, bias_kind: str = "zero",
             n_train: int | None = None) -> dict:
    """Everything a config needs: A (test rows [row0, row0+n)), A_train, B, perm, bias."""
    c = CONFIGS[name]
    n = c["N"] if n_rows is None else int(n_rows)
    nt = c["n_train"] if n_train is None else int(n_train)
    return dict(
        name=name, cfg=c["cfg"], D=c["D"], M=c["M"], C=c["C"], relu=c["relu"], dtype=c["dtype"],
        A=rows(c["dist"], c["cfg"], 0, row0, row0 + n, c["D"]),
        A_train=rows(c["dist"], c["cfg"], 1, 0, nt, c["D"]),
        B=weights(c["cfg"], c["D"], c["M"], c["b_var"]),
        perm=permutation(c["cfg"], c["D"], c["perm"]),
        bias=bias(c["cfg"], c["M"], bias_kind),
    )


def small_case(seed: int, N: int, D: int, M: int, C: int, dist: str = "mnist",
               n_train: int = 512, dtype: str = "f32", bias_kind: str = "normal") -> dict:
    """Small random cases for parity/property tests (cfg id 100+seed keeps streams apart)."""
    cfg = 100 + int(seed)
    d = "ffn" if dtype == "bf16" else dist
    return dict(
        name=f"small{seed}", cfg=cfg, D=D, M=M, C=C, relu=bool(seed % 2), dtype=dtype,
        A=rows(d, cfg, 0, 0, N, D), A_train=rows(d, cfg, 1, 0, n_train, D),
        B=weights(cfg, D, M, 2.0 / D), perm=permutation(cfg, D, "seeded"),
        bias=bias(cfg, M, bias_kind),
    )


def mlp_workload(C: int, n_rows: int, n_train: int | None = None, row0: int = 0,
                 layers=MLP_LAYERS, cfg: int = MLP_CFG["cfg"], dist: str = MLP_CFG["dist"]) -> dict:
    """BASELINE configs[3]: 3-layer ReLU MLP 3072-1024-1024-10, CIFAR-shaped input, one seeded
    permutation and B ~ N(0, 2/D_in) per layer (streams 2+10l, 3+10l), bias 0, C per layer."""
    nt = MLP_CFG["n_train"] if n_train is None else int(n_train)
    D0 = layers[0][0]
    return dict(
        A=rows(dist, cfg, 0, row0, row0 + n_rows, D0), A_train=rows(dist, cfg, 1, 0, nt, D0),
        Bs=[weights(cfg, d, m, 2.0 / d, layer=l) for l, (d, m, _) in enumerate(layers)],
        perms=[permutation(cfg, d, "seeded", layer=l) for l, (d, _, _) in enumerate(layers)],
        biases=[bias(cfg, m, "zero", layer=l) for l, (_, m, _) in enumerate(layers)],
        relus=[r for (_, _, r) in layers], Cs=[int(C)] * len(layers))
