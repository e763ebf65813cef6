"""The product's offline fitter (paper_2207_05808_b200.fit) reproduces the oracle's fit bit for
bit: same split dims, thresholds, uint8 LUT, scale and offset (readings R3-R6, R12)."""
import numpy as np
import pytest

import synth
from oracle import fit as ofit
from paper_2207_05808_b200 import fit as pfit
from tests.test_oracle_pins import exact_pq_case

KEYS = ["perm", "boundaries", "split_dim", "thresholds", "lut", "scale", "offset", "bias"]


def same(a, b):
    for k in KEYS:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        assert x.dtype == y.dtype and x.shape == y.shape, k
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), k


def test_chunk_bounds_match_oracle():
    for D, C in [(784, 16), (784, 32), (3072, 64), (4096, 256), (10, 3), (9, 9)]:
        assert np.array_equal(pfit.chunk_bounds(D, C), ofit.boundaries(D, C))


@pytest.mark.parametrize("seed,N,D,M,C,dtype", [(1, 64, 64, 24, 8, "f32"), (2, 64, 97, 33, 10, "f32"),
                                                (3, 64, 96, 40, 12, "bf16"), (4, 64, 50, 5, 50, "f32")])
def test_fit_matches_oracle_small(seed, N, D, M, C, dtype):
    w = synth.small_case(seed, N=N, D=D, M=M, C=C, dtype=dtype, n_train=700)
    bf = dtype == "bf16"
    a = ofit.fit(w["A_train"], w["B"], C, w["perm"], w["bias"], a_is_bf16=bf)
    b = pfit.fit_layer(w["A_train"], w["B"], C, w["perm"], w["bias"], a_is_bf16=bf)
    same(a, b)


def test_fit_matches_oracle_cfg1():
    w = synth.workload("cfg1", n_rows=10)
    a = ofit.fit(w["A_train"], w["B"], w["C"], w["perm"], w["bias"])
    b = pfit.fit_layer(w["A_train"], w["B"], w["C"], w["perm"], w["bias"])
    same(a, b)


def test_fit_matches_oracle_exact_pq_and_degenerate():
    A_train, _, _, B, bias = exact_pq_case(C=5, M=7)
    same(ofit.fit(A_train, B, 5, np.arange(20), bias), pfit.fit_layer(A_train, B, 5, np.arange(20), bias))
    X = np.zeros((40, 12), np.float32)        # constant data: empty nodes everywhere
    X[:20, 3] = 1.0
    B = np.random.default_rng(0).normal(size=(12, 4))
    same(ofit.fit(X, B, 3, np.arange(12), np.zeros(4)), pfit.fit_layer(X, B, 3, np.arange(12), np.zeros(4)))
