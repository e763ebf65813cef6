"""Pins for the oracle (-m "not gpu"): each test fixes part of oracle/ against something other
than itself — a worked example printed in SPEC.md, a closed form, a library routine that the
special case reduces to, brute force, or an invariant the paper states."""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle import fit as ofit

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def params_from(D, C, M, split_dim, thr, lut, perm=None, bnd=None, scale=None, offset=None,
                bias=None):
    return dict(D=D, C=C, M=M,
                perm=np.arange(D, dtype=np.int32) if perm is None else np.asarray(perm, np.int32),
                boundaries=ofit.boundaries(D, C) if bnd is None else np.asarray(bnd, np.int32),
                split_dim=np.asarray(split_dim, np.int32).reshape(C, 4),
                thresholds=np.asarray(thr, np.float32).reshape(C, 15),
                lut=np.asarray(lut, np.uint8).reshape(C, 16, M),
                scale=np.ones(M, np.float32) if scale is None else np.asarray(scale, np.float32),
                offset=np.zeros(M, np.float32) if offset is None else np.asarray(offset, np.float32),
                bias=np.zeros(M, np.float32) if bias is None else np.asarray(bias, np.float32))


def identity_lut(C=1):
    """q[c][k][0] = k: the accumulator then exposes the code sum."""
    lut = np.zeros((C, 16, 1), np.uint8)
    lut[:, :, 0] = np.arange(16)
    return lut


def read_golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                rows.append([p.strip() for p in line.split("|")])
    return rows


# ---------------------------------------------------------------------------- a2: encode
def test_encode_golden_worked_examples():
    """SPEC S:258-260 (golden file): +inf -> 0, -inf -> 15, hand-traced 1-D tree v=5.5 -> 5."""
    for name, thr, v, want in read_golden("encode_s258_s260.txt"):
        thr = np.array([float(x) for x in thr.split()], np.float32)
        p = params_from(1, 1, 1, [0, 0, 0, 0], thr, identity_lut())
        out = oracle.amm(p, np.array([[float(v)]], np.float32), relu=False, want_codes=True,
                         want_acc=True)
        assert int(out["codes"][0, 0]) == int(want), name
        assert int(out["acc"][0, 0]) == int(want), name


def bst_thresholds(s):
    """Heap-ordered thresholds of the balanced BST over sorted s_1..s_15."""
    thr = []
    for t in range(4):
        for n in range(2 ** t):
            thr.append(s[(2 * n + 1) * (2 ** (3 - t)) - 1])
    return np.array(thr, np.float32)


def test_encode_reduces_to_searchsorted():
    """Same split dim at all 4 levels + BST thresholds -> code = searchsorted(s, v, 'left')
    (number of thresholds strictly below v), ties included.  Occurs in cfg5 outlier dims."""
    g = np.random.default_rng(7)
    for trial in range(200):
        s = np.sort(g.choice(np.arange(-20, 21), 15, replace=True).astype(np.float32) / 4)
        v = np.concatenate([s, g.uniform(-6, 6, 20).astype(np.float32),
                            np.array([np.inf, -np.inf], np.float32)]).reshape(-1, 1)
        p = params_from(1, 1, 1, [0, 0, 0, 0], bst_thresholds(s), identity_lut())
        codes = oracle.amm(p, v, relu=False, want_codes=True, want_y=False)["codes"][:, 0]
        assert np.array_equal(codes, np.searchsorted(s, v[:, 0], side="left"))


class _Node:
    def __init__(self, dim, thr, left=None, right=None, leaf=None):
        self.dim, self.thr, self.left, self.right, self.leaf = dim, thr, left, right, leaf


def _build_explicit(split_dim, thr, t=0, n=0):
    """Explicit node objects (no heap arithmetic) for the recursive brute force."""
    if t == 4:
        return _Node(None, None, leaf=n)
    h = (2 ** t - 1) + n
    return _Node(split_dim[t], thr[h], _build_explicit(split_dim, thr, t + 1, 2 * n),
                 _build_explicit(split_dim, thr, t + 1, 2 * n + 1))


def _walk(node, x):
    if node.leaf is not None:
        return node.leaf
    return _walk(node.right if x[node.dim] > node.thr else node.left, x)


def test_encode_random_trees_vs_recursive_traversal():
    """Random trees, permutation and ragged chunks vs an explicit recursive traversal of the
    literally permuted and sliced row (BASELINE north_star: brute-force tree traversal)."""
    g = np.random.default_rng(11)
    for trial in range(12):
        D = int(g.integers(8, 60))
        C = int(g.integers(1, min(D, 9) + 1))
        bnd = ofit.boundaries(D, C)
        perm = g.permutation(D).astype(np.int32)
        sd = np.stack([g.integers(0, bnd[c + 1] - bnd[c], 4) for c in range(C)]).astype(np.int32)
        thr = g.normal(size=(C, 15)).astype(np.float32)
        thr[g.random((C, 15)) < 0.05] = np.inf
        A = g.normal(size=(50, D)).astype(np.float32)
        A[:, :3] = np.round(A[:, :3])               # exercise ties with integer thresholds
        thr[:, :2] = np.round(thr[:, :2])
        A[0, 0] = np.nan                            # NaN compares false -> left (reading R10)
        p = params_from(D, C, 1, sd, thr, np.zeros((C, 16, 1)), perm=perm)
        codes = oracle.amm(p, A, relu=False, want_codes=True, want_y=False)["codes"]
        for r in range(A.shape[0]):
            ap = A[r][perm]
            for c in range(C):
                tree = _build_explicit(sd[c], thr[c])
                assert codes[r, c] == _walk(tree, ap[bnd[c]:bnd[c + 1]])
        assert codes.max() < 16


# ---------------------------------------------------------------------------- a1: partition
def test_partition_invariants():
    """Chunks are contiguous, cover D once, sizes differ by <= 1, larger first;
    the synthetic permutation is a bijection."""
    for D, C in [(784, 16), (784, 32), (3072, 128), (4096, 256), (7, 7), (10, 3), (5, 1)]:
        b = ofit.boundaries(D, C)
        sizes = np.diff(b)
        assert b[0] == 0 and b[-1] == D and len(b) == C + 1
        assert sizes.max() - sizes.min() <= 1 and np.all(np.diff(sizes) <= 0)
    assert np.array_equal(np.diff(ofit.boundaries(784, 32))[[0, 15, 16, 31]], [25, 25, 24, 24])
    p = synth.permutation(2, 784, "seeded")
    assert np.array_equal(np.sort(p), np.arange(784))
    with pytest.raises(ValueError):
        ofit.boundaries(4, 5)


def test_folded_gather_equals_literal_permute_and_slice():
    """col[c][t] = perm[b_c + split_dim[c][t]] reads the same value as permute-then-slice
    (the identity the GPU plan relies on)."""
    g = np.random.default_rng(3)
    D, C = 97, 10
    perm = g.permutation(D)
    b = ofit.boundaries(D, C)
    sd = np.stack([g.integers(0, b[c + 1] - b[c], 4) for c in range(C)])
    A = g.normal(size=(20, D))
    for c in range(C):
        for t in range(4):
            col = perm[b[c] + sd[c, t]]
            assert np.array_equal(A[:, col], A[:, perm][:, b[c]:b[c + 1]][:, sd[c, t]])


# ---------------------------------------------------------------------------- tree fit
def test_tree_fit_invariants_and_rule():
    """Leaves partition the sample; within-leaf SSE non-increasing per level;
    split dim maximises pooled within-node SSE (computed here as n*var); thresholds are lower
    medians (data values) of their node; empty nodes copy the parent threshold."""
    g = np.random.default_rng(5)
    X = g.normal(size=(300, 9)) * np.array([1, 3, 2, 0.5, 1, 1, 4, 1, 0.1])
    X[:40, 2] = 0.0
    sd, thr, levels = ofit.fit_tree(X)
    assert sum(len(ix) for ix in levels[4]) == 300
    assert np.array_equal(np.sort(np.concatenate(levels[4])), np.arange(300))
    prev = np.inf
    for t in range(5):
        sse = sum(((X[ix] - X[ix].mean(0)) ** 2).sum() for ix in levels[t] if len(ix))
        assert sse <= prev + 1e-9
        prev = sse
    for t in range(4):
        pooled = np.zeros(9)
        for ix in levels[t]:
            if len(ix):
                pooled += len(ix) * X[ix].var(axis=0)
        assert pooled[sd[t]] >= pooled.max() * (1 - 1e-12)
        for n, ix in enumerate(levels[t]):
            h = 2 ** t - 1 + n
            if len(ix):
                v = np.sort(X[ix, sd[t]])
                assert thr[h] == v[(len(v) - 1) // 2]
                assert np.sum(X[ix, sd[t]] <= thr[h]) >= (len(v) + 1) // 2
            else:
                assert thr[h] == thr[(h - 1) // 2]


def test_tree_fit_empty_nodes():
    """Constant data: every threshold equals the constant, all rows go left (S:239 example),
    empty right nodes copy the parent threshold, SSE = 0; prototypes of empty leaves fall
    back to the nearest non-empty ancestor's mean."""
    X = np.full((40, 3), 2.5)
    sd, thr, levels = ofit.fit_tree(X)
    assert np.all(thr == 2.5) and sd == [0, 0, 0, 0]
    assert len(levels[4][0]) == 40 and all(len(ix) == 0 for ix in levels[4][1:])
    P = ofit.prototypes(X, levels)
    assert np.all(P == 2.5)


# ---------------------------------------------------------------------------- LUT + quantise
def test_lut_special_cases():
    """B = 0 -> zero table; identity prototypes -> T = rows of B; random P, B vs a
    direct per-entry inner product in exact rational arithmetic (rounded once)."""
    g = np.random.default_rng(1)
    P = g.normal(size=(16, 5))
    assert np.all(ofit.build_lut(P, np.zeros((5, 7))) == 0)
    B = g.normal(size=(16, 7))
    assert np.array_equal(ofit.build_lut(np.eye(16), B), B)
    Bs = g.normal(size=(5, 3))
    T = ofit.build_lut(P, Bs)
    for k in range(16):
        for m in range(3):
            # j ascending, each product rounded to fp64 then added with one rounding: simulated
            # in exact rationals (float(Fraction) is correctly rounded)
            acc = 0.0
            for j in range(5):
                acc = float(Fraction(acc) + Fraction(float(Fraction(P[k, j]) * Fraction(Bs[j, m]))))
            assert T[k, m] == acc
            exact = sum(Fraction(P[k, j]) * Fraction(Bs[j, m]) for j in range(5))
            bound = 6 * 2.0 ** -53 * sum(abs(P[k, j] * Bs[j, m]) for j in range(5))
            assert abs(float(Fraction(T[k, m]) - exact)) <= bound


def test_quantize_golden_examples():
    """SPEC S:355-357 (golden file): constant table and {0,255} table."""
    for name, vals, scale, q in read_golden("quantize_s356_s357.txt"):
        T = np.array([float(x) for x in vals.split()]).reshape(1, 16, 1)
        qq, sc, lo = ofit.quantize(T)
        assert sc[0] == float(scale), name
        assert np.array_equal(qq[0, :, 0], [int(x) for x in q.split()]), name
        assert np.array_equal(qq[0, :, 0] * sc[0] + lo[0], T[0, :, 0]), name


def test_quantize_ties_round_half_up():
    """Reading R6 at exact .5 ties (golden file tests/golden/quantize_ties_r6.txt): the
    quantiser rounds half UP, so half-to-even or truncation would fail here."""
    for name, vals, scale, q in read_golden("quantize_ties_r6.txt"):
        T = np.array([float(x) for x in vals.split()]).reshape(1, 16, 1)
        qq, sc, lo = ofit.quantize(T)
        assert sc[0] == float(scale), name
        assert np.array_equal(qq[0, :, 0], [int(x) for x in q.split()]), name


def test_quantize_error_bound():
    """|q*scale + lo - T| <= scale/2 elementwise; q uses the full [0,255] range."""
    g = np.random.default_rng(2)
    for trial in range(100):
        T = g.normal(size=(int(g.integers(1, 9)), 16, int(g.integers(1, 6)))) * g.uniform(0.01, 10)
        q, sc, lo = ofit.quantize(T)
        err = np.abs(q * sc + lo - T)
        assert np.all(err <= sc / 2 * (1 + 1e-9))
        assert np.all(q.reshape(-1, T.shape[2]).min(0) == 0)
        assert np.all(q.reshape(-1, T.shape[2]).max(0) == 255)


# ---------------------------------------------------------------------------- a3 + a4
def _random_params(g, D, C, M):
    b = ofit.boundaries(D, C)
    sd = np.stack([g.integers(0, b[c + 1] - b[c], 4) for c in range(C)])
    thr = g.uniform(0.2, 0.8, size=(C, 15))
    lut = g.integers(0, 256, size=(C, 16, M))
    return params_from(D, C, M, sd, thr, lut, perm=g.permutation(D),
                       scale=g.uniform(1e-3, 1e-2, M), offset=g.normal(size=M) * 0.1,
                       bias=g.normal(size=M) * 0.1)


def test_accumulate_equals_onehot_matmul():
    """acc = G q with G the concatenation of C one-hot 16-vectors: exact int64
    matrix product by numpy."""
    g = np.random.default_rng(4)
    D, C, M = 70, 9, 13
    p = _random_params(g, D, C, M)
    A = g.random((64, D)).astype(np.float32)
    out = oracle.amm(p, A, relu=False, want_codes=True, want_acc=True)
    G = np.zeros((64, 16 * C), np.int64)
    for c in range(C):
        G[np.arange(64), 16 * c + out["codes"][:, c]] = 1
    assert np.array_equal(out["acc"], G @ p["lut"].reshape(16 * C, M).astype(np.int64))


def test_accumulate_n1_c1_and_reordering():
    """N=1, C=1, code k -> the LUT row k; permuting codebook order (with the chunks)
    leaves the integer sums unchanged (S:393 associativity)."""
    g = np.random.default_rng(6)
    lut = g.integers(0, 256, size=(1, 16, 5))
    thr = bst_thresholds(np.arange(1, 16, dtype=np.float32))
    p = params_from(1, 1, 5, [0] * 4, thr, lut)
    for k in range(16):
        acc = oracle.amm(p, np.array([[k + 0.5]], np.float32), relu=False, want_acc=True)["acc"]
        assert np.array_equal(acc[0], lut[0, k])
    D, C, M = 48, 6, 7
    p = _random_params(g, D, C, M)
    A = g.random((30, D)).astype(np.float32)
    acc1 = oracle.amm(p, A, relu=False, want_acc=True)["acc"]
    order = g.permutation(C)
    b = p["boundaries"]
    new_perm = np.concatenate([p["perm"][b[c]:b[c + 1]] for c in order])
    sizes = np.diff(b)[order]
    p2 = dict(p, perm=new_perm, boundaries=np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32),
              split_dim=p["split_dim"][order], thresholds=p["thresholds"][order], lut=p["lut"][order])
    assert np.array_equal(oracle.amm(p2, A, relu=False, want_acc=True)["acc"], acc1)


def _round_f32(fr: Fraction) -> float:
    """Round an exact rational to the nearest fp32 (ties to even) via exact comparison."""
    x = np.float32(float(fr))  # double rounding candidate, then fix by exact comparison
    lo_ = np.nextafter(x, np.float32(-np.inf))
    hi_ = np.nextafter(x, np.float32(np.inf))
    best = min([lo_, x, hi_], key=lambda c: (abs(Fraction(float(c)) - fr),
                                           int(np.array(c, np.float32).view(np.uint32)) & 1))
    return float(best)


def test_dequant_is_one_rounding_of_exact_value():
    """y = fma(scale, acc, offtot) rounds the exact scale*acc + offtot once (reading R8), with
    offtot = fp32(C*lo + bias); ReLU gives +0 for y <= 0 (reading R9)."""
    g = np.random.default_rng(8)
    D, C, M = 40, 5, 64
    p = _random_params(g, D, C, M)
    A = g.random((16, D)).astype(np.float32)
    out = oracle.amm(p, A, relu=False, want_acc=True)
    offtot = (C * p["offset"].astype(np.float64) + p["bias"].astype(np.float64)).astype(np.float32)
    for r in range(16):
        for m in range(M):
            exact = Fraction(float(p["scale"][m])) * int(out["acc"][r, m]) + Fraction(float(offtot[m]))
            assert out["y"][r, m] == _round_f32(exact)
    yr = oracle.amm(p, A, relu=True)["y"]
    assert np.array_equal(yr, np.where(out["y"] > 0, out["y"], np.float32(0)))
    assert not np.any(np.signbit(yr))


def test_row_parallel_bit_identity_and_bf16_widening():
    """Row-parallel execution is bit-identical to sequential; bf16 input gives
    the same result as its exact fp32 widening (reading R13)."""
    w = synth.small_case(3, N=300, D=96, M=40, C=12, dtype="bf16")
    p = ofit.fit(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=True)
    o1 = oracle.amm(p, w["A"], relu=True, dtype="bf16", want_codes=True, nthreads=1)
    o4 = oracle.amm(p, w["A"], relu=True, dtype="bf16", want_codes=True, nthreads=4)
    assert np.array_equal(o1["y"], o4["y"]) and np.array_equal(o1["codes"], o4["codes"])
    of = oracle.amm(p, synth.bf16_bits_to_f32(w["A"]), relu=True, want_codes=True)
    assert np.array_equal(o1["y"].view(np.uint32), of["y"].view(np.uint32))


# ---------------------------------------------------------------------------- end to end
def exact_pq_case(C=6, M=9, n_rep=8, seed=0):
    """Every 4-dim chunk holds the 16 patterns {0,1}^4 equally often; rows equal prototypes."""
    g = np.random.default_rng(seed)
    pats = np.array([[(k >> (3 - i)) & 1 for i in range(4)] for k in range(16)], np.float32)
    D = 4 * C
    kk = np.stack([g.permutation(np.repeat(np.arange(16), n_rep)) for _ in range(C)], axis=1)
    A_train = np.concatenate([pats[kk[:, c]] for c in range(C)], axis=1)
    kt = g.integers(0, 16, size=(40, C))
    A_test = np.concatenate([pats[kt[:, c]] for c in range(C)], axis=1)
    B = g.normal(size=(D, M))
    bias = g.normal(size=M).astype(np.float32) * 0.1
    return A_train, A_test, kt, B, bias


def test_exact_pq_end_to_end():
    """BASELINE north_star / S:366: when every chunk holds exactly 16 distinct patterns
    and rows equal prototypes, the fit reproduces them (split dims 0..3, thresholds 0, code =
    pattern index, P = patterns, T = P B) and y matches a.B + bias up to LUT quantisation:
    |y - (aB + bias)| <= C*scale/2 (+ fp32 rounding)."""
    C, M = 6, 9
    A_train, A_test, kt, B, bias = exact_pq_case(C, M)
    p = ofit.fit(A_train, B, C, np.arange(4 * C), bias)
    assert np.array_equal(p["split_dim"], np.tile([0, 1, 2, 3], (C, 1)))
    assert np.all(p["thresholds"] == 0)
    out = oracle.amm(p, A_test, relu=False, want_codes=True)
    assert np.array_equal(out["codes"], kt)
    exact = A_test.astype(np.float64) @ B + bias.astype(np.float64)
    bound = C * p["scale64"] / 2 + 1e-5 * (1 + np.abs(exact))
    assert np.all(np.abs(out["y"] - exact) <= bound)
    assert np.abs(out["y"] - exact).max() > 0  # quantisation is actually exercised


def test_exact_pq_end_to_end_shuffled_permutation():
    """Exact PQ through a NON-identity permutation (P:62 a'[i] = a[perm[i]], reading R11): the
    patterns live in the permuted coordinates, the raw rows scatter them (a[perm] = a'), and B
    stays in the raw coordinates.  The fit must build chunk c's LUT from the rows B[perm[b_c:b_c+1]],
    so y matches a.B + bias within C*scale/2; a LUT built from the unpermuted rows
    B[b_c:b_c+1] misses that bound (checked, so this test can tell the two apart)."""
    C, M = 6, 9
    Ap_train, Ap_test, kt, B, bias = exact_pq_case(C, M, seed=3)
    D = 4 * C
    perm = np.random.default_rng(11).permutation(D)
    assert not np.array_equal(perm, np.arange(D))
    A_train = np.zeros_like(Ap_train)
    A_train[:, perm] = Ap_train
    A_test = np.zeros_like(Ap_test)
    A_test[:, perm] = Ap_test
    p = ofit.fit(A_train, B, C, perm, bias)
    assert np.array_equal(p["split_dim"], np.tile([0, 1, 2, 3], (C, 1)))
    assert np.all(p["thresholds"] == 0)
    out = oracle.amm(p, A_test, relu=False, want_codes=True)
    assert np.array_equal(out["codes"], kt)
    exact = A_test.astype(np.float64) @ B + bias.astype(np.float64)
    bound = C * p["scale64"] / 2 + 1e-5 * (1 + np.abs(exact))
    assert np.all(np.abs(out["y"] - exact) <= bound)
    # the misreading (LUT from unpermuted rows of B) is far outside the bound
    b = p["boundaries"]
    wrong = sum(p["prototypes"][c][kt[:, c]] @ B[b[c]:b[c + 1]] for c in range(C)) + bias
    assert np.any(np.abs(wrong - exact) > bound)


def test_fit_lut_size_and_code_range_invariants():
    """LUT = 16*C*M bytes; codes in [0,16); leaf sizes sum to n_train (BASELINE)."""
    w = synth.small_case(1, N=200, D=64, M=24, C=8)
    p = ofit.fit(w["A_train"], w["B"], w["C"], w["perm"], w["bias"])
    assert p["lut"].nbytes == 16 * 8 * 24 and p["lut"].dtype == np.uint8
    assert np.all(p["leaf_sizes"].sum(axis=1) == w["A_train"].shape[0])
    codes = oracle.amm(p, w["A"], relu=False, want_codes=True)["codes"]
    assert codes.max() < 16
    # quantised-vs-float path gap <= C*scale/2 per entry pre-nonlinearity
    acc = oracle.amm(p, w["A"], relu=False, want_acc=True)["acc"]
    Tsum = sum(p["T"][c][codes[:, c]] for c in range(8))
    deq = acc * p["scale64"] + 8 * p["lo64"]
    assert np.all(np.abs(deq - Tsum) <= 8 * p["scale64"] / 2 * (1 + 1e-9))


# ---------------------------------------------------------------------------- f3: avg16 summation
def _avg_params(C, M, lut, scale=None, offset=None, bias=None):
    """Identity-dim trees (one input dim per codebook, thresholds split [0,16) into codes)."""
    thr = np.tile(bst_thresholds(np.arange(1, 16) - 0.5), (C, 1))
    return params_from(C, C, M, np.zeros((C, 4), np.int32), thr, lut, scale=scale, offset=offset, bias=bias)


def test_avg16_golden_tree_examples():
    """tests/golden/avg16_tree_examples.txt: hand-derived 4-level rounding-average trees."""
    for name, vals, want in read_golden("avg16_tree_examples.txt"):
        v = np.array([int(x) for x in vals.split()], np.int64)
        lut = np.zeros((16, 16, 1), np.uint8)
        lut[:, :, 0] = v[:, None]                      # every code of codebook c looks up v[c]
        p = _avg_params(16, 1, lut)
        out = oracle.amm(p, np.zeros((1, 16), np.float32), relu=False, want_acc=True, summation="avg16")
        assert int(out["acc"][0, 0]) == int(want), name


def test_avg16_multiples_of_16_are_exact_and_bias_bounds():
    """Entries that are multiples of 16 never round: acc_avg * 16 == acc_exact.  For any entries
    each group's tree result exceeds the group mean by d with 0 <= d < 2, and E[d] = 1 (the
    per-level rounding adds 1/4 in expectation at each of the 4 levels, halved upwards: 4 x 1/4)."""
    rng = np.random.default_rng(7)
    C, M, N = 64, 40, 3000
    A = rng.uniform(0, 16, size=(N, C)).astype(np.float32)
    lut16 = (rng.integers(0, 16, size=(C, 16, M)) * 16).astype(np.uint8)
    p = _avg_params(C, M, lut16)
    ex = oracle.amm(p, A, relu=False, want_acc=True)["acc"]
    av = oracle.amm(p, A, relu=False, want_acc=True, summation="avg16")["acc"]
    assert np.array_equal(av * 16, ex)
    lut = rng.integers(0, 256, size=(C, 16, M)).astype(np.uint8)
    p = _avg_params(C, M, lut)
    ex = oracle.amm(p, A, relu=False, want_acc=True)["acc"].astype(np.float64)
    av = oracle.amm(p, A, relu=False, want_acc=True, summation="avg16")["acc"].astype(np.float64)
    G = C // 16
    d = av - ex / 16.0
    assert d.min() >= 0 and d.max() < 2 * G
    assert abs(d.mean() / G - 1.0) < 0.01, d.mean() / G


def test_avg16_dequant_is_one_rounding_and_rejects_ragged_C():
    """y = fmaf(16*scale, acc, offavg) with offavg = (float)(C*lo + bias - 16*(C/16)*scale): the
    exact rational 16*scale*acc + offavg rounded once to fp32 (reading R22); C % 16 != 0 refused."""
    rng = np.random.default_rng(8)
    C, M = 32, 7
    lut = rng.integers(0, 256, size=(C, 16, M)).astype(np.uint8)
    scale = rng.uniform(1e-3, 1e-2, M).astype(np.float32)
    off = rng.normal(0, 0.1, M).astype(np.float32)
    bias = rng.normal(0, 0.1, M).astype(np.float32)
    p = _avg_params(C, M, lut, scale=scale, offset=off, bias=bias)
    A = rng.uniform(0, 16, size=(50, C)).astype(np.float32)
    out = oracle.amm(p, A, relu=False, want_acc=True, summation="avg16")
    for m in range(M):
        offavg = np.float32(float(C) * float(off[m]) + float(bias[m]) - 16.0 * (C // 16) * float(scale[m]))
        for n in range(50):
            exact = Fraction(float(np.float32(16 * scale[m]))) * int(out["acc"][n, m]) + Fraction(float(offavg))
            assert out["y"][n, m] == _round_f32(exact)
    p2 = _avg_params(8, 1, np.zeros((8, 16, 1), np.uint8))
    with pytest.raises(RuntimeError):
        oracle.amm(p2, np.zeros((1, 8), np.float32), relu=False, summation="avg16")


# ---------------------------------------------------------------------------- f4: Eq. 3 LUT fit
def test_eq3_linear_single_codebook_is_bucket_ridge_mean():
    """C = 1: G^T G is diagonal (bucket counts), so Eq. 3 with sigma = bias reduces per code k to
    T[k] = (sum of the targets a.B of the rows in bucket k + lam T0[k]) / (count_k + lam)."""
    rng = np.random.default_rng(3)
    N, D, M, lam = 400, 6, 5, 2.5
    A = rng.normal(size=(N, D))
    B = rng.normal(size=(D, M))
    codes = rng.integers(0, 16, size=(N, 1)).astype(np.uint8)
    T0 = rng.normal(size=(1, 16, M))
    T = ofit.optimize_lut_linear(A, B, codes, T0, lam)
    Y = A @ B
    for k in range(16):
        rows = codes[:, 0] == k
        want = (Y[rows].sum(axis=0) + lam * T0[0, k]) / (rows.sum() + lam)
        assert np.allclose(T[0, k], want, rtol=1e-12, atol=1e-12)


def test_eq3_objective_hand_computed():
    """eq3_objective (sigma = bias then optional ReLU) on a case worked by hand:
    A = [[1],[2]], B = [[3]] -> AB = [3, 6]; codes [[0],[1]]; T[0][0] = 2.5, T[0][1] = 7 (rest 0)
    -> GT = [2.5, 7]; T0[0][0] = 2 (rest 0), lam = 0.1 -> lam*||T - T0||^2 = 0.1*(0.25 + 49) = 4.925.
    bias 0.5: sigma(AB) = [3.5, 6.5], sigma(GT) = [3.0, 7.5] -> 0.25 + 1 = 1.25; total 6.175.
    bias -4 with ReLU: [-1, 2] -> [0, 2] and [-1.5, 3] -> [0, 3] -> 1; total 5.925."""
    A = np.array([[1.0], [2.0]])
    B = np.array([[3.0]])
    codes = np.array([[0], [1]], np.uint8)
    T = np.zeros((1, 16, 1))
    T[0, 0, 0], T[0, 1, 0] = 2.5, 7.0
    T0 = np.zeros((1, 16, 1))
    T0[0, 0, 0] = 2.0
    assert ofit.eq3_objective(A, B, np.array([0.5]), codes, T, T0, 0.1, relu=False) == pytest.approx(6.175, abs=1e-12)
    assert ofit.eq3_objective(A, B, np.array([-4.0]), codes, T, T0, 0.1, relu=True) == pytest.approx(5.925, abs=1e-12)


def test_eq3_linear_optimality_and_limits():
    """The solution satisfies the normal equations, is no worse than P0 B for the objective, and
    tends to P0 B as lam grows."""
    rng = np.random.default_rng(4)
    N, D, M, C = 600, 24, 7, 4
    A = rng.normal(size=(N, D))
    B = rng.normal(size=(D, M))
    bias = rng.normal(size=M)
    codes = rng.integers(0, 16, size=(N, C)).astype(np.uint8)
    T0 = rng.normal(size=(C, 16, M))
    T = ofit.optimize_lut_linear(A, B, codes, T0, 0.3)
    G = ofit.onehot(codes)
    resid = (G.T @ G + 0.3 * np.eye(16 * C)) @ T.reshape(-1, M) - (G.T @ (A @ B) + 0.3 * T0.reshape(-1, M))
    assert np.abs(resid).max() < 1e-8
    f = lambda TT: ofit.eq3_objective(A, B, bias, codes, TT, T0, 0.3, relu=False)  # noqa: E731
    assert f(T) <= f(T0) + 1e-9
    for d in (1e-3, -1e-3):
        Tp = T.copy()
        Tp[1, 3, 2] += d
        assert f(T) <= f(Tp)
    Tbig = ofit.optimize_lut_linear(A, B, codes, T0, 1e9)
    assert np.abs(Tbig - T0).max() < 1e-5


# ---------------------------------------------------------------------------- f4: Eq. 3 with KLD
def test_eq3_kld_hand_computed_value():
    """KLD objective (P:100 softmax sigma) on a case worked by hand.
    D = 1, M = 2, C = 1, bias 0: row 1 a = 1, B = [[0, ln 3]] -> softmax(aB) = (1/4, 3/4); code 0 with
    T[0][0] = (0, 0) -> q = (1/2, 1/2); KL = 1/4 ln(1/2) + 3/4 ln(3/2).  Row 2 a = 0 -> p = (1/2, 1/2);
    code 1 with T[0][1] = (ln 3, 0) -> q = (3/4, 1/4); KL = 1/2 ln(2/3) + 1/2 ln 2.  With T0 = 0 and
    lam = 0.5 the penalty is 0.5 (ln 3)^2."""
    A = np.array([[1.0], [0.0]])
    B = np.array([[0.0, math.log(3.0)]])
    codes = np.array([[0], [1]], np.uint8)
    T = np.zeros((1, 16, 2))
    T[0, 1, 0] = math.log(3.0)
    want_kl = 0.25 * math.log(0.5) + 0.75 * math.log(1.5) + 0.5 * math.log(2.0 / 3.0) + 0.5 * math.log(2.0)
    assert ofit.eq3_objective_kld(A, B, np.zeros(2), codes, T, T, 0.5) == pytest.approx(want_kl, abs=1e-14)
    want = want_kl + 0.5 * math.log(3.0) ** 2
    assert ofit.eq3_objective_kld(A, B, np.zeros(2), codes, T, np.zeros_like(T), 0.5) == pytest.approx(want, abs=1e-14)


def test_eq3_kld_gradient_matches_central_differences():
    """SPEC S:344 example: softmax + KLD on a random 64 x 16 x 10 instance (64 rows, one codebook of
    16 codes, M = 10): the analytic gradient matches central finite differences to rel. err < 1e-4."""
    rng = np.random.default_rng(5)
    N, D, M = 64, 6, 10
    A, B, bias = rng.normal(size=(N, D)), rng.normal(size=(D, M)), rng.normal(size=M)
    codes = rng.integers(0, 16, size=(N, 1)).astype(np.uint8)
    T0 = rng.normal(size=(1, 16, M))
    T = T0 + 0.3 * rng.normal(size=T0.shape)
    g = ofit.eq3_kld_grad(A, B, bias, codes, T, T0, 0.7)
    h = 1e-6
    num = np.zeros_like(T)
    for idx in np.ndindex(T.shape):
        Tp, Tm = T.copy(), T.copy()
        Tp[idx] += h
        Tm[idx] -= h
        num[idx] = (ofit.eq3_objective_kld(A, B, bias, codes, Tp, T0, 0.7) -
                    ofit.eq3_objective_kld(A, B, bias, codes, Tm, T0, 0.7)) / (2 * h)
    assert np.abs(g - num).max() / np.abs(num).max() < 1e-4


def test_eq3_kld_softmax_shift_invariance():
    """softmax is invariant to adding one constant to a whole row, and every row holds exactly one
    code per codebook: adding kappa to all 16 entries of codebook c, in every column, adds kappa to
    every row of G T, which leaves the KL term unchanged; and the KL gradient sums to 0 over the
    outputs m of each (c, k)."""
    rng = np.random.default_rng(6)
    N, D, M, C = 50, 8, 7, 3
    A, B, bias = rng.normal(size=(N, D)), rng.normal(size=(D, M)), rng.normal(size=M)
    codes = rng.integers(0, 16, size=(N, C)).astype(np.uint8)
    T = rng.normal(size=(C, 16, M))
    T2 = T.copy()
    T2[1] += 2.5
    f = lambda TT: ofit.eq3_objective_kld(A, B, bias, codes, TT, TT, 0.0)  # noqa: E731
    assert f(T2) == pytest.approx(f(T), rel=1e-12, abs=1e-12)
    g = ofit.eq3_kld_grad(A, B, bias, codes, T, T, 0.0)
    assert np.abs(g.sum(axis=2)).max() < 1e-12


def test_eq3_kld_exact_reconstruction_is_a_fixed_point():
    """SPEC S:344 example: when G reconstructs A B exactly (exact PQ, rows equal prototypes), T = P0 B
    already gives a zero KL term and a zero gradient, so the descent returns T0 unchanged."""
    C, M = 4, 6
    A_train, _, kt, B, bias = exact_pq_case(C, M, n_rep=2, seed=7)
    p = ofit.fit(A_train, B, C, np.arange(4 * C), bias)
    codes = oracle.amm(p, A_train, relu=False, want_codes=True)["codes"]
    T0 = p["T"]
    assert ofit.eq3_objective_kld(A_train, B, bias, codes, T0, T0, 0.3) < 1e-12
    assert np.abs(ofit.eq3_kld_grad(A_train, B, bias, codes, T0, T0, 0.3)).max() < 1e-12
    T = ofit.optimize_lut_kld(A_train, B, bias, codes, T0, 0.3, steps=5, lr=0.1)
    assert np.abs(T - T0).max() < 1e-12


def test_eq3_kld_descent_lowers_the_objective():
    """Gradient descent with a small step lowers the KLD objective at every step (fixed-step GD on a
    smooth convex-in-Z objective) and ends below T0."""
    rng = np.random.default_rng(9)
    N, D, M, C = 200, 12, 5, 3
    A, B, bias = rng.normal(size=(N, D)), rng.normal(size=(D, M)), rng.normal(size=M)
    codes = rng.integers(0, 16, size=(N, C)).astype(np.uint8)
    T0 = rng.normal(size=(C, 16, M))
    f = lambda TT: ofit.eq3_objective_kld(A, B, bias, codes, TT, T0, 0.05)  # noqa: E731
    vals = [f(T0)]
    T = T0
    for _ in range(10):
        T = T - 0.02 * ofit.eq3_kld_grad(A, B, bias, codes, T, T0, 0.05)
        vals.append(f(T))
    assert all(b < a for a, b in zip(vals, vals[1:]))
