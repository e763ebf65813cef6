"""Split-packed input: a layer re-parameterised for rows that hold only the 4C split
values in [c][level] order computes the same codes, accumulators and outputs as the original layer
on whole rows.  CPU: the oracle on both parameterisations (product `split_packed` vs bench-local
`_split_packed` vs the plain gather of the oracle's own columns).  GPU: the product kernels on
packed rows against the oracle on whole rows, bit for bit."""
import numpy as np
import pytest

import oracle
import synth
from oracle import fit as ofit


def _case(seed, N, D, M, C, dtype="f32"):
    w = synth.small_case(seed, N=N, D=D, M=M, C=C, dtype=dtype, n_train=600)
    params = ofit.fit(w["A_train"], w["B"], C, w["perm"], w["bias"], a_is_bf16=dtype == "bf16")
    return w, params


@pytest.mark.parametrize("seed,N,D,M,C,dtype", [(31, 300, 97, 33, 10, "f32"), (32, 257, 784, 64, 32, "f32"),
                                                (33, 200, 300, 20, 75, "bf16")])
def test_packed_layer_equals_whole_row_layer_oracle(seed, N, D, M, C, dtype):
    from paper_2207_05808_b200 import split_packed
    import bench
    w, params = _case(seed, N, D, M, C, dtype)
    pp, cols = split_packed(params)
    pp2, cols2 = bench._split_packed(params)
    assert np.array_equal(cols, cols2) and pp["D"] == pp2["D"] == 4 * C
    assert cols.shape == (4 * C,) and cols.min() >= 0 and cols.max() < D
    A = w["A"]
    ref = oracle.amm(params, A, relu=w["relu"], dtype=dtype, want_codes=True, want_acc=True)
    got = oracle.amm(pp, np.ascontiguousarray(A[:, cols]), relu=w["relu"], dtype=dtype, want_codes=True,
                     want_acc=True)
    assert np.array_equal(got["codes"], ref["codes"])
    assert np.array_equal(got["acc"], ref["acc"])
    assert np.array_equal(got["y"].view(np.uint32), ref["y"].view(np.uint32))


def test_split_columns_follow_the_permutation_and_partition():
    """cols[c][t] = perm[b_c + split_dim[c][t]] with larger-first chunks (reading R12)."""
    from paper_2207_05808_b200.fit import split_columns, chunk_bounds
    D, C = 10, 3
    perm = np.array([9, 8, 7, 6, 5, 4, 3, 2, 1, 0])
    sd = np.array([[0, 1, 2, 3], [2, 1, 0, 0], [0, 2, 1, 2]])
    cols = split_columns(dict(D=D, C=C, perm=perm, boundaries=None, split_dim=sd))
    b = chunk_bounds(D, C)
    assert list(b) == [0, 4, 7, 10]
    assert list(cols) == [9, 8, 7, 6, 3, 4, 5, 5, 2, 0, 1, 0]


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["auto", "tc", "simt"])
def test_packed_rows_on_gpu_match_whole_row_oracle(algo):
    torch = pytest.importorskip("torch")
    from paper_2207_05808_b200 import Plan, split_packed
    from paper_2207_05808_b200._lib import ItlummError
    w, params = _case(34, 3001, 784, 512, 32)
    pp, cols = split_packed(params)
    ref = oracle.amm(params, w["A"], relu=True, want_codes=True, want_acc=True, nthreads=8)
    plan = Plan(pp, device=0)
    try:
        plan.set_algo(algo)
        A = torch.from_numpy(np.ascontiguousarray(w["A"][:, cols])).cuda()
        y = plan.amm(A, relu=True)
    except ItlummError as e:
        if e.status == 3:
            pytest.skip(str(e))
        raise
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref["y"].view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("seed,N,D,M,C,dtype", [(35, 2500, 512, 300, 64, "bf16"), (36, 1300, 1024, 96, 128, "f32"),
                                                (37, 777, 300, 40, 48, "f32")])
def test_packed_rows_register_tree_walk_paths(seed, N, D, M, C, dtype):
    """Split-packed rows through the encoder's register-threshold path (fixed codebook groups:
    C = 64 bf16 vector loads of 8 bytes, C = 128 f32, C = 48 with a partly empty second group)."""
    torch = pytest.importorskip("torch")
    from paper_2207_05808_b200 import Plan, split_packed
    w, params = _case(seed, N, D, M, C, dtype)
    pp, cols = split_packed(params)
    ref = oracle.amm(params, w["A"], relu=w["relu"], dtype=dtype, want_codes=True, nthreads=8)
    plan = Plan(pp, device=0)
    Ap = np.ascontiguousarray(w["A"][:, cols])
    A = torch.from_numpy(Ap.view(np.int16) if dtype == "bf16" else Ap).cuda()
    if dtype == "bf16":
        A = A.view(torch.bfloat16)
    codes = plan.encode(A)
    y = plan.amm(A, relu=w["relu"])
    torch.cuda.synchronize()
    c = codes.cpu().numpy()
    got = np.stack([(c[:, i // 2] >> (4 * (i % 2))) & 15 for i in range(C)], axis=1)
    assert np.array_equal(got, ref["codes"])
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref["y"].view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("seed,N,D,M,C,dtype,pad", [(41, 1, 64, 40, 8, "f32", 0), (42, 129, 200, 300, 20, "f32", 0),
                                                    (43, 1000, 500, 520, 33, "f32", 8), (44, 700, 300, 96, 12, "bf16", 0),
                                                    (45, 300, 50, 64, 4, "f32", 0)])
def test_fused_tc_on_packed_rows(seed, N, D, M, C, dtype, pad):
    """The fused tensor-core kernel on split-packed rows: f32 rows staged K-block by K-block by TMA
    into the one-hot stage and overwritten in place (C >= 8; ragged last K-block C = 20, 33; a row
    tail N = 129; two and three M slices; lda > 4C), bf16 and C < 8 on per-thread vector loads;
    bit-exact against the oracle on whole rows, alone and through AUTO."""
    torch = pytest.importorskip("torch")
    from paper_2207_05808_b200 import Plan, split_packed
    w, params = _case(seed, N, D, M, C, dtype)
    pp, cols = split_packed(params)
    ref = oracle.amm(params, w["A"], relu=w["relu"], dtype=dtype, nthreads=8)
    Ap = np.ascontiguousarray(w["A"][:, cols])
    if pad:
        Ap = np.concatenate([Ap, np.full((N, pad), np.nan, Ap.dtype)], axis=1)
    A = torch.from_numpy(Ap.view(np.int16) if dtype == "bf16" else Ap).cuda()
    if dtype == "bf16":
        A = A.view(torch.bfloat16)
    if pad:
        A = A[:, : 4 * C]
    plan = Plan(pp, device=0)
    for algo in ("tc", "auto"):
        plan.set_algo(algo)
        y = plan.amm(A, relu=w["relu"])
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy().view(np.uint32), ref["y"].view(np.uint32)), algo


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["tc", "auto"])
def test_fused_tc_packed_cfg2_full_size_sampled(algo):
    """BASELINE configs[1] split-packed at full size (N = 60000, 469 row tiles, 2 M slices): the
    fused kernel (TMA-staged rows) against encode -> accumulate for every row and the oracle on whole
    rows for sampled rows (tile and item-round boundaries, first and last rows)."""
    torch = pytest.importorskip("torch")
    from paper_2207_05808_b200 import Plan, split_packed
    w = synth.workload("cfg2")
    params = ofit.fit(w["A_train"], w["B"], w["C"], w["perm"], w["bias"])
    pp, cols = split_packed(params)
    plan = Plan(pp, device=0)
    A = torch.from_numpy(np.ascontiguousarray(w["A"][:, cols])).cuda()
    plan.set_algo("tc_pipe")
    y_pipe = plan.amm(A, relu=True)
    plan.set_algo(algo)
    y = plan.amm(A, relu=True)
    torch.cuda.synchronize()
    y, y_pipe = y.cpu().numpy(), y_pipe.cpu().numpy()
    assert np.array_equal(y.view(np.uint32), y_pipe.view(np.uint32))
    edges = np.array([0, 1, 127, 128, 255, 256, 9471, 9472, 18943, 18944, 59903, 59904, 59998, 59999])
    rows = np.unique(np.concatenate([np.random.default_rng(1).choice(60000, 2048, replace=False), edges]))
    ref = oracle.amm(params, w["A"][rows], relu=True, nthreads=8)
    assert np.array_equal(y[rows].view(np.uint32), ref["y"].view(np.uint32))
