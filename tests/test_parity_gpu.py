"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.

Parameters are fitted by the ORACLE's fitter (oracle/fit.py), so no oracle input comes from
the product.  Bar (BASELINE north_star): codes and int32 accumulators bit-exact; fp32 outputs
within 1e-6 relative + 1e-6 absolute (checked), and — because both sides evaluate the same
single fmaf (reading R8) — bit-exact as well (checked)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import fit as ofit

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL = ATOL = 1e-6
# "_sp24" / "_dense": the same schedule with the one-hot operand forced to the 2:4-sparse form
# (tcgen05.mma.sp) or the dense form; plain names use the library's choice (AUTO: dense)
ALGOS = ["auto", "simt", "tc", "tc_pipe", "tc_sp24", "tc_pipe_sp24", "tc_pipe_dense"]


def _set(plan, algo):
    for suffix, onehot in (("_sp24", "sparse24"), ("_dense", "dense")):
        if algo.endswith(suffix):
            plan.set_algo(algo[: -len(suffix)])
            plan.set_onehot(onehot)
            return
    plan.set_algo(algo)
    plan.set_onehot("auto")


def _skip_or_raise(algo, e):
    """Only an explicitly requested tensor-core schedule may refuse a shape (its documented
    EUNSUPPORTED, e.g. the fused TC kernel on a streamed LUT); AUTO and SIMT must run everything."""
    if algo.startswith("tc") and e.status == 3:
        pytest.skip(f"{algo} unsupported for this shape: {e}")
    raise e


def _plan(params, algo):
    from paper_2207_05808_b200 import Plan
    p = Plan(params, device=0)
    _set(p, algo)
    return p


def _dev(A, dtype):
    t = torch.from_numpy(np.ascontiguousarray(A.view(np.int16) if dtype == "bf16" else A)).cuda()
    return t.view(torch.bfloat16) if dtype == "bf16" else t


def unpack(codes: np.ndarray, C: int) -> np.ndarray:
    out = np.zeros((codes.shape[0], C), np.uint8)
    for c in range(C):
        b = codes[:, c // 2]
        out[:, c] = (b >> 4) if c % 2 else (b & 15)
    return out


def assert_out(gpu, ref):
    assert gpu.shape == ref.shape
    assert np.allclose(gpu, ref, rtol=RTOL, atol=ATOL), np.abs(gpu - ref).max()
    assert np.array_equal(gpu.view(np.uint32), ref.view(np.uint32)), int((gpu != ref).sum())


def run_all(params, A, relu, dtype, algo):
    """encode -> codes; lut_accumulate -> acc, out; amm (fused) -> out; all vs the oracle."""
    from paper_2207_05808_b200._lib import ItlummError
    ref = oracle.amm(params, A, relu=relu, dtype=dtype, want_codes=True, want_acc=True, nthreads=8)
    plan = _plan(params, "simt")
    Ad = _dev(A, dtype)
    codes = plan.encode(Ad)
    torch.cuda.synchronize()
    assert np.array_equal(unpack(codes.cpu().numpy(), params["C"]), ref["codes"])
    if params["C"] % 2:
        assert np.all(codes.cpu().numpy()[:, -1] >> 4 == 0)     # R14 padding nibble
    try:
        _set(plan, algo)
    except ItlummError as e:
        _skip_or_raise(algo, e)
    # the fused call and the two-step call are checked independently: a schedule that refuses one
    # of them must not hide the other
    skipped = []
    try:
        y = plan.amm(Ad, relu=relu)
        torch.cuda.synchronize()
        assert_out(y.cpu().numpy(), ref["y"])
    except ItlummError as e:
        skipped.append(e)
    try:
        acc = torch.empty((A.shape[0], params["M"]), dtype=torch.int32, device="cuda")
        out, _ = plan.lut_accumulate(codes, acc=acc, relu=relu)
        torch.cuda.synchronize()
        assert np.array_equal(acc.cpu().numpy().astype(np.int64), ref["acc"])
        assert_out(out.cpu().numpy(), ref["y"])
        out2, _ = plan.lut_accumulate(codes, relu=relu)          # fp32 only (the TMA-store epilogue)
        torch.cuda.synchronize()
        assert_out(out2.cpu().numpy(), ref["y"])
    except ItlummError as e:
        skipped.append(e)
    if skipped:
        _skip_or_raise(algo, skipped[0])
    return plan, ref


CASES = [
    # seed, N, D, M, C, dtype   (ragged N vs every tile height, odd C, M not a multiple of 16)
    (1, 1000, 64, 24, 8, "f32"),
    (2, 777, 97, 33, 10, "f32"),
    (3, 1500, 96, 40, 12, "bf16"),
    (4, 300, 50, 5, 50, "f32"),
    (5, 2049, 784, 512, 32, "f32"),
    (6, 513, 200, 1000, 17, "f32"),
    (7, 129, 300, 129, 300, "f32"),       # C > 257: 16-bit SWAR lanes flushed
    (8, 1, 31, 1, 1, "f32"),
    (9, 4097, 256, 256, 64, "bf16"),
    (10, 3000, 4096, 512, 256, "bf16"),   # cfg5-shaped: LUT K-blocks streamed (too large to stay resident)
    (14, 700, 2048, 300, 512, "f32"),     # streamed LUT, M not a multiple of the 256-column slice
]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("seed,N,D,M,C,dtype", CASES)
def test_parity_small(seed, N, D, M, C, dtype, algo):
    w = synth.small_case(seed, N=N, D=D, M=M, C=C, dtype=dtype, n_train=600)
    params = ofit.fit(w["A_train"], w["B"], C, w["perm"], w["bias"], a_is_bf16=dtype == "bf16")
    run_all(params, w["A"], w["relu"], dtype, algo)


@pytest.mark.parametrize("algo", ALGOS)
def test_parity_cfg1_full(algo):
    """BASELINE configs[0] at its full size (N = 1000)."""
    w = synth.workload("cfg1")
    params = ofit.fit(w["A_train"], w["B"], w["C"], w["perm"], w["bias"])
    run_all(params, w["A"], w["relu"], "f32", algo)


@pytest.mark.parametrize("algo", ALGOS)
def test_parity_cfg2_full_sampled(algo):
    """BASELINE configs[1] at full size N = 60000 in the bench launch configuration: sampled rows
    against the oracle, every row's fused output against encode -> lut_accumulate."""
    from paper_2207_05808_b200._lib import ItlummError
    w = synth.workload("cfg2")
    params = ofit.fit(w["A_train"], w["B"], w["C"], w["perm"], w["bias"])
    plan = _plan(params, "simt")
    Ad = _dev(w["A"], "f32")
    codes = plan.encode(Ad)
    try:
        _set(plan, algo)
        y = plan.amm(Ad, relu=True)
        y2, _ = plan.lut_accumulate(codes, relu=True)
    except ItlummError as e:
        _skip_or_raise(algo, e)
    torch.cuda.synchronize()
    y, y2, codes = y.cpu().numpy(), y2.cpu().numpy(), codes.cpu().numpy()
    assert np.array_equal(y.view(np.uint32), y2.view(np.uint32))
    rows = np.unique(np.concatenate([np.random.default_rng(0).choice(60000, 1500, replace=False),
                                     [0, 1, 59998, 59999]]))
    ref = oracle.amm(params, w["A"][rows], relu=True, want_codes=True, nthreads=8)
    assert np.array_equal(unpack(codes[rows], 32), ref["codes"])
    assert_out(y[rows], ref["y"])
    assert np.all(y >= 0) and not np.any(np.signbit(y))


@pytest.mark.parametrize("algo", ALGOS)
def test_edge_strides_alignment_and_specials(algo):
    """lda > D, ldo > M, a misaligned output base (scalar-store path), +-inf thresholds, NaN and
    +-inf inputs, N = 0."""
    from paper_2207_05808_b200._lib import ItlummError
    w = synth.small_case(11, N=600, D=80, M=48, C=10, n_train=500)
    params = ofit.fit(w["A_train"], w["B"], 10, w["perm"], w["bias"])
    params["thresholds"][0, :] = np.inf
    params["thresholds"][1, :] = -np.inf
    A = np.zeros((600, 91), np.float32)
    A[:, :80] = w["A"]
    A[3, :] = np.nan
    A[4, :] = np.inf
    A[5, :] = -np.inf
    ref = oracle.amm(params, A, relu=True, want_codes=True)
    plan = _plan(params, "simt")
    try:
        _set(plan, algo)
        Ad = torch.from_numpy(A).cuda()
        big = torch.full((600, 64), -7.0, device="cuda")
        plan.amm(Ad[:, :], out=big[:, :48], relu=True)
        raw = torch.full((600 * 48 + 1,), -7.0, device="cuda")
        mis = raw[1:].view(600, 48)
        plan.amm(Ad, out=mis, relu=True)
        empty = plan.amm(Ad[:0], relu=True)
    except ItlummError as e:
        _skip_or_raise(algo, e)
    torch.cuda.synchronize()
    assert_out(big[:, :48].cpu().numpy(), ref["y"])
    assert np.all(big[:, 48:].cpu().numpy() == -7.0)
    assert_out(mis.cpu().numpy(), ref["y"])
    assert raw[0].item() == -7.0 and empty.shape == (0, 48)
    assert plan.last_launch_count == 0   # N = 0 launches nothing


def test_amm_host_end_to_end():
    """itlumm_amm_host (host buffers, chunked H2D / kernel / D2H) equals the oracle."""
    w = synth.small_case(12, N=70000, D=64, M=40, C=8, n_train=500)
    params = ofit.fit(w["A_train"], w["B"], 8, w["perm"], w["bias"])
    from paper_2207_05808_b200 import Plan
    plan = Plan(params)
    A = torch.from_numpy(w["A"]).pin_memory()
    y = plan.amm_host(A, relu=True)
    assert plan.last_launch_count >= 1
    ref = oracle.amm(params, w["A"], relu=True, nthreads=8)
    assert_out(y.numpy(), ref["y"])


def test_error_paths_on_device():
    from paper_2207_05808_b200 import Plan
    from paper_2207_05808_b200._lib import ItlummError
    w = synth.small_case(13, N=10, D=40, M=8, C=4, n_train=200)
    params = ofit.fit(w["A_train"], w["B"], 4, w["perm"], w["bias"])
    plan = Plan(params)
    A = torch.from_numpy(w["A"]).cuda()
    # the binding rejects what raw pointers cannot show: width, dtype, device, strides
    with pytest.raises(ValueError):
        plan.amm(A[:, :30].contiguous())             # fewer than D columns
    with pytest.raises(TypeError):
        plan.amm(A.double())
    with pytest.raises(ValueError):
        plan.amm(A, out=torch.empty((10, 4), device="cuda"))   # fewer than M columns
    with pytest.raises(ValueError):
        plan.amm(A.cpu())                            # host rows to a device call
    with pytest.raises(ValueError):
        plan.amm(A.t().contiguous().t())             # column-major rows
    with pytest.raises(TypeError):
        plan.lut_accumulate(plan.encode(A), acc=torch.empty((10, 8), dtype=torch.int64, device="cuda"))
    # the C ABI itself: strides inconsistent with the plan are ESHAPE, host pointers are EINVAL
    import ctypes
    from paper_2207_05808_b200 import _lib
    lib = _lib.load()
    out = torch.empty((10, 8), device="cuda")
    st = lib.itlumm_amm(plan._h, ctypes.c_void_p(A.data_ptr()), _lib.F32, 30, 10,
                        ctypes.c_void_p(out.data_ptr()), 8, 0, None)
    assert st == _lib.ESHAPE and "lda" in lib.itlumm_last_error().decode()
    st = lib.itlumm_amm(plan._h, ctypes.c_void_p(A.data_ptr()), _lib.F32, 40, 10,
                        ctypes.c_void_p(out.data_ptr()), 4, 0, None)
    assert st == _lib.ESHAPE
    Ah = A.cpu()
    st = lib.itlumm_amm(plan._h, ctypes.c_void_p(Ah.data_ptr()), _lib.F32, 40, 10,
                        ctypes.c_void_p(out.data_ptr()), 8, 0, None)
    assert st == _lib.EINVAL and "device memory" in lib.itlumm_last_error().decode()


def _mlp_case(C, n_rows, n_train, layers):
    w = synth.mlp_workload(C, n_rows, n_train=n_train, layers=layers)
    oparams = oracle.fit_mlp(w["A_train"], w["Bs"], w["Cs"], w["perms"], w["biases"], w["relus"])
    return w, oparams


@pytest.mark.parametrize("C,layers", [
    (8, [(96, 64, True), (64, 48, True), (48, 10, False)]),
    (5, [(97, 33, True), (33, 17, True), (17, 3, False)]),     # odd widths: padded compact rows
])
def test_mlp_chain_small(C, layers):
    """itlumm_mlp (hidden layers compute only the columns the next layer splits on) equals the
    oracle running every layer in full; the product fit through the GPU chain equals the oracle's
    fit (O9) bit for bit."""
    from paper_2207_05808_b200 import Mlp, fit_mlp
    w, oparams = _mlp_case(C, 2500, 700, layers)
    pparams = fit_mlp(w["A_train"], w["Bs"], w["Cs"], w["perms"], w["biases"], w["relus"])
    for po, pp in zip(oparams, pparams):
        for k in ("split_dim", "thresholds", "lut", "scale", "offset"):
            assert np.array_equal(np.asarray(po[k]).view(np.uint8), np.asarray(pp[k]).view(np.uint8)), k
    mlp = Mlp(oparams, w["relus"])
    widths = mlp.widths()
    assert widths[-1] == layers[-1][1] and all(widths[l] <= min(4 * C, layers[l][1]) for l in range(2))
    y = mlp.forward(torch.from_numpy(w["A"]).cuda())
    torch.cuda.synchronize()
    ref = oracle.mlp_forward(oparams, w["relus"], w["A"])
    assert_out(y.cpu().numpy(), ref)


@pytest.mark.parametrize("C", [16, 64, 128, 256])
def test_mlp_cfg4_shapes_sampled(C):
    """BASELINE configs[3] layer shapes 3072-1024-1024-10 (N = 70000 rows: two 65536-row seed
    chunks, ragged tail), sampled rows against the oracle's full-layer chain."""
    from paper_2207_05808_b200 import Mlp
    w, oparams = _mlp_case(C, 70000, 4096, synth.MLP_LAYERS)
    mlp = Mlp(oparams, w["relus"])
    y = mlp.forward(torch.from_numpy(w["A"]).cuda())
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    rows = sample_rows(70000, 1200, seed=1)
    ref = oracle.mlp_forward(oparams, w["relus"], w["A"][rows])
    assert_out(y[rows], ref)


@pytest.mark.parametrize("seed,N,D,M,C,dtype", [(21, 1000, 64, 40, 16, "f32"), (22, 777, 200, 300, 32, "f32"),
                                                (23, 1500, 512, 96, 64, "bf16"), (24, 300, 1024, 48, 256, "f32")])
def test_parity_avg16(seed, N, D, M, C, dtype):
    """avg16 summation (reading R22) on the CUDA-core kernels: codes, group-average sums and fp32
    outputs bit-exact vs the oracle, fused and two-step; the exact plan is unaffected."""
    from paper_2207_05808_b200 import Plan
    w = synth.small_case(seed, N=N, D=D, M=M, C=C, dtype=dtype, n_train=600)
    params = ofit.fit(w["A_train"], w["B"], C, w["perm"], w["bias"], a_is_bf16=dtype == "bf16")
    ref = oracle.amm(params, w["A"], relu=w["relu"], dtype=dtype, want_acc=True, nthreads=8, summation="avg16")
    plan = Plan(params)
    plan.set_summation("avg16")
    Ad = _dev(w["A"], dtype)
    y = plan.amm(Ad, relu=w["relu"])
    codes = plan.encode(Ad)
    acc = torch.empty((N, M), dtype=torch.int32, device="cuda")
    y2, _ = plan.lut_accumulate(codes, acc=acc, relu=w["relu"])
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy().astype(np.int64), ref["acc"])
    assert_out(y.cpu().numpy(), ref["y"])
    assert_out(y2.cpu().numpy(), ref["y"])
    plan.set_summation("exact")
    ye = plan.amm(Ad, relu=w["relu"])
    torch.cuda.synchronize()
    assert_out(ye.cpu().numpy(), oracle.amm(params, w["A"], relu=w["relu"], dtype=dtype, nthreads=8)["y"])


def test_parity_one_cta_streamed_lut_kernel():
    """ITLUMM_PAIR=0 keeps streamed LUTs on the 1-CTA k_tc (developer knob, read at library load):
    that schedule stays bit-exact vs the oracle on the small streamed cases and on cfg3 C=128 at full
    size (several slices, full work rounds)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, synth, oracle\n"
        "from oracle import fit as ofit\n"
        "from paper_2207_05808_b200 import Plan\n"
        "from tests.test_parity_gpu import sample_rows\n"
        "for seed, N, D, M, C, dt in [(9, 4097, 256, 256, 64, 'bf16'), (10, 3000, 4096, 512, 256, 'bf16'), (14, 700, 2048, 300, 512, 'f32')]:\n"
        "    w = synth.small_case(seed, N=N, D=D, M=M, C=C, dtype=dt, n_train=600)\n"
        "    p = ofit.fit(w['A_train'], w['B'], C, w['perm'], w['bias'], a_is_bf16=dt == 'bf16')\n"
        "    ref = oracle.amm(p, w['A'], relu=w['relu'], dtype=dt, nthreads=8)['y']\n"
        "    A = torch.from_numpy(w['A'].view(np.int16) if dt == 'bf16' else w['A']).cuda()\n"
        "    A = A.view(torch.bfloat16) if dt == 'bf16' else A\n"
        "    for oh in ('dense', 'sparse24'):\n"
        "        pl = Plan(p); pl.set_onehot(oh)\n"
        "        y = pl.amm(A, relu=w['relu']).cpu().numpy()\n"
        "        assert np.array_equal(y.view(np.uint32), ref.view(np.uint32)), (seed, oh)\n"
        "w = synth.workload('cfg3_c128')\n"
        "p = ofit.fit(w['A_train'], w['B'], w['C'], w['perm'], w['bias'])\n"
        "y = Plan(p).amm(torch.from_numpy(w['A']).cuda()).cpu().numpy()\n"
        "rows = sample_rows(w['A'].shape[0], 2048, seed=5)\n"
        "ref = oracle.amm(p, w['A'][rows], relu=False, nthreads=8)['y']\n"
        "assert np.array_equal(y[rows].view(np.uint32), ref.view(np.uint32))\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ITLUMM_PAIR="0", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def sample_rows(N: int, n: int, seed: int = 0) -> np.ndarray:
    """At least n distinct rows of an N-row call: the first and last rows, both sides of every
    128-row (1-CTA tile) and 256-row (CTA-pair tile) boundary among the first and last 8 tiles and
    among 32 random tiles, the 262144-row scratch-chunk edges, and random rows."""
    g = np.random.default_rng(seed)
    picks = [0, 1, 2, N - 3, N - 2, N - 1]
    ntile = (N + 127) // 128
    tiles = set(range(min(8, ntile))) | set(range(max(0, ntile - 8), ntile))
    tiles |= set(g.choice(ntile, min(32, ntile), replace=False).tolist())
    for t in tiles:
        for d in (-1, 0, 1, 127):
            picks.append(t * 128 + d)
    for e in range(262144, N + 1, 262144):
        picks += [e - 1, e]
    rows = np.unique(np.clip(np.array(picks), 0, N - 1))
    if len(rows) < n:
        rest = np.setdiff1d(np.arange(N), rows)
        rows = np.unique(np.concatenate([rows, g.choice(rest, min(n - len(rows), len(rest)), replace=False)]))
    return rows


@pytest.mark.parametrize("name,onehot", [("cfg3_c64", "auto"), ("cfg3_c64", "sparse24"), ("cfg3_c64", "dense"),
                                         ("cfg3_c128", "auto"), ("cfg3_c128", "sparse24"), ("cfg3_c128", "dense"),
                                         ("cfg5", "auto"), ("cfg5", "dense")])
def test_benched_streamed_lut_shapes_full_size_sampled(name, onehot):
    """BASELINE configs[2] (C = 64, 128) and configs[4] at FULL size in the launch configuration
    bench.py times (AUTO: encode -> CTA-pair tensor-core accumulate over a streamed LUT with several
    slices and many full work rounds): >= 4096 sampled rows, chosen across tile and slice-row
    boundaries, bit-exact vs the oracle; every row finite."""
    from paper_2207_05808_b200 import Plan
    w = synth.workload(name)
    dtype = w["dtype"]
    params = ofit.fit(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=dtype == "bf16")
    plan = Plan(params)
    plan.set_onehot(onehot)
    N = w["A"].shape[0]
    y = plan.amm(_dev(w["A"], dtype), relu=w["relu"])
    torch.cuda.synchronize()
    assert plan.last_launch_count == 2 * ((N + 262143) // 262144)    # encode + accumulate per chunk
    y = y.cpu().numpy()
    rows = sample_rows(N, 4096, seed=3)
    assert len(rows) >= 4096
    ref = oracle.amm(params, w["A"][rows], relu=w["relu"], dtype=dtype, nthreads=16)["y"]
    assert_out(y[rows], ref)
    assert np.all(np.isfinite(y))


def test_eq3_lut_optimisation_gpu_vs_oracle():
    """f4 (Eq. 3): the GPU fit's linear solution equals the oracle's fp64 normal-
    equation solution; the ReLU refinement lowers the ReLU objective; the requantised layer keeps
    kernel/oracle parity (only LUT values change) and reconstructs sigma(A B) at least as well
    as the prototype table on the training rows."""
    from paper_2207_05808_b200 import Plan, fit_layer
    from paper_2207_05808_b200.fit import optimize_lut
    w = synth.small_case(41, N=2000, D=96, M=24, C=8, n_train=1500)
    p = fit_layer(w["A_train"], w["B"], 8, w["perm"], w["bias"])
    po = ofit.fit(w["A_train"], w["B"], 8, w["perm"], w["bias"])       # the oracle's own fit
    lin = optimize_lut(p, w["A_train"], w["B"], lam=0.5)
    op = oracle.amm(po, w["A_train"], relu=False, want_codes=True, nthreads=8)
    Tref = ofit.optimize_lut_linear(w["A_train"], w["B"], op["codes"], po["T"], 0.5)
    assert np.allclose(lin["T"], Tref, rtol=1e-7, atol=1e-9)
    obj = lambda T, relu: ofit.eq3_objective(w["A_train"], w["B"], w["bias"], op["codes"], T, po["T"], 0.5, relu)  # noqa: E731
    assert obj(lin["T"], False) <= obj(po["T"], False)
    rel = optimize_lut(p, w["A_train"], w["B"], lam=0.5, relu=True, iters=100)
    assert obj(rel["T"], True) <= obj(lin["T"], True) + 1e-6
    plan = Plan(rel)
    y = plan.amm(torch.from_numpy(w["A"]).cuda(), relu=True)
    torch.cuda.synchronize()
    rel_o = ofit.requantize(po, rel["T"])      # oracle params: its own trees + the fitted table
    assert_out(y.cpu().numpy(), oracle.amm(rel_o, w["A"], relu=True, nthreads=8)["y"])


def test_eq3_kld_lut_optimisation_gpu_vs_oracle():
    """f4 with the KLD objective (P:100 softmax sigma): the GPU descent (codes
    from the encode kernel, fp64 torch) follows the oracle's fp64 descent step for step (same start
    P0 B, same steps, same rate; only the summation order differs), lowers the oracle's KLD objective,
    quantises to the same LUT, and that layer keeps kernel/oracle parity."""
    from paper_2207_05808_b200 import Plan
    from paper_2207_05808_b200.fit import optimize_lut
    w = synth.small_case(42, N=1500, D=80, M=12, C=6, n_train=1200)
    po = ofit.fit(w["A_train"], w["B"], 6, w["perm"], w["bias"])
    gpu = optimize_lut(po, w["A_train"], w["B"], lam=0.2, iters=40, lr=2e-3, objective="kld")
    codes = oracle.amm(po, w["A_train"], relu=False, want_codes=True, nthreads=8)["codes"]
    Tref = ofit.optimize_lut_kld(w["A_train"], w["B"], w["bias"], codes, po["T"], 0.2, steps=40, lr=2e-3)
    assert np.abs(gpu["T"] - Tref).max() <= 1e-9 * (1 + np.abs(Tref).max())
    f = lambda T: ofit.eq3_objective_kld(w["A_train"], w["B"], w["bias"], codes, T, po["T"], 0.2)  # noqa: E731
    assert f(Tref) < f(po["T"])
    ro = ofit.requantize(po, Tref)
    assert np.array_equal(gpu["lut"], ro["lut"]) and np.array_equal(gpu["scale"], ro["scale"])
    y = Plan(ro).amm(torch.from_numpy(w["A"]).cuda(), relu=False)
    torch.cuda.synchronize()
    assert_out(y.cpu().numpy(), oracle.amm(ro, w["A"], relu=False, nthreads=8)["y"])


@pytest.mark.parametrize("name", ["cfg2", "cfg3_c64", "cfg5"])
def test_gpu_tree_fit_equals_oracle_at_baseline_scale(name):
    """f4 tree fitting on the GPU (fit_trees_gpu: batched per-level SSE and lower medians) at the
    BASELINE configs' training sizes: split dims, thresholds and the whole fitted layer (LUT, scale,
    offset) bit-identical to the oracle's plain per-node fit (R3-R5)."""
    from paper_2207_05808_b200 import fit_layer
    w = synth.workload(name, n_rows=0)
    bf16 = w["dtype"] == "bf16"
    pg = fit_layer(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=bf16, device=0)
    po = ofit.fit(w["A_train"], w["B"], w["C"], w["perm"], w["bias"], a_is_bf16=bf16)
    for k in ("split_dim", "thresholds", "lut", "scale", "offset"):
        assert np.array_equal(np.asarray(pg[k]).view(np.uint8), np.asarray(po[k]).view(np.uint8)), k


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_strided_rows_bulk_copy_path_and_scratch_chunking(dtype):
    """Rows with lda > D but 16-byte aligned go through the per-row bulk copies of the streaming
    encoder; N above the plan's 262144-row code scratch runs in chunks; both bit-exact."""
    from paper_2207_05808_b200 import Plan
    N, D, M, C = 300001, 32, 24, 8
    w = synth.small_case(51, N=N, D=D, M=M, C=C, dtype=dtype, n_train=500)
    params = ofit.fit(w["A_train"], w["B"], C, w["perm"], w["bias"], a_is_bf16=dtype == "bf16")
    pad = 8                                            # lda = 40 elements: rows stay 16-byte aligned
    Ah = np.zeros((N, D + pad), np.uint16 if dtype == "bf16" else np.float32)
    Ah[:, :D] = w["A"]
    plan = Plan(params)
    y = plan.amm(_dev(Ah, dtype), relu=True)
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    rows = np.unique(np.concatenate([np.random.default_rng(2).choice(N, 3000, replace=False),
                                     [0, 262143, 262144, N - 1]]))
    ref = oracle.amm(params, Ah[rows], relu=True, dtype=dtype, nthreads=8)["y"]
    assert_out(y[rows], ref)
