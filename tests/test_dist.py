"""Multi-process host logic of the row-sharded path on CPU (gloo, world_size 2): shard arithmetic,
the one-time parameter broadcast, and the max-over-ranks timing reduction.
The data path has no collective, so these are the only distributed pieces."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import synth  # noqa: E402
from paper_2207_05808_b200 import dist as pdist  # noqa: E402
from paper_2207_05808_b200 import fit_layer  # noqa: E402


def test_shard_rows_cover_exactly_once():
    for n in [0, 1, 7, 1000, 60000, 1048576]:
        for world in [1, 2, 3, 4, 8]:
            spans = [pdist.shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    with pytest.raises(ValueError):
        pdist.shard_rows(10, 2, 2)


def test_weak_rows_disjoint():
    spans = [pdist.weak_rows(1000, r) for r in range(8)]
    assert all(b - a == 1000 for a, b in spans)
    assert all(spans[i][1] == spans[i + 1][0] for i in range(7))


def test_sharded_rows_equal_unsharded_stream():
    """A shard regenerates exactly its rows of the seeded stream (chunked seeding), so the
    concatenation over ranks equals the P = 1 input bit for bit."""
    full = synth.rows("mnist", 2, 0, 0, 70000, 64)
    parts = [synth.rows("mnist", 2, 0, *pdist.shard_rows(70000, 3, r), 64) for r in range(3)]
    assert np.array_equal(np.concatenate(parts), full)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        params = None
        if rank == 0:
            w = synth.small_case(31, N=16, D=40, M=12, C=5, n_train=300)
            params = fit_layer(w["A_train"], w["B"], 5, w["perm"], w["bias"])
        got = pdist.broadcast_params(params, torch.device("cpu"))
        mx = pdist.max_over_ranks(float(rank + 1) * 1.5, torch.device("cpu"))
        q.put((rank, {k: (np.asarray(v).tobytes() if not isinstance(v, int) else v)
                      for k, v in got.items()}, mx))
    finally:
        dist.destroy_process_group()


def test_broadcast_params_and_max_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r, got, mx = q.get(timeout=120)
        res[r] = (got, mx)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res[0][0] == res[1][0]                  # every field identical on both ranks
    assert res[0][1] == res[1][1] == 3.0           # max over ranks
    w = synth.small_case(31, N=16, D=40, M=12, C=5, n_train=300)
    ref = fit_layer(w["A_train"], w["B"], 5, w["perm"], w["bias"])
    for name, dt in pdist.PARAM_FIELDS:
        assert res[1][0][name] == np.ascontiguousarray(ref[name], dtype=dt).tobytes(), name


def _worker_layers(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layers = None
        if rank == 0:
            w = synth.small_case(32, N=16, D=33, M=7, C=4, n_train=300)
            p1 = fit_layer(w["A_train"], w["B"], 4, w["perm"], w["bias"])
            w2 = synth.small_case(33, N=16, D=7, M=3, C=2, n_train=300)
            p2 = fit_layer(w2["A_train"], w2["B"], 2, w2["perm"], w2["bias"])
            layers = [p1, p2]
        got = pdist.broadcast_layers(layers, torch.device("cpu"))
        q.put((rank, [{k: (np.asarray(v).tobytes() if not isinstance(v, int) else v) for k, v in p.items()}
                      for p in got]))
    finally:
        dist.destroy_process_group()


def test_broadcast_layers_one_payload_gloo_world2():
    """Several layers (an MLP) in one packed payload: identical on both ranks, equal to the fit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_layers, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert res[0] == res[1] and len(res[0]) == 2
    assert (res[1][0]["D"], res[1][0]["C"], res[1][0]["M"]) == (33, 4, 7)
    assert (res[1][1]["D"], res[1][1]["C"], res[1][1]["M"]) == (7, 2, 3)


def test_pack_params_round_trip_and_single_payload():
    w = synth.small_case(34, N=16, D=29, M=5, C=3, n_train=200)
    p = fit_layer(w["A_train"], w["B"], 3, w["perm"], w["bias"])
    hdr, payload = pdist.pack_params([p])
    assert hdr.tolist() == [1, 29, 3, 5] and payload.dtype == np.uint8 and payload.size % 4 == 0
    q = pdist.unpack_params(hdr, payload)[0]
    for name, dt in pdist.PARAM_FIELDS:
        assert np.array_equal(np.asarray(p[name], dt), q[name]), name


def _worker_shard_gpu(rank, world, port, q, N):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import fit as ofit
        from paper_2207_05808_b200 import Plan
        params = None
        if rank == 0:
            w = synth.small_case(35, N=16, D=300, M=600, C=64, n_train=800)
            params = ofit.fit(w["A_train"], w["B"], 64, w["perm"], w["bias"])
        params = pdist.broadcast_params(params, torch.device("cpu"))
        r0, r1 = pdist.shard_rows(N, world, rank)
        A = synth.rows("mnist", 135, 0, r0, r1, 300)              # the rank's rows of the seeded stream
        y = Plan(params, device=0).amm(torch.from_numpy(A).cuda(), relu=True)
        torch.cuda.synchronize()
        q.put((rank, y.cpu().numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_row_sharded_ranks_equal_single_gpu_and_oracle():
    """World size 2 on one GPU (gloo for the broadcast; the ranks' kernels never wait on each
    other): each rank runs its contiguous shard of a fixed N through Plan.amm (a streamed-LUT,
    several-slice shape).  The concatenated shard outputs equal the single-process output and the
    oracle bit for bit (row-parallel bit identity)."""
    import oracle
    from oracle import fit as ofit
    from paper_2207_05808_b200 import Plan
    N = 5001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_shard_gpu, args=(r, 2, port, q, N)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ys = np.concatenate([np.frombuffer(res[r], np.float32).reshape(-1, 600) for r in range(2)])
    w = synth.small_case(35, N=16, D=300, M=600, C=64, n_train=800)
    params = ofit.fit(w["A_train"], w["B"], 64, w["perm"], w["bias"])
    A = synth.rows("mnist", 135, 0, 0, N, 300)
    y1 = Plan(params, device=0).amm(torch.from_numpy(A).cuda(), relu=True).cpu().numpy()
    ref = oracle.amm(params, A, relu=True, nthreads=8)["y"]
    assert ys.shape == (N, 600)
    assert np.array_equal(ys.view(np.uint32), y1.view(np.uint32))
    assert np.array_equal(ys.view(np.uint32), ref.view(np.uint32))
