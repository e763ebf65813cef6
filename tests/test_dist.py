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
