"""world_size-2 gloo tests (CPU) of the host side of the N > 1 path:
the NCCL unique id that bench.py broadcasts from rank 0 arrives intact on every
rank, and the group-sharded exchange protocol of the engine (each rank owns
J/G contiguous groups; slices are all-gathered and combined in rank order,
DESIGN.md "Multi-GPU") reproduces the unsharded statistics bit for bit and
gives identical decisions on every rank.  bench.py's own multi-rank helpers
(plan_workload, broadcast_id, max_over_ranks) run under gloo as they do under
NCCL, and the library's loopback all-gather (the exchange primitive of the
sharded engine's in-process transport, libsps.so host code) runs on host
threads without a device."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slice_stats(theta, J, N, G, r, shift):
    """Per-rank slice, laid out like the engine's stats slice: [J/G x d group sums | d x d M]."""
    Jl = J // G
    d = theta.shape[1]
    th = theta[r * Jl * N:(r + 1) * Jl * N]
    gs = th.reshape(Jl, N, d).sum(axis=1)
    c = th - shift
    M = c.T @ c
    return np.concatenate([gs.ravel(), M.ravel()])


def _combine(gathered, J, N, G, d, shift, a):
    """Rank-order combination (as finalize_body): theta-bar, V, RNE of monitor a."""
    Jl = J // G
    S = np.concatenate([g[:Jl * d].reshape(Jl, d) for g in gathered])
    M = sum(g[Jl * d:].reshape(d, d) for g in gathered)
    P = J * N
    bar = S.sum(axis=0) / P
    V = (M - P * np.outer(bar - shift, bar - shift)) / (P - 1)
    gj = S @ a / N
    vhat = N / (J - 1) * ((gj - gj.mean()) ** 2).sum()
    rne = (a @ V @ a) * (P - 1) / P / vhat
    return bar, V, rne


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. NCCL unique id from rank 0 reaches every rank intact
        import paper_1304_4333_b200 as sps

        ids = [sps.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        allid = [None] * world
        dist.all_gather_object(allid, ids[0])
        ok_id = len(ids[0]) == 128 and all(x == ids[0] for x in allid)
        # 2. sharded exchange protocol
        J, N, d = 8, 64, 5
        rng = np.random.default_rng(0)  # same particles on every rank
        theta = rng.normal(size=(J * N, d)) + rng.normal(size=(J, 1, d)).repeat(N, 1).reshape(J * N, d) * 0.1
        shift = theta[:7].mean(axis=0)
        a = np.linspace(0.5, 1.5, d)
        mine = _slice_stats(theta, J, N, world, rank, shift)
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        bar, V, rne = _combine(gathered, J, N, world, d, shift, a)
        ref = _combine([_slice_stats(theta, J, N, 1, 0, shift)], J, N, 1, d, shift, a)
        res = [None] * world
        dist.all_gather_object(res, (bar.tobytes(), V.tobytes(), float(rne)))
        same_on_ranks = all(x == res[0] for x in res)
        close_to_ref = np.allclose(bar, ref[0], rtol=1e-13) and np.allclose(V, ref[1], rtol=1e-12) and \
            abs(rne - ref[2]) < 1e-12 * ref[2]
        # 3. bench.py's multi-rank helpers, exactly as the N > 1 bench calls them (gloo instead of NCCL)
        import bench

        bid = bench.broadcast_id(dist, rank, sps.nccl_unique_id)
        allb = [None] * world
        dist.all_gather_object(allb, bid)
        ok_bench_id = len(bid) == 128 and all(x == bid for x in allb) and bid != ids[0]  # fresh id per call
        tmax = bench.max_over_ranks(dist, world, 10.0 + rank * 2.5, "cpu")
        plan = bench.plan_workload(world)
        ok_bench = ok_bench_id and tmax == 10.0 + (world - 1) * 2.5 and plan["scaling"] == "strong" and \
            plan["J"] * plan["N"] == 1 << 20 and plan["J"] % world == 0
        q.put((rank, ok_id, same_on_ranks, close_to_ref and ok_bench))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_protocol(world):
    import paper_1304_4333_b200 as sps

    sps.build()  # the ranks load libsps.so (ncclGetUniqueId needs no GPU)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_id, same, close in out:
        assert ok_id and same and close, (rank, ok_id, same, close)


@pytest.mark.parametrize("G", [2, 3, 8])
def test_library_loopback_allgather_host_threads(G):
    """libsps.so's loopback all-gather (sps_test_loopback_allgather; host only): G threads, 40 rounds of
    varying sizes (0 included) -- every rank receives all ranks' bytes in rank order every round, and
    fast ranks never overwrite a round the slow ones are still reading (double-buffered generations)."""
    import threading

    import paper_1304_4333_b200 as sps
    from paper_1304_4333_b200 import api

    sps.build()
    lid = sps.loopback_unique_id()
    rounds = 40
    sizes = [(37 * r) % 1001 for r in range(rounds)]
    payload = lambda rank, r: np.full(sizes[r], (rank * 41 + r * 7) % 251, dtype=np.uint8)  # noqa: E731
    got = {}
    errs = []

    def worker(rank):
        try:
            for r in range(rounds):
                got[(rank, r)] = api.test_loopback_allgather(lid, rank, G, payload(rank, r))
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(q,)) for q in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    assert not errs, errs
    for r in range(rounds):
        want = np.concatenate([payload(q, r) for q in range(G)])
        for rank in range(G):
            assert np.array_equal(got[(rank, r)], want), (rank, r)


def test_library_loopback_allgather_bad_args():
    import paper_1304_4333_b200 as sps
    from paper_1304_4333_b200 import api

    sps.build()
    lid = sps.loopback_unique_id()
    with pytest.raises(sps.SpsError):
        api.test_loopback_allgather(lid, 2, 2, np.zeros(4, np.uint8))  # rank >= G
    with pytest.raises(sps.SpsError):
        api.test_loopback_allgather(b"not-a-loopback-id".ljust(128, b"\0"), 0, 1, np.zeros(4, np.uint8))
    assert np.array_equal(api.test_loopback_allgather(lid, 0, 1, np.arange(5, dtype=np.uint8)), np.arange(5))
    with pytest.raises(sps.SpsError):  # the group was registered with G = 1
        api.test_loopback_allgather(lid, 0, 2, np.zeros(4, np.uint8))
