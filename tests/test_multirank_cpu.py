"""world_size-2 gloo tests (CPU) of the host side of the N > 1 path:
the NCCL unique id that bench.py broadcasts from rank 0 arrives intact on every
rank, and the group-sharded exchange protocol of the engine (each rank owns
J/G contiguous groups; slices are all-gathered and combined in rank order,
DESIGN.md "Multi-GPU") reproduces the unsharded statistics bit for bit and
gives identical decisions on every rank."""
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
        q.put((rank, ok_id, same_on_ranks, close_to_ref))
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
