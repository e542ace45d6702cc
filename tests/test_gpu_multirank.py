"""Sharded (G > 1) engine on one GPU through the in-process loopback transport
(include/sps.h sps_loopback_unique_id): one host thread per rank, each with its
own context and stream; exchange steps meet at a host barrier (no kernel waits
on another rank).  The sharded run must reproduce the single-rank run (same
cycle schedule, M-step counts, h trace; log ML and moments to 1e-9) and the
oracle (1e-6), and the ranks' particle shards must concatenate to the
single-rank particles."""
import threading

import numpy as np
import pytest

import sps_synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sps():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1304_4333_b200 as pkg

    pkg.build()
    return pkg


def _sharded(sps, G, X, y, cov, J, N, seed, **kw):
    lid = sps.loopback_unique_id()
    out = [None] * G
    errs = []

    def worker(r):
        try:
            s = sps.Sps(X, y, np.zeros(cov.shape[0]), cov, J=J, N=N, seed=seed, rank=r, nranks=G, nccl_id=lid, **kw)
            assert s.J_local == J // G and s.group0 == r * J // G
            rep = s.run()
            out[r] = (rep, s.particles())
            s.close()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("tempering", [0, 1])
def test_loopback_sharded_matches_single_rank(sps, orc, G, tempering):
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    J, N, seed = 8, 128, 3
    s = sps.Sps(X, y, np.zeros(4), cov, J=J, N=N, seed=seed, tempering=tempering)
    single = s.run()
    th1, L1, lp1 = s.particles()
    s.close()
    res = _sharded(sps, G, X, y, cov, J, N, seed, tempering=tempering)
    for r, (rep, (th, L, lp)) in enumerate(res):
        assert rep["L"] == single["L"]
        assert np.array_equal(rep["t_cycle"], single["t_cycle"])
        assert np.array_equal(rep["R_cycle"], single["R_cycle"])
        assert np.array_equal(rep["h_cycle"], single["h_cycle"])
        assert abs(rep["logml"] - single["logml"]) < 1e-9
        assert abs(rep["logml_nse"] - single["logml_nse"]) < 1e-9
        assert np.allclose(rep["mean"], single["mean"], atol=1e-9, rtol=0)
        assert rep["pairs"] == single["pairs"]
    th = np.concatenate([r[1][0] for r in res])
    assert np.allclose(th, th1, atol=1e-11, rtol=0)
    o = orc.run(X, y, 2, J, N, seed=seed, prior_mean=np.zeros(4), prior_cov=cov, tempering=tempering)
    assert abs(res[0][0]["logml"] - o["logml"]) <= 1e-6
    assert np.all(np.abs(res[0][0]["mean"] - o["mean"]) <= 1e-6)


def test_loopback_sharded_two_pass_and_predictive(sps, orc):
    """Algorithm 3 pass 2 (fixed design: the ESS partials are still gathered for the predictive
    likelihoods, Sigma_lr replayed on every rank) and the log predictive likelihoods, sharded over
    G = 2 loopback ranks, against the single-rank context on the same design."""
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    J, N = 8, 128
    o1, o2 = orc.two_pass(X, y, 2, J, N, 4, 5, np.zeros(4), cov)
    s = sps.Sps(X, y, np.zeros(4), cov, J=J, N=N, seed=5, pass_=1)
    s.set_design(o1)
    single = s.run()
    s.close()
    lid = sps.loopback_unique_id()
    out = [None] * 2
    errs = []

    def worker(r):
        try:
            c = sps.Sps(X, y, np.zeros(4), cov, J=J, N=N, seed=5, pass_=1, rank=r, nranks=2, nccl_id=lid)
            c.set_design(o1)
            out[r] = c.run()
            c.close()
        except Exception as e:
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    for rep in out:
        assert np.array_equal(rep["R_cycle"], single["R_cycle"]) and np.array_equal(rep["t_cycle"], single["t_cycle"])
        assert abs(rep["logml"] - single["logml"]) < 1e-9
        assert np.allclose(rep["logpl"], single["logpl"], atol=1e-9, rtol=0)
        assert np.allclose(rep["mean"], single["mean"], atol=1e-9, rtol=0)
    assert abs(out[0]["logml"] - o2["logml"]) <= 1e-6
    assert np.all(np.abs(out[0]["logpl"] - o2["logpl"]) <= 1e-9)


def _check_sharded(res, single, o, tol_single=1e-9):
    for rep, _ in res:
        assert rep["L"] == single["L"] == o["L"]
        assert np.array_equal(rep["t_cycle"], single["t_cycle"]) and np.array_equal(rep["t_cycle"], o["t_cycle"])
        assert np.array_equal(rep["R_cycle"], single["R_cycle"]) and np.array_equal(rep["R_cycle"], o["R_cycle"])
        assert np.array_equal(rep["h_cycle"], single["h_cycle"])
        assert abs(rep["logml"] - single["logml"]) < tol_single
        assert np.allclose(rep["mean"], single["mean"], atol=tol_single, rtol=0)
    assert abs(res[0][0]["logml"] - o["logml"]) <= 1e-6
    assert abs(res[0][0]["logml_nse"] - o["logml_nse"]) <= 1e-6
    assert np.all(np.abs(res[0][0]["mean"] - o["mean"]) <= 1e-6)


@pytest.mark.parametrize("G", [2, 8])
def test_loopback_sharded_d25(sps, orc, G):
    """The bench shape's kernels (d = 25: k_propose_rb<7>, k_accept_tile<4>, warp Cholesky at d = 25) on
    the sharded path, G = 2 and 8 ranks of the German-credit-shaped data."""
    X, y = sps_synth.config_data("cfg2", n=300)
    cov = orc.g_prior(X, 2, 1.0 / 16)
    J, N, seed = 8, 256, 2
    s = sps.Sps(X, y, np.zeros(25), cov, J=J, N=N, seed=seed)
    single = s.run()
    s.close()
    o = orc.run(X, y, 2, J, N, seed=seed, prior_mean=np.zeros(25), prior_cov=cov)
    _check_sharded(_sharded(sps, G, X, y, cov, J, N, seed), single, o)


def test_large_J_unstaged_finalize(sps, orc):
    """J = 8192 groups (J x d too large to stage in the finalize block's shared memory): theta-bar and
    the monitor group means come from the column sums / group means k_mom_reduce writes into the stats
    slice -- single rank and G = 8 loopback ranks (1024 groups each) against the oracle."""
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    J, N, seed = 8192, 16, 1
    s = sps.Sps(X, y, np.zeros(4), cov, J=J, N=N, seed=seed)
    single = s.run()
    s.close()
    o = orc.run(X, y, 2, J, N, seed=seed, prior_mean=np.zeros(4), prior_cov=cov)
    assert o["status"] == 0
    _check_sharded([(single, None)], single, o)
    _check_sharded(_sharded(sps, 8, X, y, cov, J, N, seed), single, o)
