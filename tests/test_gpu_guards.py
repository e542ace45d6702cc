"""Out-of-bounds write check of every kernel family (include/sps.h sps_check_guards): with SPS_GUARD=1
each device buffer of a context sits between two 256-byte guard zones; after whole runs of every
engine path (data / power tempering, the d = 4 / 25 / 30 / 100 kernel instantiations, the INT8 K1,
the fused M step, Algorithm 3's record / replay, large J, the sharded engine, sps_loglik on ragged
particle counts and ranges) no zone may have been written.  compute-sanitizer is closed on this GPU
pool; this is the repo's own bounds check.  The detector itself is pinned by a planted 8-byte
overrun (SPS_GUARD_POKE) that must be reported naming the buffer."""
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


@pytest.fixture(autouse=True)
def _guarded(monkeypatch):
    monkeypatch.setenv("SPS_GUARD", "1")


def _run_checked(sps, X, y, cov, J, N, seed, **kw):
    s = sps.Sps(X, y, np.zeros(cov.shape[0]), cov, J=J, N=N, seed=seed, **kw)
    rep = s.run()
    s.check_guards()
    s.close()
    return rep


@pytest.mark.parametrize("tempering", [0, 1])
def test_guards_cfg1(sps, tempering):
    X, y = sps_synth.config_data("cfg1")
    rep = _run_checked(sps, X, y, sps.g_prior(X, 2, 0.25), 4, 128, 2, tempering=tempering)
    assert rep["L"] > 1


@pytest.mark.parametrize("tempering", [0, 1])
def test_guards_d25(sps, tempering):
    X, y = sps_synth.config_data("cfg2", n=300)
    _run_checked(sps, X, y, sps.g_prior(X, 2, 1.0 / 16), 8, 256, 1, tempering=tempering)


def test_guards_cfg2_full(sps):
    """The bench workload itself (J = 64 x N = 1024: the 16-CTA cluster reduce, persistent K1 grids)."""
    X, y = sps_synth.config_data("cfg2")
    _run_checked(sps, X, y, sps.g_prior(X, 2, 1.0 / 16), 64, 1024, 1)


def test_guards_multinomial(sps):
    X, y = sps_synth.config_data("cfg3", n=400)
    _run_checked(sps, X, y, sps.g_prior(X, 4, 1.0), 8, 256, 1, C_=4)


def test_guards_d100_int8_k1(sps, monkeypatch):
    monkeypatch.setenv("SPS_OZ_MINRANGE", "1")  # the INT8 K1 on every range
    X, y = sps_synth.make_data(200, 100, 2, 30, (0.0,), 0.15, seed=5)
    _run_checked(sps, X, y, sps.g_prior(X, 2, 0.25), 8, 128, 2)


@pytest.mark.parametrize("k", [4, 25])
def test_guards_fused_mstep(sps, monkeypatch, k):
    monkeypatch.setenv("SPS_FUSED", "1")
    if k == 4:
        X, y = sps_synth.config_data("cfg1")
    else:
        X, y = sps_synth.config_data("cfg2", n=300)
    _run_checked(sps, X, y, sps.g_prior(X, 2, 0.25), 8, 256, 3)


def test_guards_large_J(sps):
    """J = 8192 groups of 16: the finalize reads the group means from the slices (not staged)."""
    X, y = sps_synth.config_data("cfg2", n=200)
    _run_checked(sps, X, y, sps.g_prior(X, 2, 1.0 / 16), 8192, 16, 4)


def test_guards_two_pass_and_predictive(sps):
    X, y = sps_synth.config_data("cfg1")
    s = sps.Sps(X, y, np.zeros(4), sps.g_prior(X, 2, 0.25), J=4, N=128, seed=5)
    p1, p2 = s.two_pass(6, 7)
    assert p1["L"] == p2["L"]
    s.predictive()
    s.moments(np.eye(4))
    s.particles()
    s.check_guards()
    s.close()


def test_guards_loglik_ragged(sps):
    import torch

    X, y = sps_synth.config_data("cfg2", n=333)
    s = sps.Sps(X, y, np.zeros(25), np.eye(25), J=2, N=4, seed=1)
    for P, t0, t1 in ((1037, 0, 333), (1, 5, 6), (4097, 17, 301), (65, 0, 0), (300000, 0, 333)):
        th = torch.tensor(sps_synth.particles(P, 25, scale=0.1, seed=P), device="cuda")
        out = s.loglik_tensor(th, t0, t1)
        assert out.shape[0] == P
    s.check_guards()
    s.close()


def test_guards_sharded_loopback(sps):
    X, y = sps_synth.config_data("cfg2", n=300)
    cov = sps.g_prior(X, 2, 1.0 / 16)
    lid = sps.loopback_unique_id()
    errs = []

    def worker(r):
        try:
            s = sps.Sps(X, y, np.zeros(25), cov, J=8, N=128, seed=2, rank=r, nranks=2, nccl_id=lid)
            s.run()
            s.check_guards()
            s.close()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs


@pytest.mark.parametrize("name", ["&c->theta", "&c->part", "&c->slice"])
def test_guards_detect_planted_overrun(sps, monkeypatch, name):
    monkeypatch.setenv("SPS_GUARD_POKE", name)
    X, y = sps_synth.config_data("cfg1")
    s = sps.Sps(X, y, np.zeros(4), sps.g_prior(X, 2, 0.25), J=4, N=128, seed=2)
    with pytest.raises(sps.SpsError) as e:
        s.check_guards()
    assert e.value.status == 9 and name in str(e.value) and "8 bytes" in str(e.value)
    s.close()


def test_guards_off_is_config_error(sps, monkeypatch):
    monkeypatch.setenv("SPS_GUARD", "0")
    X, y = sps_synth.config_data("cfg1")
    s = sps.Sps(X, y, np.zeros(4), sps.g_prior(X, 2, 0.25), J=4, N=128, seed=2)
    with pytest.raises(sps.SpsError) as e:
        s.check_guards()
    assert e.value.status == 2
    s.close()
