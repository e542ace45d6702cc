"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element on the same seeded inputs.  Bars (BASELINE.json north_star):
bit-exact for random streams, resampling indices and accept decisions;
per-particle log-likelihood within 1e-10 relative; log ML and posterior
means within 1e-6 absolute."""
import math

import numpy as np
import pytest

import sps_synth

pytestmark = pytest.mark.gpu

LL_RTOL = 1e-10


@pytest.fixture(scope="module")
def sps():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1304_4333_b200 as pkg

    pkg.build()
    return pkg


@pytest.fixture(scope="module")
def api(sps):
    from paper_1304_4333_b200 import api

    return api


# ------------------------------------------------------------------ random streams
def test_philox_bit_exact(api, orc):
    rng = np.random.default_rng(0)
    ctrs = rng.integers(0, 2**32, size=(4096, 4), dtype=np.uint64).astype(np.uint32)
    key = np.array([0xA4093822, 0x299F31D0], dtype=np.uint32)
    got = api.test_philox(ctrs, key)
    for i in range(0, 4096, 37):
        assert list(got[i]) == orc.philox(ctrs[i], key)
    kat = api.test_philox(np.zeros((1, 4), np.uint32), np.zeros(2, np.uint32))
    assert list(kat[0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]


def test_normals_bit_exact(api, orc):
    for seed, ident, step, tag in [(1, 0, 0, 1), (2**40 + 5, 123, 77, 2), (9, 65535, 3, 2)]:
        a = api.test_normals(seed, ident, step, tag, 101)
        b = orc.normals(seed, ident, step, tag, 101)
        assert np.array_equal(a, b)


def test_portable_functions_bit_exact(api, orc):
    rng = np.random.default_rng(1)
    u = np.concatenate([rng.uniform(2**-53, 1, 20000), 2.0 ** -rng.uniform(0, 53, 5000)])
    assert np.array_equal(api.test_portable(0, u), np.array([orc.plog(x) for x in u]))
    x = -rng.uniform(0, 720, 20000)
    assert np.array_equal(api.test_portable(1, x), np.array([orc.pexp(v) for v in x]))
    sc = api.test_portable(2, u[:5000]).reshape(-1, 2)
    want = np.array([orc.psincos2pi(v) for v in u[:5000]])
    assert np.array_equal(sc, want)


# ------------------------------------------------------------------ resampling / accept
@pytest.mark.parametrize("scheme", [0, 1, 2])
@pytest.mark.parametrize("N", [1, 7, 128, 1000, 1024, 4099, 16384])
def test_resample_int_bit_exact(api, orc, scheme, N):
    rng = np.random.default_rng(N * 3 + scheme)
    for trial in range(3):
        q = rng.integers(0, 2**32 + 1, N, dtype=np.uint64)
        if trial == 1:
            q[rng.uniform(size=N) < 0.8] = 0  # sparse weights
        if trial == 2:
            q[:] = 0
            q[N // 2] = 2**32  # degenerate: one particle
        if q.sum() == 0:
            q[0] = 1
        a = rng.integers(0, 2**52, N, dtype=np.uint64)
        assert np.array_equal(api.test_resample_int(q, scheme, a), orc.resample_int(q, scheme, a))


@pytest.mark.parametrize("scheme", [0, 1, 2])
def test_resample_group_bit_exact(api, orc, scheme):
    rng = np.random.default_rng(10 + scheme)
    for N, sd in [(128, 0.5), (1024, 3.0), (1000, 30.0), (4096, 1e-3)]:
        lw = rng.normal(0, sd, N) - 50
        got = api.test_resample_group(lw, scheme, 77, 3, 11)
        assert np.array_equal(got, orc.resample_group(lw, scheme, 77, 3, 11))


def test_accept_bit_exact(api, orc):
    rng = np.random.default_rng(5)
    P = 20000
    seed, step = 123456789, 42
    u = np.array([orc.accept_uniform(seed, p, step) for p in range(P)])
    logu = np.array([orc.plog(v) for v in u])
    delta = logu + rng.choice([-1e-12, 0.0, 1e-12, -1.0, 1.0], size=P)  # ties and near-ties
    delta[::7] = rng.normal(0, 3, delta[::7].size)
    got = api.test_accept(delta, seed, step)
    want = (logu < delta).astype(np.uint8)
    assert np.array_equal(got, want)


# ------------------------------------------------------------------ log-likelihood
def _loglik_case(sps, orc, X, y, C, theta, t0, t1):
    import torch

    n, k = X.shape
    d = k * (C - 1)
    s = sps.Sps(X, y, np.zeros(d), np.eye(d), J=2, N=4, seed=1, C_=C)
    th = torch.tensor(theta, device="cuda")
    got = s.loglik_tensor(th, t0, t1).cpu().numpy()
    s.close()
    want = orc.loglik_range(theta, X, y, C, t0, t1)
    err = np.abs(got - want)
    tol = LL_RTOL * np.abs(want) + 1e-300
    assert np.all(err <= tol), (err / np.maximum(np.abs(want), 1e-300)).max()
    return got, want


@pytest.mark.parametrize("C,k", [(2, 1), (2, 4), (2, 7), (2, 25), (2, 32), (2, 42), (2, 64), (3, 4), (3, 10),
                                 (4, 10), (4, 16), (5, 6), (8, 3)])
def test_loglik_parity_shapes(sps, orc, C, k):
    rng = np.random.default_rng(100 + 10 * C + k)
    n = 333  # several chunks and a ragged tail
    X = np.column_stack([np.ones(n), rng.normal(size=(n, k - 1))]) if k > 1 else np.ones((n, 1))
    y = rng.integers(0, C, n).astype(np.int32)
    P = 1000 + 37  # ragged particle tiles
    theta = rng.normal(0, 0.4, (P, k * (C - 1)))
    _loglik_case(sps, orc, X, y, C, theta, 0, n)
    _loglik_case(sps, orc, X, y, C, theta[:5], 17, 18)  # one observation
    got, _ = _loglik_case(sps, orc, X, y, C, theta[:64], 100, 100)  # empty range
    assert np.all(got == 0.0)


def test_loglik_extreme_and_degenerate(sps, orc):
    rng = np.random.default_rng(7)
    n, k = 200, 5
    X = np.column_stack([np.ones(n), rng.normal(size=(n, k - 1))])
    y = rng.integers(0, 2, n).astype(np.int32)
    theta = np.concatenate([rng.normal(0, 20, (64, k)),      # |eta| up to ~100: e^-|s| underflow paths
                            rng.normal(0, 300, (16, k)),     # |eta| > 708: clamp path
                            np.zeros((8, k))])               # theta = 0 -> -n log 2
    got, want = _loglik_case(sps, orc, X, y, 2, theta, 0, n)
    assert np.allclose(got[-8:], -n * math.log(2), rtol=1e-14)


@pytest.mark.parametrize("C", [3, 4, 6])
def test_loglik_multinomial_extreme(sps, orc, C):
    """Multinomial K1: the unshifted 1 + sum e^eta form for |eta| < 704 and the max-shifted
    fallback (|eta| >= 704 in some class) on the same observations; theta = 0 -> -n log C."""
    rng = np.random.default_rng(70 + C)
    n, k = 150, 4
    X = np.column_stack([np.ones(n), rng.normal(size=(n, k - 1))])
    y = rng.integers(0, C, n).astype(np.int32)
    d = k * (C - 1)
    theta = np.concatenate([rng.normal(0, 30, (64, d)),     # |eta| up to ~200: large products of v
                            rng.normal(0, 400, (16, d)),    # |eta| > 704: shifted fallback
                            np.zeros((8, d))])
    theta[64:72, 0] = 705.0  # one class just past the switch, the rest moderate
    theta[64:72, 1:] = rng.normal(0, 0.1, (8, d - 1))
    got, _ = _loglik_case(sps, orc, X, y, C, theta, 0, n)
    assert np.allclose(got[-8:], -n * math.log(C), rtol=1e-14)


def test_loglik_full_size_cfg2_sampled(sps, orc):
    """configs[1] at full size (P = 65536, n = 1000) in the bench launch
    configuration; 512 sampled particles recomputed by the oracle."""
    import torch

    X, y = sps_synth.config_data("cfg2")
    P, d = 64 * 1024, 25
    theta = sps_synth.particles(P, d, scale=0.3)
    s = sps.Sps(X, y, np.zeros(d), np.eye(d), J=64, N=1024, seed=1)
    got = s.loglik_tensor(torch.tensor(theta, device="cuda")).cpu().numpy()
    s.close()
    idx = np.random.default_rng(0).choice(P, 512, replace=False)
    want = orc.loglik_range(theta[idx], X, y, 2)
    assert np.all(np.abs(got[idx] - want) <= LL_RTOL * np.abs(want))


def test_loglik_multinomial_cfg3_sampled(sps, orc):
    import torch

    X, y = sps_synth.config_data("cfg3")
    d = 30
    P = 8192
    theta = sps_synth.particles(P, d, scale=0.2, seed=3)
    s = sps.Sps(X, y, np.zeros(d), np.eye(d), J=8, N=1024, seed=1, C_=4)
    got = s.loglik_tensor(torch.tensor(theta, device="cuda")).cpu().numpy()
    s.close()
    idx = np.random.default_rng(1).choice(P, 128, replace=False)
    want = orc.loglik_range(theta[idx], X, y, 4)
    assert np.all(np.abs(got[idx] - want) <= LL_RTOL * np.abs(want))


# ------------------------------------------------------------------ whole runs
def _compare_runs(g, o):
    assert g["L"] == o["L"]
    assert np.array_equal(g["t_cycle"], o["t_cycle"])
    assert np.array_equal(g["R_cycle"], o["R_cycle"])
    assert np.array_equal(g["h_cycle"], o["h_cycle"])
    assert abs(g["logml"] - o["logml"]) <= 1e-6
    assert np.all(np.abs(g["mean"] - o["mean"]) <= 1e-6)
    assert np.all(np.abs(g["sd"] - o["sd"]) <= 1e-6)
    assert abs(g["logml_nse"] - o["logml_nse"]) <= 1e-6
    assert np.all(np.abs(g["nse"] - o["nse"]) <= 1e-6)
    if "logpl" in o:  # log predictive likelihoods (data tempering, R18)
        assert np.all(np.abs(g["logpl"] - o["logpl"]) <= 1e-9)


@pytest.mark.parametrize("tempering", [0, 1])
@pytest.mark.parametrize("seed", [1, 2])
def test_run_parity_cfg1(sps, orc, tempering, seed):
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    o = orc.run(X, y, 2, 4, 128, seed=seed, prior_mean=np.zeros(4), prior_cov=cov, tempering=tempering)
    s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=seed, tempering=tempering)
    g = s.run()
    s.close()
    assert o["status"] == 0
    _compare_runs(g, o)


@pytest.mark.parametrize("scheme", [1, 2])
def test_run_parity_resampling_schemes(sps, orc, scheme):
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    o = orc.run(X, y, 2, 4, 128, seed=3, prior_mean=np.zeros(4), prior_cov=cov, resampling=scheme)
    s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=3, resampling=scheme)
    g = s.run()
    s.close()
    _compare_runs(g, o)


def test_run_parity_multinomial(sps, orc):
    X, y = sps_synth.make_data(120, 3, 3, 2, (0.2, -0.3), 0.4, seed=11)
    cov = orc.g_prior(X, 3, 0.5)
    d = 6
    o = orc.run(X, y, 3, 4, 256, seed=4, prior_mean=np.zeros(d), prior_cov=cov)
    s = sps.Sps(X, y, np.zeros(d), cov, J=4, N=256, seed=4, C_=3)
    g = s.run()
    s.close()
    _compare_runs(g, o)


def test_g_prior_and_moments_match_oracle(sps, orc):
    X, y = sps_synth.config_data("cfg1")
    for C in (2, 3):
        assert np.allclose(sps.g_prior(X, C, 0.25), orc.g_prior(X, C, 0.25), rtol=1e-12, atol=1e-14)
    cov = orc.g_prior(X, 2, 0.25)
    s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=8)
    th, L, lp = s.particles()
    A = np.random.default_rng(0).normal(size=(3, 4))
    mean, sd, nse, rne = s.moments(A)
    s.close()
    for i in range(3):
        m2, sd2, nse2, rne2 = orc.group_stats((th @ A[i]).reshape(4, 128))
        assert abs(mean[i] - m2) < 1e-12 and abs(sd[i] - sd2) < 1e-10 and abs(nse[i] - nse2) < 1e-10
        assert abs(rne[i] - rne2) < 1e-8 * rne2
    # initial particles: the INIT stream through the prior factor, like the oracle
    Lp = orc.cholesky(cov)
    z = orc.normals(1 if False else 8, 5, 0, orc.TAG_INIT, 4)
    assert np.allclose(th[5], Lp @ z, rtol=1e-14, atol=1e-15)


def test_predictive_api(sps, orc):
    """sps_predictive between cycles: the absorbed prefix matches the oracle's full-run values
    (same streams), the rest is refused until absorbed; power tempering has none."""
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    o = orc.run(X, y, 2, 4, 128, seed=1, prior_mean=np.zeros(4), prior_cov=cov)
    s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=1)
    t, _, inc = s.cphase()
    got = s.predictive(0, t)
    assert np.all(np.abs(got - o["logpl"][:t]) <= 1e-9)
    assert abs(got.sum() - inc) <= 1e-10
    with pytest.raises(sps.SpsError):
        s.predictive(0, t + 1)
    s.close()
    s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=1, tempering=1)
    with pytest.raises(sps.SpsError):
        s.predictive(0, 1)
    s.close()


@pytest.mark.parametrize("C", [2, 3])
def test_cphase_scan_ragged_chunks(sps, orc, C):
    """Data-tempering C phase (K2 scan + K3 ESS) on a fixed schedule whose chunks are 1, 3, 7, 15
    and 34 observations (chunk quarters empty, ragged and uneven) over J x N = 3 x 11 particles
    (a partial particle block): after each C + S phase every particle's L equals its ancestor's L
    plus the oracle's log-likelihood of the absorbed observations, and the log-ML increment is the
    pooled log mean weight."""
    rng = np.random.default_rng(500 + C)
    n, k = 60, 5
    X = np.column_stack([np.ones(n), rng.normal(size=(n, k - 1))])
    y = rng.integers(0, C, n).astype(np.int32)
    d = k * (C - 1)
    s = sps.Sps(X, y, np.zeros(d), 0.25 * np.eye(d), J=3, N=11, seed=9, C_=C)
    try:
        t_prev = 0
        th0, L0, _ = s.particles()
        for t in [1, 4, 11, 26, 60]:
            t_new, _, inc = s.cphase(t_target=t)
            assert t_new == t
            lw = orc.loglik_range(th0, X, y, C, t_prev, t)
            want_inc = np.logaddexp.reduce(lw) - math.log(lw.size)
            assert abs(inc - want_inc) <= 1e-9 * max(1.0, abs(want_inc))
            th1, L1, _ = s.particles()
            for i in range(th1.shape[0]):
                a = np.flatnonzero(np.all(th0 == th1[i], axis=1))
                assert a.size >= 1, "resampled particle is not a copy of an ancestor"  # copies share L
                want = L0[a[0]] + lw[a[0]]
                assert abs(L1[i] - want) <= LL_RTOL * abs(want) + 1e-12
            th0, L0, t_prev = th1, L1, t
    finally:
        s.close()
