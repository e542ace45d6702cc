"""Pins for the oracle's whole Algorithm 2 run: limiting
cases the paper states, invariants of the trace, and the d <= 2 quadrature
posterior (tests/quadrature.py)."""
import math

import numpy as np
import pytest

import sps_synth
from tests import quadrature


def _tiny_binary(n=40, seed=3):
    rng = np.random.default_rng(seed)
    X = np.column_stack([np.ones(n), rng.normal(size=n)])
    p = 1 / (1 + np.exp(-(0.3 + 0.8 * X[:, 1])))
    y = (rng.uniform(size=n) < p).astype(np.int32)
    return X, y


def test_flat_likelihood_one_cycle(orc):
    """X = 0: every particle has the same likelihood, ESS never drops (uniform
    weights), one cycle, logML = T log(1/C)."""
    n, k, C = 25, 3, 3
    X = np.zeros((n, k))
    y = (np.arange(n) % C).astype(np.int32)
    d = k * (C - 1)
    r = orc.run(X, y, C, 4, 64, seed=2, prior_mean=np.zeros(d), prior_cov=np.eye(d),
                monitors=np.eye(d)[:2])
    assert r["status"] == 0 and r["L"] == 1 and list(r["t_cycle"]) == [n]
    assert r["logml"] == pytest.approx(n * math.log(1.0 / C), rel=1e-13)
    assert r["logml_nse"] < 1e-12


def test_dogmatic_prior_one_cycle(orc):
    X, y = _tiny_binary()
    r = orc.run(X, y, 2, 4, 64, seed=2, prior_mean=np.array([0.3, 0.8]), prior_cov=1e-14 * np.eye(2))
    assert r["status"] == 0 and r["L"] == 1


def test_trace_invariants_and_determinism(orc):
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    a = orc.run(X, y, 2, 4, 128, seed=5, prior_mean=np.zeros(4), prior_cov=cov, n_threads=1)
    b = orc.run(X, y, 2, 4, 128, seed=5, prior_mean=np.zeros(4), prior_cov=cov, n_threads=4)
    assert a["status"] == 0
    for key in ("logml", "mean", "sd", "t_cycle", "R_cycle", "h_cycle"):
        assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), key
    t = a["t_cycle"]
    assert np.all(np.diff(t) > 0) and t[-1] == 100
    assert np.all(a["R_cycle"] >= 1)
    assert np.all((a["h_cycle"] >= 10) & (a["h_cycle"] <= 100))
    h_prev = 50
    for R, h in zip(a["R_cycle"], a["h_cycle"]):  # h moves by one hundredth per step
        assert abs(h - h_prev) <= R
        h_prev = h
    assert np.all(a["min_rne"][:-1] >= 0.35) and a["min_rne"][-1] >= 0.9
    assert a["logml"] == pytest.approx(a["logml_inc"].sum(), abs=1e-10)
    c = orc.run(X, y, 2, 4, 128, seed=6, prior_mean=np.zeros(4), prior_cov=cov)
    assert c["logml"] != a["logml"]


@pytest.mark.parametrize("mode", ["data", "power"])
def test_quadrature_binary_d2(orc, mode):
    """Binary intercept + slope (d=2): posterior mean of theta'xbar and logML
    within 3 NSE of the quadrature values in >= 8 of 10 seeds."""
    X, y = _tiny_binary()
    cov = orc.g_prior(X, 2, 0.25)
    fn = X.mean(axis=0)[None, :]
    qml, qmean = quadrature.posterior(X, y, 2, np.zeros(2), cov, fn)
    qml2, _ = quadrature.posterior(X, y, 2, np.zeros(2), cov, fn, nodes=401)
    assert abs(qml - qml2) < 1e-8  # quadrature self-convergence
    ok_m = ok_l = 0
    for seed in range(1, 11):
        r = orc.run(X, y, 2, 10, 400, seed=seed, prior_mean=np.zeros(2), prior_cov=cov,
                    tempering=orc.DATA if mode == "data" else orc.POWER)
        assert r["status"] == 0
        ok_m += abs(r["mean"][0] - qmean[0]) <= 3 * r["nse"][0]
        ok_l += abs(r["logml"] - qml) <= 3 * r["logml_nse"]
    assert ok_m >= 8 and ok_l >= 8, (ok_m, ok_l)


def test_quadrature_multinomial_intercepts(orc):
    """C=3 intercept-only model (d=2), exchangeable g-prior."""
    rng = np.random.default_rng(9)
    n = 30
    X = np.ones((n, 1))
    y = rng.choice(3, size=n, p=[0.5, 0.3, 0.2]).astype(np.int32)
    cov = orc.g_prior(X, 3, 1.0)
    fns = np.eye(2)
    qml, qmean = quadrature.posterior(X, y, 3, np.zeros(2), cov, fns)
    ok = 0
    for seed in range(1, 11):
        r = orc.run(X, y, 3, 10, 400, seed=seed, prior_mean=np.zeros(2), prior_cov=cov, report_fns=fns)
        assert r["status"] == 0
        ok += (np.all(np.abs(r["mean"] - qmean) <= 3 * r["nse"])
               and abs(r["logml"] - qml) <= 3 * r["logml_nse"])
    assert ok >= 8, ok


def test_resampling_schemes_agree(orc):
    X, y = _tiny_binary()
    cov = orc.g_prior(X, 2, 0.25)
    fn = X.mean(axis=0)[None, :]
    _, qmean = quadrature.posterior(X, y, 2, np.zeros(2), cov, fn)
    for scheme in (orc.SYSTEMATIC, orc.MULTINOMIAL):
        r = orc.run(X, y, 2, 10, 400, seed=4, prior_mean=np.zeros(2), prior_cov=cov, resampling=scheme)
        assert r["status"] == 0
        assert abs(r["mean"][0] - qmean[0]) <= 4 * r["nse"][0]


@pytest.mark.parametrize("mode", ["data", "power"])
def test_two_pass_quadrature_and_agreement(orc, mode):
    """Algorithm 3: pass 2 replays pass 1's design exactly (same L, t_l / phi_l, R_l)
    with fresh random numbers; its posterior mean and logML are within 3 NSE of the quadrature values in
    >= 8 of 10 seeds (the fixed-design SMC the CLT covers), and pass 1 and pass 2 agree within 3 combined
    NSE in >= 8 of 10 (the paper's Table 2 property)."""
    X, y = _tiny_binary()
    cov = orc.g_prior(X, 2, 0.25)
    fn = X.mean(axis=0)[None, :]
    qml, qmean = quadrature.posterior(X, y, 2, np.zeros(2), cov, fn)
    ok_m = ok_l = ok_a = 0
    tmp = orc.DATA if mode == "data" else orc.POWER
    for seed in range(1, 11):
        p1, p2 = orc.two_pass(X, y, 2, 10, 400, seed, 5000 + seed, np.zeros(2), cov, tempering=tmp)
        assert p1["status"] == 0 and p2 is not None and p2["status"] == 0
        assert p2["L"] == p1["L"] and list(p2["R_cycle"]) == list(p1["R_cycle"])
        if mode == "data":
            assert list(p2["t_cycle"]) == list(p1["t_cycle"])
        else:
            assert list(p2["phi_cycle"]) == list(p1["phi_cycle"])
        assert p1["sigma"].shape == (p1["total_m_steps"], 2, 2)
        ok_m += abs(p2["mean"][0] - qmean[0]) <= 3 * p2["nse"][0]
        ok_l += abs(p2["logml"] - qml) <= 3 * p2["logml_nse"]
        ok_a += abs(p1["logml"] - p2["logml"]) <= 3 * math.hypot(p1["logml_nse"], p2["logml_nse"])
    assert ok_m >= 8 and ok_l >= 8 and ok_a >= 8, (ok_m, ok_l, ok_a)


def test_two_pass_sigma_is_the_pass1_proposal(orc):
    """The recorded Sigma_lr are the matrices pass 1 factored: symmetric positive definite, and replaying
    them with pass 1's own seed and pass tag reproduces pass 1 exactly (same particles, same logML)."""
    X, y = _tiny_binary()
    cov = orc.g_prior(X, 2, 0.25)
    p1 = orc.run(X, y, 2, 4, 128, seed=3, prior_mean=np.zeros(2), prior_cov=cov, record_sigma=True,
                 return_theta=True)
    for S in p1["sigma"]:
        assert np.allclose(S, S.T) and np.all(np.linalg.eigvalsh(S) > 0)
    again = orc.run(X, y, 2, 4, 128, seed=3, prior_mean=np.zeros(2), prior_cov=cov, replay=p1, return_theta=True)
    assert again["logml"] == p1["logml"] and np.array_equal(again["theta"], p1["theta"])


# ---------------------------------------------------------------- log predictive likelihoods (R18)
def test_predictive_flat_likelihood(orc):
    """X = 0: p(y_s | theta) = 1/C for every theta, so every one-step-ahead predictive
    probability is exactly 1/C whatever the weights."""
    n, k, C = 25, 3, 3
    X = np.zeros((n, k))
    y = (np.arange(n) % C).astype(np.int32)
    d = k * (C - 1)
    r = orc.run(X, y, C, 4, 64, seed=2, prior_mean=np.zeros(d), prior_cov=np.eye(d), monitors=np.eye(d)[:2])
    assert np.allclose(r["logpl"], math.log(1.0 / C), rtol=1e-13, atol=0)


def test_predictive_chain_rule(orc):
    """p(y_{1:T}) = prod_s p(y_s | y_{1:s-1}): the predictive log likelihoods add up to the log ML,
    cycle by cycle (the cycle's increment) and in total."""
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    r = orc.run(X, y, 2, 4, 128, seed=5, prior_mean=np.zeros(4), prior_cov=cov)
    lp = r["logpl"]
    assert np.all(np.isfinite(lp)) and np.all(lp < 0)
    assert lp.sum() == pytest.approx(r["logml"], abs=1e-10)
    t0 = 0
    for t, inc in zip(r["t_cycle"], r["logml_inc"]):
        assert lp[t0:t].sum() == pytest.approx(inc, abs=1e-11)
        t0 = t


def test_predictive_quadrature_prefixes(orc):
    """Cumulative predictive sum_{s<=t} log p(y_s|y_{1:s-1}) = log p(y_{1:t}): against the d=2
    quadrature log ML of the first t observations, within 3 NSE in >= 8 of 10 seeds, at
    t = 10, 20, 30 (the intermediate posteriors' particle representations)."""
    X, y = _tiny_binary()
    cov = orc.g_prior(X, 2, 0.25)
    fn = X.mean(axis=0)[None, :]
    ts = (10, 20, 30)
    q = {t: quadrature.posterior(X[:t], y[:t], 2, np.zeros(2), cov, fn)[0] for t in ts}
    ok = 0
    for seed in range(1, 11):
        r = orc.run(X, y, 2, 10, 400, seed=seed, prior_mean=np.zeros(2), prior_cov=cov)
        cum = np.cumsum(r["logpl"])
        ok += all(abs(cum[t - 1] - q[t]) <= 3 * r["logml_nse"] for t in ts)
    assert ok >= 8, ok
