"""Pins for the oracle's model arithmetic (PAPER.md:115-128 eq. plogit,
PAPER.md:637-685 priors): closed forms, invariants, and a 120-digit decimal
evaluation of the softmax written independently here."""
import math
from decimal import Decimal, getcontext

import numpy as np
import pytest

getcontext().prec = 120


def hp_logp(theta, x, y, C):
    """log P(Y=y|x,theta) in 120-digit decimal; theta blocks 1..C-1, eta_0 = 0."""
    k = len(x)
    etas = [Decimal(0)]
    for c in range(1, C):
        s = Decimal(0)
        for i in range(k):
            s += Decimal(float(theta[(c - 1) * k + i])) * Decimal(float(x[i]))
        etas.append(s)
    den = sum((e.exp() for e in etas), Decimal(0))
    return etas[y] - den.ln()


def test_logp_closed_forms(orc):
    x = np.array([1.0, -0.3, 2.0])
    for C in (2, 3, 4, 7):
        th = np.zeros(3 * (C - 1))
        for y in range(C):
            assert abs(orc.logp(th, x, y, C) - math.log(1.0 / C)) < 1e-15
    # C=2, eta = log 2, y = 1 (non-reference) -> log(2/3); y = 0 -> log(1/3)
    th = np.array([math.log(2.0), 0.0, 0.0])
    assert abs(orc.logp(th, np.array([1.0, 5.0, -1.0]), 1, 2) - math.log(2 / 3)) < 1e-15
    assert abs(orc.logp(th, np.array([1.0, 5.0, -1.0]), 0, 2) - math.log(1 / 3)) < 1e-15


@pytest.mark.parametrize("C", [2, 3, 4])
def test_logp_probabilities_sum_to_one(orc, C):
    rng = np.random.default_rng(C)
    for _ in range(50):
        k = 5
        th = rng.normal(0, 2, k * (C - 1))
        x = rng.normal(0, 1, k)
        tot = sum(math.exp(orc.logp(th, x, y, C)) for y in range(C))
        assert abs(tot - 1.0) < 1e-12


@pytest.mark.parametrize("C", [2, 3, 4])
def test_logp_matches_high_precision(orc, C):
    rng = np.random.default_rng(10 + C)
    for scale in (0.1, 1.0, 10.0, 40.0):
        for _ in range(10):
            k = 4
            th = rng.normal(0, scale, k * (C - 1))
            x = rng.normal(0, 1, k)
            y = int(rng.integers(C))
            want = hp_logp(th, x, y, C)
            got = orc.logp(th, x, y, C)
            # relative error bounded by the conditioning |eta| eps of the dot products
            assert abs(Decimal(got) - want) <= Decimal(1e-13) * abs(want) + Decimal(1e-300)


def test_logp_shift_invariance_via_reference(orc):
    """Changing the reference category (adding -theta_c to every block,
    PAPER.md:649-658) leaves log-probabilities unchanged."""
    rng = np.random.default_rng(3)
    C, k = 4, 3
    full = rng.normal(0, 1, (C, k))
    full[0] = 0.0
    x = rng.normal(0, 1, k)
    for ref in range(C):
        shifted = full - full[ref]
        # relabel so that `ref` becomes label 0
        order = [ref] + [c for c in range(C) if c != ref]
        th = np.concatenate([shifted[c] for c in order[1:]])
        for y in range(C):
            assert abs(orc.logp(th, x, order.index(y), C) - orc.logp(full[1:].ravel(), x, y, C)) < 1e-13


def test_loglik_range_additive_and_high_precision(orc):
    rng = np.random.default_rng(4)
    n, k, C, P = 40, 3, 3, 6
    X = rng.normal(0, 1, (n, k))
    y = rng.integers(0, C, n).astype(np.int32)
    th = rng.normal(0, 1, (P, k * (C - 1)))
    full = orc.loglik_range(th, X, y, C, 0, n)
    a = orc.loglik_range(th, X, y, C, 0, 17)
    b = orc.loglik_range(th, X, y, C, 17, n)
    assert np.allclose(a + b, full, rtol=1e-13, atol=0)
    assert np.all(orc.loglik_range(th, X, y, C, 5, 5) == 0.0)  # empty range
    for p in range(P):
        want = sum((hp_logp(th[p], X[t], int(y[t]), C) for t in range(n)), Decimal(0))
        assert abs(Decimal(full[p]) - want) <= Decimal(1e-13) * abs(want)
    # theta = 0 -> -n log C exactly (up to rounding of the sum)
    z = orc.loglik_range(np.zeros((2, k * (C - 1))), X, y, C)
    assert np.allclose(z, -n * math.log(C), rtol=1e-14)


def test_loglik_extreme_separation_relative_accuracy(orc):
    """|eta| ~ 40: every term ~ -e^-40; the log1p form keeps relative accuracy."""
    n, k = 30, 2
    X = np.column_stack([np.ones(n), np.linspace(1, 2, n)])
    y = np.ones(n, dtype=np.int32)
    th = np.array([[20.0, 15.0]])
    got = orc.loglik_range(th, X, y, 2)[0]
    want = sum((hp_logp(th[0], X[t], 1, 2) for t in range(n)), Decimal(0))
    assert abs(Decimal(got) - want) <= Decimal(1e-13) * abs(want)


def test_cholesky_and_prior_quad(orc):
    rng = np.random.default_rng(5)
    d = 7
    A = rng.normal(0, 1, (d, d))
    S = A @ A.T + d * np.eye(d)
    L = orc.cholesky(S)
    assert np.allclose(np.triu(L, 1), 0)
    assert np.allclose(L @ L.T, S, rtol=1e-13, atol=1e-13)
    mu = rng.normal(0, 1, d)
    assert orc.prior_quad(L, mu, mu) == 0.0
    for _ in range(5):
        th = rng.normal(0, 1, d)
        want = -0.5 * (th - mu) @ np.linalg.solve(S, th - mu)
        assert abs(orc.prior_quad(L, mu, th) - want) < 1e-12 * abs(want)
        # symmetry f(mu + delta) = f(mu - delta)
        assert abs(orc.prior_quad(L, mu, 2 * mu - th) - orc.prior_quad(L, mu, th)) < 1e-12 * abs(want)
    with pytest.raises(np.linalg.LinAlgError):
        orc.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))


def test_g_prior_orthonormal_design(orc):
    """X'X = T I  ->  Sigma = g I, blocks 2 Sigma / Sigma."""
    T, k, g = 64, 4, 0.25
    Q, _ = np.linalg.qr(np.random.default_rng(6).normal(size=(T, k)))
    X = Q * math.sqrt(T)
    cov2 = orc.g_prior(X, 2, g)
    assert np.allclose(cov2, 2 * g * np.eye(k), atol=1e-12)
    cov3 = orc.g_prior(X, 3, g)
    want = np.block([[2 * g * np.eye(k), g * np.eye(k)], [g * np.eye(k), 2 * g * np.eye(k)]])
    assert np.allclose(cov3, want, atol=1e-12)


def test_g_prior_log_odds_variance_is_2gk(orc):
    """R9: the average prior variance of the log odds x_t'theta under the
    printed Sigma = g T (X'X)^-1 equals 2 g k, not the 2 g of PAPER.md:674-678."""
    rng = np.random.default_rng(7)
    T, k, g = 500, 6, 1.0 / 16
    X = np.column_stack([np.ones(T), rng.normal(size=(T, k - 1))])
    cov = orc.g_prior(X, 2, g)
    avg = np.mean([X[t] @ cov @ X[t] for t in range(T)])
    assert abs(avg - 2 * g * k) < 1e-10
