"""Brute-force posterior by tensor Gauss-Legendre quadrature for d <= 2.

Independent of oracle/ and of the CUDA path: its own numpy log-likelihood
(logaddexp), its own Gaussian log-density.  Used to pin the oracle's log
marginal likelihood and posterior means.
"""
from __future__ import annotations

import numpy as np
from scipy import optimize


def _loglik_grid(T, X, y, C):
    """T: (G, d) parameter points; returns (G,) sum_t log p(y_t | x_t, theta)."""
    n, k = X.shape
    G = T.shape[0]
    out = np.zeros(G)
    for t in range(n):
        etas = [np.zeros(G)] + [T[:, c * k:(c + 1) * k] @ X[t] for c in range(C - 1)]
        E = np.stack(etas, axis=1)
        lse = np.logaddexp.reduce(E, axis=1)
        out += E[:, y[t]] - lse
    return out


def _logprior(T, mu, cov):
    d = mu.shape[0]
    Ci = np.linalg.inv(cov)
    D = T - mu
    _, logdet = np.linalg.slogdet(cov)
    return -0.5 * np.einsum("gi,ij,gj->g", D, Ci, D) - 0.5 * d * np.log(2 * np.pi) - 0.5 * logdet


def posterior(X, y, C, mu, cov, fns, nodes=301, width=12.0):
    """Return (logML, E[f_i(theta)] for rows f_i of fns)."""
    X = np.asarray(X, float)
    mu = np.asarray(mu, float)
    cov = np.asarray(cov, float)
    d = mu.shape[0]
    assert d <= 2

    def nlp(th):
        return -(_loglik_grid(th[None, :], X, y, C)[0] + _logprior(th[None, :], mu, cov)[0])

    res = optimize.minimize(nlp, mu.copy(), method="BFGS", options=dict(gtol=1e-10))
    mode = res.x
    # numerical Hessian for the box
    h = 1e-4
    H = np.zeros((d, d))
    for i in range(d):
        for j in range(d):
            ei = np.eye(d)[i] * h
            ej = np.eye(d)[j] * h
            H[i, j] = (nlp(mode + ei + ej) - nlp(mode + ei - ej) - nlp(mode - ei + ej) + nlp(mode - ei - ej)) / (4 * h * h)
    sd = np.sqrt(np.diag(np.linalg.inv(H)))
    xg, wg = np.polynomial.legendre.leggauss(nodes)
    axes, wts = [], []
    for i in range(d):
        lo, hi = mode[i] - width * sd[i], mode[i] + width * sd[i]
        axes.append(0.5 * (hi - lo) * xg + 0.5 * (hi + lo))
        wts.append(0.5 * (hi - lo) * wg)
    if d == 1:
        T = axes[0][:, None]
        W = wts[0]
    else:
        A, B = np.meshgrid(axes[0], axes[1], indexing="ij")
        T = np.column_stack([A.ravel(), B.ravel()])
        W = np.outer(wts[0], wts[1]).ravel()
    lp = _loglik_grid(T, X, y, C) + _logprior(T, mu, cov)
    m = lp.max()
    wexp = W * np.exp(lp - m)
    Z = wexp.sum()
    logml = m + np.log(Z)
    means = [(wexp * (T @ f)).sum() / Z for f in np.atleast_2d(fns)]
    return float(logml), np.array(means)
