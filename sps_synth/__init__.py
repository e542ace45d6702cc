"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic: it only draws data sets
(X, y) with the shapes, value distributions and class balance of the paper's
workloads (Table 1) as recipes in DESIGN.md "Input recipe",
and fixed seeds.  The Gaussian prior the method uses is built by the method's
own g-prior helper (oracle or library), not here.
"""
from __future__ import annotations

import numpy as np

DATA_SEED = 1304

# name -> (n, k, C, J, N, g, n_cont, intercepts, slope_sd)
CONFIGS = {
    # configs[0]: tiny binary case the oracle finishes in seconds
    "cfg1": dict(n=100, k=4, C=2, J=4, N=128, g=0.25, n_cont=1, intercept=(0.0,), slope_sd=0.5),
    # configs[1]: German-credit shape (n=1000, k=25, ~30% positives), g = 1/16
    "cfg2": dict(n=1000, k=25, C=2, J=64, N=1024, g=1.0 / 16, n_cont=3, intercept=(-0.85,), slope_sd=0.3),
    # configs[2]: multinomial C=4, k=10 (Transportation-like), g = 1
    "cfg3": dict(n=5000, k=10, C=4, J=128, N=1024, g=1.0, n_cont=9, intercept=(0.3, -0.2, 0.1), slope_sd=0.3),
    # configs[3]: large binary, n=1e5, k=100
    "cfg4": dict(n=100000, k=100, C=2, J=1024, N=1024, g=0.25, n_cont=30, intercept=(0.0,), slope_sd=0.15),
}


def make_data(n: int, k: int, C: int, n_cont: int, intercept, slope_sd: float, seed: int = DATA_SEED):
    """X[:,0] = 1; n_cont N(0,1) columns; the rest Bernoulli(p_j), p_j ~ U(0.1, 0.5).
    y drawn from the multinomial logit with reference label 0 and a true
    coefficient draw (intercepts given, slopes N(0, slope_sd^2))."""
    rng = np.random.default_rng(seed)
    X = np.empty((n, k), dtype=np.float64)
    X[:, 0] = 1.0
    n_cont = min(n_cont, k - 1)
    if n_cont > 0:
        X[:, 1:1 + n_cont] = rng.standard_normal((n, n_cont))
    nb = k - 1 - n_cont
    if nb > 0:
        pj = rng.uniform(0.1, 0.5, size=nb)
        X[:, 1 + n_cont:] = (rng.uniform(size=(n, nb)) < pj).astype(np.float64)
    B = np.zeros((C, k))
    for c in range(1, C):
        B[c, 0] = intercept[(c - 1) % len(intercept)]
        B[c, 1:] = rng.normal(0.0, slope_sd, size=k - 1)
    # data-generating process only (not the method): draw y_t with softmax probabilities
    eta = X @ B.T
    eta -= eta.max(axis=1, keepdims=True)
    pr = np.exp(eta)
    pr /= pr.sum(axis=1, keepdims=True)
    cum = np.cumsum(pr, axis=1)
    u = rng.uniform(size=(n, 1))
    y = np.minimum((u > cum).sum(axis=1), C - 1).astype(np.int32)
    return X, y


def config_data(name: str, n: int | None = None, seed: int = DATA_SEED):
    c = CONFIGS[name]
    return make_data(n or c["n"], c["k"], c["C"], c["n_cont"], c["intercept"], c["slope_sd"], seed)


def particles(P: int, d: int, scale: float = 0.3, seed: int = 7):
    """Random particle matrix theta (P x d) for loglik parity/bench inputs."""
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, scale, size=(P, d))
