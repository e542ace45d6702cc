"""Pins for the oracle's SPS pieces: ESS, resampling
(PAPER.md:297-305), NSE/RNE (Table 5 golden fixture), and
the power-tempering search (R5)."""
import csv
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_ess_arithmetic(orc):
    assert orc.ess(np.zeros(37)) == pytest.approx(37.0, rel=1e-15)
    lw = np.log(np.array([2.0, 1.0, 1.0, 1e-300]))  # weights {2,1,1,~0}: 16/6
    assert orc.ess(lw) == pytest.approx(16.0 / 6.0, rel=1e-14)
    lw = np.array([0.0] + [-1e4] * 9)
    assert orc.ess(lw) == 1.0
    rng = np.random.default_rng(0)
    for _ in range(50):
        lw = rng.normal(0, rng.uniform(0.1, 30), 200)
        e = orc.ess(lw)
        assert 1.0 <= e <= 200.0
        # shift invariance (max subtraction): +-500
        assert orc.ess(lw + 500) == pytest.approx(e, rel=1e-12)
        assert orc.ess(lw - 500) == pytest.approx(e, rel=1e-12)
        w = np.exp(lw - lw.max())
        assert e == pytest.approx(w.sum() ** 2 / (w ** 2).sum(), rel=1e-12)


def test_resample_deterministic_cases(orc):
    N = 8
    q = np.full(N, 2**32, dtype=np.uint64)
    for scheme in (orc.RESIDUAL, orc.SYSTEMATIC):
        assert np.array_equal(orc.resample_int(q, scheme, np.zeros(N, np.uint64)), np.arange(N))
    q = np.array([2**31, 2**31, 0, 0], dtype=np.uint64)  # normalized {.5,.5,0,0}
    assert list(orc.resample_int(q, orc.RESIDUAL, np.zeros(4, np.uint64))) == [0, 0, 1, 1]


def _counts(anc, N):
    return np.bincount(anc, minlength=N)


@pytest.mark.parametrize("scheme", [0, 1, 2])
def test_resample_unbiased(orc, scheme):
    """E[count_n] = N q_n / Q (Chopin 2004), 4000 replications."""
    rng = np.random.default_rng(1 + scheme)
    N = 16
    q = rng.integers(0, 2**32, N).astype(np.uint64)
    q[3] = 0
    Q = int(q.sum())
    R = 4000
    tot = np.zeros(N)
    sq = np.zeros(N)
    for r in range(R):
        a = rng.integers(0, 2**52, N, dtype=np.uint64)
        c = _counts(orc.resample_int(q, scheme, a), N)
        assert c.sum() == N and c[3] == 0
        expect = N * q.astype(float) / Q
        if scheme == orc.RESIDUAL:
            assert np.all(c >= np.floor(N * q.astype(object) // Q).astype(int))
        if scheme == orc.SYSTEMATIC:  # counts are floor or ceil of N w
            assert np.all((c == np.floor(expect)) | (c == np.ceil(expect)))
        tot += c
        sq += c * c
    mean = tot / R
    se = np.sqrt(np.maximum(sq / R - mean**2, 1e-12) / R)
    assert np.all(np.abs(mean - N * q.astype(float) / Q) <= 4 * se + 1e-9)


def test_resample_group_uses_stream_and_is_ascending(orc):
    rng = np.random.default_rng(3)
    lw = rng.normal(0, 2, 64)
    a = orc.resample_group(lw, orc.RESIDUAL, 11, 5, 2)
    b = orc.resample_group(lw, orc.RESIDUAL, 11, 5, 2)
    assert np.array_equal(a, b) and np.all(np.diff(a) >= 0)
    # equals the integer core fed q_n = floor(pexp(lw-max) 2^32) and the RESAMPLE draws
    q = np.array([math.floor(orc.pexp(v - lw.max()) * 2.0**32) for v in lw], dtype=np.uint64)
    draws = np.array([orc.resample_a52(11, 5, 2, r) for r in range(64)], dtype=np.uint64)
    assert np.array_equal(a, orc.resample_int(q, orc.RESIDUAL, draws))
    # uniform weights -> identity (residual copies every particle once)
    assert np.array_equal(orc.resample_group(np.full(64, -3.0), orc.RESIDUAL, 1, 0, 1), np.arange(64))


def test_group_stats_spec_examples(orc):
    mean, sd, nse, rne = orc.group_stats(np.array([[0.0], [2.0]]))  # J=2, N=1 -> vhat=2, NSE=1
    assert mean == 1.0 and nse == pytest.approx(1.0)
    mean, sd, nse, rne = orc.group_stats(np.array([[0.0, 1.0], [1.0, 2.0]]))
    assert rne == pytest.approx(0.5) and mean == 1.0
    mean, sd, nse, rne = orc.group_stats(np.full((3, 4), 2.5))
    assert nse == 0.0 and rne == math.inf


def test_group_stats_identities(orc):
    rng = np.random.default_rng(4)
    for _ in range(20):
        J, N = int(rng.integers(2, 9)), int(rng.integers(1, 50))
        g = rng.normal(0, 1, (J, N)) + rng.normal(0, 0.3, (J, 1))
        mean, sd, nse, rne = orc.group_stats(g)
        gbar = g.mean()
        vhat = N / (J - 1) * ((g.mean(axis=1) - gbar) ** 2).sum()
        assert mean == pytest.approx(gbar, abs=1e-14)
        assert rne * vhat * J * N == pytest.approx(((g - gbar) ** 2).sum(), rel=1e-12)
        assert nse == pytest.approx(math.sqrt(vhat / (J * N)), rel=1e-12)
        assert nse == pytest.approx(sd / math.sqrt(rne * J * N), rel=1e-12)
        # permutation invariance
        assert orc.group_stats(g[::-1, ::-1])[0] == pytest.approx(mean, abs=1e-14)


def test_table5_pins_nse_reading():
    """R2: every SPS entry of Table 5 satisfies NSE = sd / (RNE J N)^1/2, i.e.
    NSE = [(JN)^-1 vhat]^1/2; the printed [J^-1 vhat]^1/2 matches none."""
    ok = mis = rows = 0
    with open(os.path.join(GOLDEN, "table5_sps.csv")) as f:
        for row in csv.reader(line for line in f if not line.startswith("#")):
            _, _, _, J, N, sd_s, nse_s, rne_s, _ = row
            J, N, sd, nse, rne = int(J), int(N), float(sd_s), float(nse_s), float(rne_s)
            half = 0.5 * 10 ** -len(nse_s.split(".")[1])
            lo = (sd - 5e-4) / math.sqrt((rne + 5e-3) * J * N) - half
            hi = (sd + 5e-4) / math.sqrt((rne - 5e-3) * J * N) + half
            ok += lo <= nse <= hi
            vhat = sd**2 / rne
            mis += abs(math.sqrt(vhat / J) - nse) <= half
            rows += 1
    assert rows == 52
    assert ok >= 48  # 4 rows carry other misprints (Germany GPU, Cars GPU, Caesarean 2 GPU)
    assert mis == 0


def test_power_search_brackets_threshold(orc):
    rng = np.random.default_rng(5)
    P = 500
    L = rng.normal(-300, 40, P)
    rem = 1.0
    dphi = orc.power_search(L, rem)
    q = round(dphi / 2.0**-48)
    assert dphi == (q * 2.0**-48) * rem

    def ess_at(dp):
        w = np.exp(dp * (L - L.max()))
        return w.sum() ** 2 / (w ** 2).sum()

    assert ess_at(dphi) >= 0.5 * P
    assert ess_at(((q + 1) * 2.0**-48) * rem) < 0.5 * P
    # flat log-likelihood: the whole remaining increment is taken
    assert orc.power_search(np.full(P, -3.0), 0.37) == 0.37
