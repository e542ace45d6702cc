"""Pins for the oracle's random streams (R15).

Philox4x32-10 is pinned by the Random123 known-answer tests; the conversions
by exact arithmetic; the portable elementary functions by the platform libm
(an independent implementation) to a few ulp; the normals by their moments
and a Kolmogorov-Smirnov test against scipy's normal CDF.
"""
import math

import numpy as np
import pytest
from scipy import stats


# Random123 kat_vectors for philox4x32_10 (Salmon et al., SC'11).
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_kat(orc, ctr, key, want):
    assert tuple(orc.philox(ctr, key)) == want


def test_u01_exact(orc):
    assert orc.u01(0, 0) == 2.0**-53
    assert orc.u01(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0**-53
    # 2*(x>>12)+1 over 2^53, exact
    hi, lo = 0x12345678, 0x9ABCDEF0
    x = (hi << 32) | lo
    assert orc.u01(hi, lo) == (2 * (x >> 12) + 1) / 2.0**53


def _ulps(a, b):
    return abs(a - b) / math.ulp(max(abs(b), 1e-300))


def test_plog_matches_libm(orc):
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(2.0**-53, 1.0, 2000), 2.0 ** -rng.uniform(0, 60, 2000), [1.0, 0.5, 2.0**-53]])
    worst = max(_ulps(orc.plog(x), math.log(x)) for x in xs if x != 1.0)
    assert worst <= 2.0
    assert orc.plog(1.0) == 0.0
    for e in range(1, 60):  # exact powers of two: e * ln2 split
        assert abs(orc.plog(2.0**-e) - (-e * math.log(2))) <= 2 * math.ulp(e * math.log(2))


def test_pexp_matches_libm(orc):
    rng = np.random.default_rng(1)
    xs = np.concatenate([-rng.uniform(0, 700, 3000), -rng.uniform(0, 1, 1000), [0.0, -1e-300]])
    worst = max(_ulps(orc.pexp(x), math.exp(x)) for x in xs)
    assert worst <= 4.0
    assert orc.pexp(0.0) == 1.0
    assert orc.pexp(-709.0) == 0.0  # R8: below -708 the weight is defined as 0


def test_psincos_matches_libm(orc):
    import mpmath

    mpmath.mp.dps = 40
    rng = np.random.default_rng(2)
    for u in rng.uniform(0, 1, 2000):
        s, c = orc.psincos2pi(u)
        a = 2 * mpmath.pi * mpmath.mpf(float(u))  # exact u, exact 2 pi u
        assert abs(s - float(mpmath.sin(a))) <= 3e-16
        assert abs(c - float(mpmath.cos(a))) <= 3e-16
    assert orc.psincos2pi(0.25) == (1.0, 0.0) or orc.psincos2pi(0.25)[1] == -0.0


def test_normals_distribution(orc):
    z = np.concatenate([orc.normals(99, p, 3, orc.TAG_PROPOSAL, 50) for p in range(2000)])
    n = z.size
    assert abs(z.mean()) < 4 / math.sqrt(n)
    assert abs(z.var() - 1) < 4 * math.sqrt(2 / n)
    assert stats.kstest(z, "norm").pvalue > 1e-3
    # streams keyed by (id, step, tag): distinct keys give distinct draws
    a = orc.normals(99, 0, 0, orc.TAG_PROPOSAL, 8)
    b = orc.normals(99, 0, 1, orc.TAG_PROPOSAL, 8)
    c = orc.normals(99, 0, 0, orc.TAG_INIT, 8)
    assert not np.array_equal(a, b) and not np.array_equal(a, c)
    # odd counts take the cosine half of the last block
    assert np.array_equal(orc.normals(5, 1, 2, 2, 7), orc.normals(5, 1, 2, 2, 8)[:7])


def test_box_muller_construction(orc):
    """z_0 = sqrt(-2 log u1) cos(2 pi u2) with (u1, u2) from block 0."""
    seed, p, step = 1234567890123, 17, 5
    w = orc.philox([0, p, step, orc.TAG_PROPOSAL], [seed & 0xFFFFFFFF, seed >> 32])
    u1, u2 = orc.u01(w[0], w[1]), orc.u01(w[2], w[3])
    z = orc.normals(seed, p, step, orc.TAG_PROPOSAL, 2)
    r = math.sqrt(-2 * math.log(u1))
    assert abs(z[0] - r * math.cos(2 * math.pi * u2)) < 1e-14
    assert abs(z[1] - r * math.sin(2 * math.pi * u2)) < 1e-14


def test_accept_and_resample_uniforms(orc):
    us = np.array([orc.accept_uniform(3, p, 9) for p in range(20000)])
    assert us.min() > 0 and us.max() < 1
    assert stats.kstest(us, "uniform").pvalue > 1e-3
    a = np.array([orc.resample_a52(3, 2, 7, r) for r in range(20000)], dtype=np.float64)
    assert a.max() < 2.0**52
    assert stats.kstest((2 * a + 1) / 2.0**53, "uniform").pvalue > 1e-3
    # draw r uses block r//2, word pair r%2
    w = orc.philox([1, 2, 7, orc.TAG_RESAMPLE], [3, 0])
    assert orc.resample_a52(3, 2, 7, 3) == (((w[2] << 32) | w[3]) >> 12)
