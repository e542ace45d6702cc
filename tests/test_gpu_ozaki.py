"""K1 on the INT8 tensor cores (ozaki.cuh): binary model, 64 <= k <= 128, the
contraction x~_t' theta_p rebuilt from 7 x 7 int8 slices (levels a + b <= 6) accumulated in TMEM by
tcgen05.mma.kind::i8.  Bar: the north_star's 1e-10 relative per-particle log-likelihood against the
oracle ("evaluate to machine accuracy"), on ragged particle and observation tiles,
single-observation and empty ranges, chunk starts that are not tile aligned, wide dynamic ranges of
X and theta, and the extreme |eta| paths of the epilogue."""
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


@pytest.fixture(autouse=True)
def _int8_path_for_every_range(monkeypatch):
    """The engine takes the INT8 path only for ranges >= 512 observations (below, the FP64 DMMA kernel
    is faster); these tests exercise it on short ranges too (read at sps_create)."""
    monkeypatch.setenv("SPS_OZ_MINRANGE", "1")


def _case(sps, orc, X, y, theta, t0, t1):
    import torch

    n, k = X.shape
    s = sps.Sps(X, y, np.zeros(k), np.eye(k), J=2, N=4, seed=1)
    got = s.loglik_tensor(torch.tensor(theta, device="cuda"), t0, t1).cpu().numpy()
    s.close()
    want = orc.loglik_range(theta, X, y, 2, t0, t1)
    err = np.abs(got - want)
    assert np.all(err <= LL_RTOL * np.abs(want) + 1e-300), (err / np.maximum(np.abs(want), 1e-300)).max()
    return got


@pytest.mark.parametrize("k", [64, 65, 80, 100, 120])
def test_ozaki_loglik_shapes(sps, orc, k):
    rng = np.random.default_rng(900 + k)
    n = 333  # 11 observation tiles of 32, ragged
    X = np.column_stack([np.ones(n), rng.normal(size=(n, 30)), (rng.uniform(size=(n, k - 31)) < 0.3)])
    y = rng.integers(0, 2, n).astype(np.int32)
    P = 1000 + 37  # ragged particle tiles of 128
    theta = rng.normal(0, 0.15, (P, k))
    _case(sps, orc, X, y, theta, 0, n)
    _case(sps, orc, X, y, theta, 17, 301)   # chunk bounds inside observation tiles
    _case(sps, orc, X, y, theta[:5], 40, 41)  # one observation
    got = _case(sps, orc, X, y, theta[:200], 100, 100)  # empty range
    assert np.all(got == 0.0)


def test_ozaki_dynamic_range_and_extremes(sps, orc):
    rng = np.random.default_rng(11)
    n, k = 257, 100
    X = np.column_stack([np.ones(n), rng.normal(size=(n, k - 1)) * np.exp(rng.uniform(-6, 6, k - 1))])
    y = rng.integers(0, 2, n).astype(np.int32)
    theta = np.concatenate([rng.normal(0, 1e-3, (128, k)) * np.exp(rng.uniform(-4, 4, k)),
                            rng.normal(0, 5.0, (64, k)),       # |eta| >> 708: clamp path
                            np.zeros((8, k))])                 # theta = 0 -> -n log 2
    got = _case(sps, orc, X, y, theta, 0, n)
    assert np.allclose(got[-8:], -n * math.log(2), rtol=1e-14)


def test_ozaki_cfg4_shard_full_data(sps, orc):
    """configs[3] shape: n = 1e5, k = 100, one GPU's shard of 128 x 1024 particles; full-data L_p on
    64 sampled particles against the oracle."""
    import torch

    X, y = sps_synth.config_data("cfg4")
    P = 131072
    theta = sps_synth.particles(P, 100, scale=0.05, seed=4)
    s = sps.Sps(X, y, np.zeros(100), np.eye(100), J=2, N=4, seed=1)
    got = s.loglik_tensor(torch.tensor(theta, device="cuda")).cpu().numpy()
    s.close()
    idx = np.random.default_rng(3).choice(P, 64, replace=False)
    want = orc.loglik_range(theta[idx], X, y, 2)
    assert np.all(np.abs(got[idx] - want) <= LL_RTOL * np.abs(want))


_RUN = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_1304_4333_b200 as sps, sps_synth
X, y = sps_synth.make_data(200, 100, 2, 30, (0.0,), 0.15, seed=5)
s = sps.Sps(X, y, np.zeros(100), sps.g_prior(X, 2, 0.25), J=8, N=128, seed=2)
r = s.run()
s.close()
print("RESULT" + json.dumps(dict(L=r["L"], R=[int(v) for v in r["R_cycle"]], logml=r["logml"], mean=list(r["mean"]))))
"""


def test_ozaki_whole_run_engine_modes():
    """A d = 100 run (K1 on the INT8 tensor cores inside the M-step graphs: the particle images are
    allocated at create, never inside a capture) gives the same result bit for bit under the device
    loop, per-step graph replays and plain launches, and the FP64 DMMA kernel's schedule and log ML."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for tag, env in (("loop", {}), ("noloop", {"SPS_NO_LOOP": "1"}), ("nograph", {"SPS_NO_GRAPH": "1"}),
                     ("dmma", {"SPS_NO_OZAKI": "1"})):
        e = dict(os.environ)
        e.update(env)
        p = subprocess.run([sys.executable, "-c", _RUN.format(root=root)], env=e, capture_output=True, text=True,
                           timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        out[tag] = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("RESULT")][-1][6:])
    assert out["loop"] == out["noloop"] == out["nograph"]
    assert out["dmma"]["L"] == out["loop"]["L"] and out["dmma"]["R"] == out["loop"]["R"]
    assert abs(out["dmma"]["logml"] - out["loop"]["logml"]) <= 1e-9


def test_ozaki_nonfinite_theta_reported(sps):
    """A NaN in theta makes L_p NaN on the INT8 path too (the row scale carries it), so sps_sync reports
    SPS_E_NUMERIC naming the particle."""
    import torch

    X, y = sps_synth.config_data("cfg4", n=300)
    s = sps.Sps(X, y, np.zeros(100), np.eye(100), J=2, N=4, seed=1)
    th = torch.tensor(sps_synth.particles(500, 100, scale=0.05), device="cuda")
    th[321, 57] = float("nan")
    out = torch.empty(500, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    s.loglik(th.data_ptr(), 500, 100, 0, 300, out.data_ptr())
    with pytest.raises(sps.SpsError) as e:
        s.sync()
    assert e.value.status == 4 and "p = 321" in str(e.value) and "t = 0" in str(e.value)
    s.close()


def test_ozaki_run_parity_power_vs_oracle(sps, orc):
    """A whole Algorithm 2 run with K1 on the INT8 tensor cores (d = 100) under power tempering -- every
    M step evaluates the full-data likelihood of theta* -- against the oracle (data tempering at d = 100:
    tests/test_gpu_large.py::test_run_parity_large_d, which takes the same K1 path)."""
    X, y = sps_synth.make_data(150, 100, 2, 30, (0.0,), 0.15, seed=7)
    cov = orc.g_prior(X, 2, 0.25)
    o = orc.run(X, y, 2, 8, 128, seed=3, prior_mean=np.zeros(100), prior_cov=cov, tempering=orc.POWER)
    s = sps.Sps(X, y, np.zeros(100), cov, J=8, N=128, seed=3, tempering=1)
    g = s.run()
    s.close()
    assert o["status"] == 0 and g["L"] == o["L"]
    assert np.array_equal(g["R_cycle"], o["R_cycle"])
    assert np.allclose(g["phi_cycle"], o["phi_cycle"], rtol=0, atol=1e-12)
    assert abs(g["logml"] - o["logml"]) <= 1e-6
    assert np.all(np.abs(g["mean"] - o["mean"]) <= 1e-6)


def test_ozaki_switch_within_run_vs_oracle(sps, orc, monkeypatch):
    """Default switch (INT8 path for ranges >= 512 observations, FP64 DMMA below) inside one run: k = 40,
    n = 600, the late cycles' M steps cross 512 -- the schedule, log ML and means match the oracle."""
    monkeypatch.delenv("SPS_OZ_MINRANGE", raising=False)
    X, y = sps_synth.make_data(600, 40, 2, 12, (-0.5,), 0.3, seed=21)
    cov = orc.g_prior(X, 2, 0.25)
    o = orc.run(X, y, 2, 8, 128, seed=4, prior_mean=np.zeros(40), prior_cov=cov)
    s = sps.Sps(X, y, np.zeros(40), cov, J=8, N=128, seed=4)
    g = s.run()
    s.close()
    assert o["status"] == 0 and o["t_cycle"][-2] >= 512  # the last cycles run K1 on the INT8 path
    assert g["L"] == o["L"] and np.array_equal(g["t_cycle"], o["t_cycle"])
    assert np.array_equal(g["R_cycle"], o["R_cycle"])
    assert abs(g["logml"] - o["logml"]) <= 1e-6
    assert np.all(np.abs(g["mean"] - o["mean"]) <= 1e-6)
