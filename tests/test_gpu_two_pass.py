"""GPU parity of Algorithm 3 (two passes) through the C ABI
(sps_record_sigma / sps_get_sigma / sps_set_design / sps_run):

* pass 1 records the same design as the oracle's pass 1 on the same streams:
  identical t_l / phi_l, R_l, and Sigma_lr = (h/100) V_lr within the rounding
  of two summation orders of V (shifted one-pass moments on the GPU, two-pass
  in the oracle; R11);
* pass 2 with a given design (stream pass tag 1, fixed t_l, R_l, Sigma_lr)
  matches the oracle's pass 2 with the same design: identical schedule and h
  trace, log ML and posterior moments within 1e-6 absolute (north_star bar).
"""
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


def _compare(g, o):
    assert g["L"] == o["L"]
    assert np.array_equal(g["t_cycle"], o["t_cycle"])
    assert np.array_equal(g["phi_cycle"], o["phi_cycle"])
    assert np.array_equal(g["R_cycle"], o["R_cycle"])
    assert np.array_equal(g["h_cycle"], o["h_cycle"])
    assert abs(g["logml"] - o["logml"]) <= 1e-6
    assert abs(g["logml_nse"] - o["logml_nse"]) <= 1e-6
    for key in ("mean", "sd", "nse"):
        assert np.all(np.abs(g[key] - o[key]) <= 1e-6), key
    if "logpl" in o:
        assert np.all(np.abs(g["logpl"] - o["logpl"]) <= 1e-9)


def _sigma_close(a, b):
    """Sigma_lr of both sides: equal up to summation-order rounding of V."""
    assert a.shape == b.shape
    scale = np.sqrt(np.abs(np.einsum("sii->si", b)))  # per-step coordinate sd
    tol = 1e-9 * scale[:, :, None] * scale[:, None, :]
    assert np.all(np.abs(a - b) <= tol)


@pytest.mark.parametrize("tempering", [0, 1])
def test_two_pass_parity_cfg1(sps, orc, tempering):
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    mu = np.zeros(4)
    o1, o2 = orc.two_pass(X, y, 2, 4, 128, 5, 6, mu, cov, tempering=tempering)
    assert o1["status"] == 0 and o2["status"] == 0
    s = sps.Sps(X, y, mu, cov, J=4, N=128, seed=5, tempering=tempering)
    g1, g2 = s.two_pass(5, 6)
    # pass 1: same adaptive run as the oracle's, same recorded design
    _compare(g1, o1)
    _sigma_close(g1["sigma"], o1["sigma"])
    # pass 2 on the oracle's design, both sides fed identical Sigma_lr
    s.reset(6, 1)
    s.set_design(o1)
    g2o = s.run()
    s.set_design(None)
    _compare(g2o, o2)
    # the GPU's own pass 2 (its own design) against the oracle replaying that design
    o2g = orc.run(X, y, 2, 4, 128, 6, mu, cov, tempering=tempering, replay=g1, pass_=1)
    _compare(g2, o2g)
    assert g2["total_m_steps"] == g1["total_m_steps"]
    # pass 2 reruns the fixed design: R_l and t_l of pass 1, not its own adaptive choices
    assert np.array_equal(g2["R_cycle"], g1["R_cycle"]) and np.array_equal(g2["t_cycle"], g1["t_cycle"])
    s.close()


def test_two_pass_parity_multinomial(sps, orc):
    X, y = sps_synth.make_data(120, 3, 3, 2, (0.2, -0.3), 0.4, seed=11)
    cov = orc.g_prior(X, 3, 0.5)
    d = 6
    mu = np.zeros(d)
    o1, o2 = orc.two_pass(X, y, 3, 4, 256, 7, 8, mu, cov)
    s = sps.Sps(X, y, mu, cov, J=4, N=256, seed=7, C_=3)
    g1, _ = s.two_pass(7, 8)
    _compare(g1, o1)
    _sigma_close(g1["sigma"], o1["sigma"])
    s.reset(8, 1)
    s.set_design(o1)
    g2 = s.run()
    s.close()
    _compare(g2, o2)


def test_design_replay_of_its_own_pass_is_exact(sps, orc):
    """Replaying pass 1's own design with pass 1's seed and pass tag reproduces pass 1
    step for step (the design is exactly what the adaptive run did)."""
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=9)
    s.record_sigma(True)
    g1 = s.run()
    g1["sigma"] = s.sigma(0, g1["total_m_steps"])
    s.record_sigma(False)
    s.reset(9, 0)
    s.set_design(g1)
    g1r = s.run()
    s.set_design(None)
    s.close()
    for key in ("t_cycle", "R_cycle", "h_cycle"):
        assert np.array_equal(g1r[key], g1[key])
    assert g1r["logml"] == g1["logml"]
    assert np.array_equal(g1r["mean"], g1["mean"])


def test_design_api_errors(sps):
    X, y = sps_synth.config_data("cfg1")
    s = sps.Sps(X, y, np.zeros(4), np.eye(4), J=4, N=128, seed=1)
    with pytest.raises(sps.SpsError):
        s.sigma(0, 1)  # nothing recorded
    bad = dict(t_cycle=[50, 40], R_cycle=[1, 1], sigma=np.tile(np.eye(4), (2, 1, 1)))
    with pytest.raises(sps.SpsError):
        s.set_design(bad)
    s.close()


def test_sigma_record_grows_across_phases(sps, orc):
    """A small max_m_steps makes the Sigma_lr record reserve per M phase (mstep + max_m_steps + 2)
    and grow several times during the run; the record still matches the oracle's, step for step."""
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    o1 = orc.run(X, y, 2, 4, 128, 3, np.zeros(4), cov, record_sigma=True, max_m_steps=30)
    s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=3, max_m_steps=30)
    s.record_sigma(True)
    g1 = s.run()
    sig = s.sigma(0, g1["total_m_steps"])
    with pytest.raises(sps.SpsError):
        s.sigma(0, g1["total_m_steps"] + 5)  # beyond the steps run
    s.close()
    _compare(g1, o1)
    _sigma_close(sig, o1["sigma"])
