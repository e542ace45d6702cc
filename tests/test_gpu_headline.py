"""GPU vs oracle whole-run parity at the shapes the bench and BASELINE.json configs run
(north_star: "logML and posterior moments match the oracle"; PAPER.md:813-816 log ML,
PAPER.md:160-223 moments), plus the boundary's error paths.

* d = 25 (German-credit shape, k = 25): the k_propose_rb<7> / k_accept_tile<4> / d = 25 warp
  Cholesky instantiations the bench runs;
* C = 4, k = 10 (d = 30, configs[2] shape): the multinomial K1 and the d = 30 M-step kernels;
* configs[1] at full size (n = 1000, k = 25, J = 64 x N = 1024, g = 1/16): the bench workload itself,
  including the 16-CTA cluster reduce over 64 groups; the oracle's wall time is written to
  gpurun_out/ as the same-config CPU figure.

Bars: identical cycle schedule t_l, M-step counts R_l and h trace; log ML, means, sd, NSE within 1e-6
absolute; the per-cycle min monitor RNE within 1e-6 relative."""
import json
import os
import platform
import subprocess
import time

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
    assert o["status"] == 0
    assert g["L"] == o["L"]
    assert np.array_equal(g["t_cycle"], o["t_cycle"])
    assert np.array_equal(g["R_cycle"], o["R_cycle"])
    assert np.array_equal(g["h_cycle"], o["h_cycle"])
    assert g["h_final"] == o["h_final"] and g["total_m_steps"] == o["total_m_steps"]
    assert np.allclose(g["min_rne"], o["min_rne"], rtol=1e-6, atol=0)
    assert np.all(np.abs(g["logml_inc"] - o["logml_inc"]) <= 1e-8)
    assert abs(g["logml"] - o["logml"]) <= 1e-6
    assert abs(g["logml_nse"] - o["logml_nse"]) <= 1e-6
    for key in ("mean", "sd", "nse"):
        assert np.all(np.abs(g[key] - o[key]) <= 1e-6), key
    assert np.allclose(g["rne"], o["rne"], rtol=1e-6)


@pytest.mark.parametrize("seed", [1, 2])
def test_run_parity_d25(sps, orc, seed):
    X, y = sps_synth.config_data("cfg2", n=300)
    cov = orc.g_prior(X, 2, 1.0 / 16)
    o = orc.run(X, y, 2, 8, 256, seed=seed, prior_mean=np.zeros(25), prior_cov=cov)
    s = sps.Sps(X, y, np.zeros(25), cov, J=8, N=256, seed=seed)
    g = s.run()
    s.close()
    _compare(g, o)


def test_run_parity_d25_power(sps, orc):
    X, y = sps_synth.config_data("cfg2", n=300)
    cov = orc.g_prior(X, 2, 1.0 / 16)
    o = orc.run(X, y, 2, 8, 256, seed=3, prior_mean=np.zeros(25), prior_cov=cov, tempering=orc.POWER)
    s = sps.Sps(X, y, np.zeros(25), cov, J=8, N=256, seed=3, tempering=1)
    g = s.run()
    s.close()
    _compare(g, o)
    # phi_l on the 2^-48 grid: the cached full-data L agree to summation-order rounding, so the search may
    # land one grid step apart (R5)
    assert np.allclose(g["phi_cycle"], o["phi_cycle"], rtol=0, atol=1e-12)


def test_run_parity_multinomial_c4_k10(sps, orc):
    X, y = sps_synth.config_data("cfg3", n=400)
    cov = orc.g_prior(X, 4, 1.0)
    o = orc.run(X, y, 4, 8, 256, seed=1, prior_mean=np.zeros(30), prior_cov=cov)
    s = sps.Sps(X, y, np.zeros(30), cov, J=8, N=256, seed=1, C_=4)
    g = s.run()
    s.close()
    _compare(g, o)


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def test_run_parity_cfg2_full(sps, orc):
    """configs[1] exactly as bench.py runs it (J = 64 x N = 1024, n = 1000, k = 25, g = 1/16, seed 1)."""
    X, y = sps_synth.config_data("cfg2")
    cov = orc.g_prior(X, 2, 1.0 / 16)
    s = sps.Sps(X, y, np.zeros(25), cov, J=64, N=1024, seed=1)
    g = s.run()
    s.close()
    t0 = time.perf_counter()
    o = orc.run(X, y, 2, 64, 1024, seed=1, prior_mean=np.zeros(25), prior_cov=cov, n_threads=os.cpu_count())
    dt = time.perf_counter() - t0
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "oracle_cfg2_full.json"), "w") as f:
        json.dump({"config": "configs[1]: n=1000, k=25, J=64 x N=1024, g=1/16, seed 1, data tempering",
                   "oracle_wall_s": dt, "pairs": o["pairs"], "pairs_per_s": o["pairs"] / dt,
                   "threads": os.cpu_count(), "cpu_model": _cpu_model(), "cycles": o["L"],
                   "m_steps": o["total_m_steps"], "logml_oracle": o["logml"], "logml_gpu": g["logml"]}, f, indent=1)
    _compare(g, o)


# ------------------------------------------------------------------ boundary error paths
def test_loglik_nonfinite_names_particle_and_observation(sps):
    """sps_loglik: a non-finite L_p is reported as SPS_E_NUMERIC naming (p, t) (
    PAPER.md:129-131), by the next sps_sync; the context stays usable."""
    import torch

    X, y = sps_synth.config_data("cfg2", n=300)
    cov = sps.g_prior(X, 2, 1.0 / 16)
    s = sps.Sps(X, y, np.zeros(25), cov, J=8, N=256, seed=1)
    th = torch.tensor(sps_synth.particles(1000, 25), device="cuda")
    th[737, 4] = float("nan")
    out = torch.empty(1000, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    s.loglik(th.data_ptr(), 1000, 25, 17, 300, out.data_ptr())
    with pytest.raises(sps.SpsError) as e:
        s.sync()
    assert e.value.status == 4 and "p = 737" in str(e.value) and "t = 17" in str(e.value)
    # overflow: theta_1 = 1e308 overflows eta_t = s_t x_t1 theta_1 (s_t = 1 - 2 y_t, R17) at the first t
    # with s_t x_t1 > DBL_MAX / 1e308, where softplus(+inf) = inf
    th = torch.tensor(sps_synth.particles(64, 25), device="cuda")
    th[5, 1] = 1e308
    s.loglik(th.data_ptr(), 64, 25, 0, 300, out.data_ptr())
    sgn = 1.0 - 2.0 * y
    with np.errstate(over="ignore"):
        eta = sgn * X[:, 1] * 1e308
    t_bad = int(np.flatnonzero(eta == np.inf)[0])
    with pytest.raises(sps.SpsError) as e:
        s.sync()
    assert e.value.status == 4 and "p = 5" in str(e.value) and f"t = {t_bad}" in str(e.value)
    th[5, 1] = 0.1
    s.loglik(th.data_ptr(), 64, 25, 0, 300, out.data_ptr())
    s.sync()  # cleared: finite again
    assert torch.isfinite(out[:64]).all()
    s.close()


def test_logml_many_cycles_small_increment_buffer(sps, orc, monkeypatch):
    """more cycles than the device increment buffer holds (SPS_INC_CAP = 3 here,
    1024 by default) -- every increment is pulled before its slot is reused."""
    monkeypatch.setenv("SPS_INC_CAP", "3")
    X, y = sps_synth.config_data("cfg1")
    cov = orc.g_prior(X, 2, 0.25)
    o = orc.run(X, y, 2, 4, 128, seed=2, prior_mean=np.zeros(4), prior_cov=cov)
    s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=2)
    g = s.run()
    s.close()
    assert o["L"] > 3
    _compare(g, o)


def test_reset_rerun_bit_identical_cfg2(sps):
    """Back-to-back runs on one context (the bench's timed loop): sps_reset(seed) restores every piece of
    device state a run reads, so the same seed reproduces the run bit for bit after another seed's run
    (no state carried from the previous run's last M step, cycle or increment buffer)."""
    X, y = sps_synth.config_data("cfg2")
    cov = sps.g_prior(X, 2, 1.0 / 16)
    s = sps.Sps(X, y, np.zeros(25), cov, J=64, N=1024, seed=1)
    res = []
    for seed in (5, 6, 5, 5):
        s.reset(seed)
        r = s.run()
        res.append((r["logml"], r["L"], r["total_m_steps"], r["mean"].tobytes()))
    s.close()
    assert res[0] == res[2] == res[3]
    assert res[1] != res[0]


def test_concurrent_independent_contexts(sps):
    """Two independent contexts driven from two host threads at once on one GPU (own streams, shared
    process-wide state: kernel attributes, the pinned control-slab pool) give the same results, bit for
    bit, as the same runs one after the other."""
    import threading

    X, y = sps_synth.config_data("cfg2", n=300)
    cov = sps.g_prior(X, 2, 1.0 / 16)

    def one(seed):
        s = sps.Sps(X, y, np.zeros(25), cov, J=8, N=256, seed=seed)
        r = s.run()
        s.close()
        return r["logml"], r["L"], r["total_m_steps"], r["mean"].tobytes()

    seq = [one(11), one(12)]
    par = [None, None]
    errs = []

    def worker(q, seed):
        try:
            par[q] = one(seed)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(q, 11 + q)) for q in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    assert par == seq
