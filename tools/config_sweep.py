"""Every BASELINE.json config on one B200 (the bench line is configs[1] only): full-data K1
pairs/s and, where a full run fits in seconds, the whole Algorithm 2 run (wall, pairs/s, log ML);
plus the oracle on a bounded host sample of the same shape (pairs/s, threads used).

    python tools/config_sweep.py [--no-oracle] > profiles/r01_config_sweep.json

configs[0] cfg1 (n=100, k=4, 4x128), configs[1] cfg2 (n=1000, k=25, 64x1024), configs[2] cfg3
(multinomial C=4, k=10, n=5000, 128x1024), configs[3] cfg4 (n=1e5, k=100: one GPU's shard of
1024x1024 = 128x1024 particles; full-data K1 and one C-phase-free M-step-size evaluation only), configs[4]
cfg5 (cfg2 data, 2^14 .. 2^22 particles: full runs up to 2^20, K1 at every size).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

FP64_PEAK = 37.07  # TF/s, measured (profiles/r01_fp64_peaks.json)


def k1_rate(ctx, P, d, n, reps=10):
    th = torch.randn(P, d, dtype=torch.float64, device="cuda") * (0.3 if d <= 30 else 0.05)
    out = torch.empty(P, dtype=torch.float64, device="cuda")
    for _ in range(2):
        ctx.loglik(th.data_ptr(), P, d, 0, n, out.data_ptr())
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        ctx.loglik(th.data_ptr(), P, d, 0, n, out.data_ptr())
    ctx.sync()
    ms = (time.perf_counter() - t0) / reps * 1e3
    return ms, P * n / (ms * 1e-3)


def full_run(ctx, seeds=(2, 3)):
    ctx.run()  # warm-up (graphs, plans)
    best = None
    for s in seeds:
        ctx.reset(s)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = ctx.run()
        dt = time.perf_counter() - t0
        if best is None or dt < best[0]:
            best = (dt, rep)
    dt, rep = best
    return {"wall_s": dt, "pairs_per_s": rep["pairs"] / dt, "cycles": rep["L"], "m_steps": rep["total_m_steps"],
            "logml": rep["logml"], "logml_nse": rep["logml_nse"]}


def oracle_sample(X, y, C, J, N, g):
    import oracle

    d = X.shape[1] * (C - 1)
    cov = oracle.g_prior(X, C, g)
    t0 = time.perf_counter()
    r = oracle.run(X, y, C, J, N, seed=1, prior_mean=np.zeros(d), prior_cov=cov, n_threads=os.cpu_count())
    dt = time.perf_counter() - t0
    return {"pairs_per_s": r["pairs"] / dt, "seconds": dt, "threads": os.cpu_count(), "sample": f"J={J} x N={N} full run"}


def oracle_loglik(X, y, C, P, d):
    import oracle

    th = sps_synth.particles(P, d, scale=0.05 if d > 30 else 0.3, seed=11)
    t0 = time.perf_counter()
    oracle.loglik_range(th, X, y, C)
    dt = time.perf_counter() - t0
    return {"pairs_per_s": P * X.shape[0] / dt, "seconds": dt, "sample": f"{P} particles x full n, one evaluation"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--only", default=None, help="one of cfg1..cfg4, cfg5 (skip the rest)")
    a = ap.parse_args()
    out = {"gpu": torch.cuda.get_device_name(0), "host_threads": os.cpu_count(), "configs": {}}
    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        if a.only and a.only != name:
            continue
        c = sps_synth.CONFIGS[name]
        X, y = sps_synth.config_data(name)
        n, k = X.shape
        C = c["C"]
        d = k * (C - 1)
        J, N = c["J"], c["N"]
        if name == "cfg4":
            J = J // 8  # one GPU's shard of the 8-GPU configuration
        cov = sps.g_prior(X, C, c["g"])
        ctx = sps.Sps(X, y, np.zeros(d), cov, J=J, N=N, seed=1, C_=C)
        P = J * N
        ms, rate = k1_rate(ctx, P, d, n, reps=3 if name == "cfg4" else 10)
        ent = {"n": n, "k": k, "C": C, "J": J, "N": N, "particles": P,
               "k1_full_data": {"ms": ms, "pairs_per_s": rate,
                                "frac_fp64_peak": rate * (2 * d + (11 if C == 2 else 0)) / 1e12 / FP64_PEAK}}
        if name != "cfg4":
            ent["run"] = full_run(ctx)
        ctx.close()
        if not a.no_oracle:
            if name in ("cfg1", "cfg2"):
                ent["oracle"] = oracle_sample(X, y, C, J if name == "cfg1" else 16, N if name == "cfg1" else 256, c["g"])
            else:
                ent["oracle"] = oracle_loglik(X, y, C, 256 if name == "cfg4" else 2048, d)
        out["configs"][name] = ent
        print(name, json.dumps(ent), file=sys.stderr, flush=True)
    # configs[4]: particle sweep at the cfg2 shape
    if a.only and a.only != "cfg5":
        print(json.dumps(out, indent=1))
        return
    X, y = sps_synth.config_data("cfg2")
    cov = sps.g_prior(X, 2, 1.0 / 16)
    sweep = {}
    for logP in range(14, 23, 2):
        P = 1 << logP
        N = 1024
        J = P // N
        ctx = sps.Sps(X, y, np.zeros(25), cov, J=J, N=N, seed=1)
        ms, rate = k1_rate(ctx, P, 25, 1000, reps=5)
        ent = {"particles": P, "k1_full_data": {"ms": ms, "pairs_per_s": rate,
                                                "frac_fp64_peak": rate * 61 / 1e12 / FP64_PEAK}}
        if logP <= 20:
            ent["run"] = full_run(ctx, seeds=(2,))
        ctx.close()
        sweep[f"2^{logP}"] = ent
        print("cfg5", logP, json.dumps(ent), file=sys.stderr, flush=True)
    out["configs"]["cfg5_sweep"] = sweep
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
