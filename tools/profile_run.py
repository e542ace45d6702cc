"""One cfg2 SPS run (after one warm-up run) for ncu launch lists / captures.

    python tools/profile_run.py [--runs R] [--loglik-only]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--loglik-only", action="store_true")
ap.add_argument("--nt", type=int, default=0, help="--loglik-only: observation range [0, nt) (0: all)")
ap.add_argument("--J", type=int, default=64, help="groups of 1024 (1024: P = 2^20)")
ap.add_argument("--power", action="store_true", help="power tempering (north_star bisection C phase)")
a = ap.parse_args()
X, y = sps_synth.config_data("cfg2")
cov = sps.g_prior(X, 2, 1.0 / 16)
ctx = sps.Sps(X, y, np.zeros(25), cov, J=a.J, N=1024, seed=1, tempering=1 if a.power else 0)
if a.loglik_only:
    import torch

    th = torch.randn(a.J * 1024, 25, dtype=torch.float64, device="cuda") * 0.3
    for _ in range(5):
        ctx.loglik_tensor(th, 0, a.nt or None)
else:
    ctx.run()  # warm-up
    for r in range(a.runs):
        ctx.reset(seed=2 + r)
        rep = ctx.run()
        print("run", r, "cycles", rep["L"], "msteps", rep["total_m_steps"], "logml", rep["logml"])
ctx.close()
