"""K1 throughput vs observation range n_t (cfg2 data, P = 65536, d = 25): event-timed K1 launches
through sps_loglik (profiling counters), pairs/s and fraction of the FP64-pipe pair rate.
Env: SPS_K1_SK=0 (chunk planner instead of stream-K), SPS_K1_TAB (exp table)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

X, y = sps_synth.config_data("cfg2")
ctx = sps.Sps(X, y, np.zeros(25), sps.g_prior(X, 2, 1.0 / 16), J=64, N=1024, seed=1)
P = 65536
th = torch.randn(P, 25, dtype=torch.float64, device="cuda") * 0.3
out = torch.empty(P, dtype=torch.float64, device="cuda")
PEAK_PAIRS = 37.07e12 / 2 / 36.0  # FP64 FMA-slot rate / slots per pair (25 contraction + 11 epilogue)
ctx.set_profiling(True)
for nt in [8, 16, 32, 64, 128, 200, 256, 384, 512, 768, 1000]:
    for _ in range(3):
        ctx.loglik(th.data_ptr(), P, 25, 0, nt, out.data_ptr())
    ctx.sync()
    c0 = ctx.counters()
    R = 30
    for _ in range(R):
        ctx.loglik(th.data_ptr(), P, 25, 0, nt, out.data_ptr())
    ctx.sync()
    c1 = ctx.counters()
    ms = (c1["cat_ms"]["k1"] - c0["cat_ms"]["k1"]) / R
    rate = P * nt / (ms * 1e-3)
    print(f"n_t {nt:5d}: K1 {ms*1e3:7.2f} us  {rate:.3e} pairs/s  frac {rate / PEAK_PAIRS:.3f}", flush=True)
ctx.close()
