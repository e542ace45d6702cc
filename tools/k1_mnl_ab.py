"""A/B of the multinomial K1 kernels on the configs[2] shape (C = 4, k = 10, n = 5000,
P = 128 x 1024): full-data evaluations timed with CUDA events; pairs/s and the fraction of the
measured FP64 peak counting the contraction alone (2 k (C-1) flops per pair) and with the epilogue.

    [SPS_MNL_DFMA=1] python tools/k1_mnl_ab.py   (the round-2 variants "pad" / "rem" were removed after this A/B)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

PEAK = 37.07
X, y = sps_synth.config_data("cfg3")
n, k = X.shape
C, P, d = 4, 128 * 1024, 30
ctx = sps.Sps(X, y, np.zeros(d), sps.g_prior(X, C, 1.0), J=4, N=128, seed=1, C_=C)
th = torch.tensor(sps_synth.particles(P, d, scale=0.3, seed=3), device="cuda")
out = torch.empty(P, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    ctx.loglik(th.data_ptr(), P, d, 0, n, out.data_ptr())
ctx.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    ctx.loglik(th.data_ptr(), P, d, 0, n, out.data_ptr())
ctx.sync()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
pairs = P * n / (ms * 1e-3)
print(json.dumps({"variant": os.environ.get("SPS_MNL_VAR", "dfma" if os.environ.get("SPS_MNL_DFMA") else "default"),
                  "ms": ms, "pairs_per_s": pairs, "frac_contraction": pairs * 2 * k * (C - 1) / 1e12 / PEAK,
                  "frac_61ops": pairs * 61 / 1e12 / PEAK}))
ctx.close()
