"""K1 on one GPU's configs[3] shard (n = 1e5, k = 100, P = 128 x 1024): full-data evaluations
timed with CUDA events, the INT8 tensor-core kernel (ozaki.cuh, default for binary k >= 64) or the
FP64 DMMA kernel (SPS_NO_OZAKI=1).  pairs/s, the FP64-equivalent fraction (2k + 11 ops per pair
against the measured 37.07 TF DMMA peak) and, for the INT8 path, the int8 MMA work
(KB x 32 x 28 MACs per pair) against the nominal 4.5 POPS dense int8 rate.

    [SPS_NO_OZAKI=1] python tools/k1_oz_ab.py [--n N] [--P P]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100000)
ap.add_argument("--P", type=int, default=131072)
ap.add_argument("--k", type=int, default=100, help="covariates (configs[3] recipe with k columns)")
a = ap.parse_args()
if a.k == 100:
    X, y = sps_synth.config_data("cfg4", n=a.n)
else:  # the configs[3] recipe at another k: ~30% continuous columns, the rest 0/1
    X, y = sps_synth.make_data(a.n, a.k, 2, max(1, (3 * a.k) // 10), (0.0,), 0.15)
n, k = X.shape
ctx = sps.Sps(X, y, np.zeros(k), np.eye(k), J=2, N=4, seed=1)
th = torch.tensor(sps_synth.particles(a.P, k, scale=0.05, seed=4), device="cuda")
out = torch.empty(a.P, dtype=torch.float64, device="cuda")
for _ in range(2):
    ctx.loglik(th.data_ptr(), a.P, k, 0, n, out.data_ptr())
ctx.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    ctx.loglik(th.data_ptr(), a.P, k, 0, n, out.data_ptr())
ctx.sync()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
pairs = a.P * n / (ms * 1e-3)
oz = os.environ.get("SPS_NO_OZAKI") is None and k >= int(os.environ.get("SPS_OZ_MINK", "64"))
KB = (k + 31) // 32
print(json.dumps({"kernel": "int8 tcgen05 (ozaki)" if oz else "fp64 DMMA", "n": n, "k": k, "P": a.P, "ms": ms,
                  "pairs_per_s": pairs, "fp64_equiv_frac": pairs * (2 * k + 11) / 1e12 / 37.07,
                  "int8_mma_frac": (pairs * KB * 32 * 28 * 2 / 4.5e15) if oz else None,
                  "checksum": float(out.sum().item())}))
ctx.close()
