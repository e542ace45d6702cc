"""One full-data K1 evaluation at a BASELINE config (for ncu captures of the likelihood kernel).

    python tools/k1_once.py cfg3 [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = sps_synth.CONFIGS[name]
X, y = sps_synth.config_data(name)
n, k = X.shape
C = c["C"]
d = k * (C - 1)
J = c["J"] // (8 if name == "cfg4" else 1)
ctx = sps.Sps(X, y, np.zeros(d), sps.g_prior(X, C, c["g"]), J=J, N=c["N"], seed=1, C_=C)
P = J * c["N"]
th = torch.randn(P, d, dtype=torch.float64, device="cuda") * (0.3 if d <= 30 else 0.05)
out = torch.empty(P, dtype=torch.float64, device="cuda")
for _ in range(reps):
    ctx.loglik(th.data_ptr(), P, d, 0, n, out.data_ptr())
ctx.sync()
print(name, P, n, float(out.sum()))
ctx.close()
