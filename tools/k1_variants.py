"""K1 variant A/B on the cfg2 workload (SPS_K1_VAR selects; one variant per process).

    SPS_K1_VAR=w2 python tools/k1_variants.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

X, y = sps_synth.config_data("cfg2")
ctx = sps.Sps(X, y, np.zeros(25), sps.g_prior(X, 2, 1.0 / 16), J=64, N=1024, seed=1)
th = torch.randn(65536, 25, dtype=torch.float64, device="cuda") * 0.3
for _ in range(3):
    ctx.loglik_tensor(th)
torch.cuda.synchronize()
t0 = time.perf_counter()
R = 20
for _ in range(R):
    ctx.loglik_tensor(th)
torch.cuda.synchronize()
ll_ms = (time.perf_counter() - t0) / R * 1e3
ctx.run()
ts = []
for r in range(3):
    ctx.reset(seed=2 + r)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = ctx.run()
    ts.append(time.perf_counter() - t0)
print(f"VAR={os.environ.get('SPS_K1_VAR', 'default'):8s} loglik_full {ll_ms:.3f} ms  run {min(ts)*1e3:.1f} ms "
      f"(msteps {rep['total_m_steps']}) logml {rep['logml']:.10f}")
ctx.close()
