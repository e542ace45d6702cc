"""Host cost of the per-phase M-step graph capture (cfg2), graphs vs streams."""
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
ctx.run()
best = 1e9
for r in range(3):
    ctx.reset(seed=2 + r)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = ctx.run()
    best = min(best, time.perf_counter() - t0)
cnt = ctx.counters()
print(f"graph={'off' if os.environ.get('SPS_NO_GRAPH') else 'on'} run {best*1e3:.1f} ms  cats:",
      {k: (round(v, 2), cnt["cat_n"][k]) for k, v in cnt["cat_ms"].items() if k.startswith("host")})
ctx.close()
