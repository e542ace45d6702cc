"""Host-side costs of one cfg2 run (no profiling events): M-phase graph capture/update, launch and
wait time, syncs; plus the wall time between M phases (C phase + S phase + graph build)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

X, y = sps_synth.config_data("cfg2")
ctx = sps.Sps(X, y, np.zeros(25), sps.g_prior(X, 2, 1.0 / 16), J=64, N=1024, seed=1)
ctx.run()
ctx.reset(2)
t_c = t_m = 0.0
nc = 0
while True:
    t0 = time.perf_counter()
    try:
        t, phi, _ = ctx.cphase()
    except sps.SpsError:
        break
    ctx.sync()
    t1 = time.perf_counter()
    R, rne, h = ctx.mphase()
    t2 = time.perf_counter()
    t_c += t1 - t0
    t_m += t2 - t1
    nc += 1
    if t == ctx.n:
        break
c = ctx.counters()
print(f"cycles {nc}: C+S phases {t_c*1e3:.2f} ms ({t_c/nc*1e6:.1f} us/cycle), M phases {t_m*1e3:.2f} ms")
print("host graph build ms", round(c["cat_ms"]["host_graph_build"], 3), "launch ms", round(c["cat_ms"]["host_mstep_launch"], 3),
      "wait ms", round(c["cat_ms"]["host_mstep_wait"], 3), "syncs", c["syncs"], "graph updates/instantiations",
      c["cat_n"]["host_graph_build"])
ctx.close()
