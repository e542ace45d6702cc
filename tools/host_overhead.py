"""Host-side costs of one cfg2 run (no profiling): M-step graph capture + update, launch and wait
times per run, and the run's wall time, to bound the GPU idle time the host causes.

    python tools/host_overhead.py [J]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

J = int(sys.argv[1]) if len(sys.argv) > 1 else 64
X, y = sps_synth.config_data("cfg2")
ctx = sps.Sps(X, y, np.zeros(25), sps.g_prior(X, 2, 1.0 / 16), J=J, N=1024, seed=1)
ctx.run()
for seed in (2, 3, 4):
    ctx.reset(seed)
    t0 = time.perf_counter()
    rep = ctx.run()
    wall = time.perf_counter() - t0
    c = ctx.counters()
    cm = c["cat_ms"]
    print(f"seed {seed}: wall {wall * 1e3:.2f} ms, cycles {rep['L']}, M steps {rep['total_m_steps']}, "
          f"host graph build {cm['host_graph_build']:.2f} ms (updates+1000*inst {c['cat_n']['host_graph_build']}), "
          f"host M-phase launch {cm['host_mstep_launch']:.2f} ms, host M-phase wait {cm['host_mstep_wait']:.2f} ms, "
          f"syncs {c['syncs']}, launches {c['launches']}")
ctx.close()
