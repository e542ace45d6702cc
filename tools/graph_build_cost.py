"""Host graph-build cost per fresh and reused context (cfg2): instantiation of the device-side M-phase
loop graph on a new context vs executable-graph updates per M phase on a reused one.

    python tools/graph_build_cost.py
"""
import os, sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import paper_1304_4333_b200 as sps, sps_synth
X, y = sps_synth.config_data("cfg2")
cov = sps.g_prior(X, 2, 1.0 / 16)
for r in range(3):
    t0 = time.perf_counter()
    c = sps.Sps(X, y, np.zeros(25), cov, J=64, N=1024, seed=1 + r)
    rep = c.run()
    cn = c.counters()
    t1 = time.perf_counter()
    c.reset(5); rep2 = c.run(); cn2 = c.counters()
    t2 = time.perf_counter()
    c.close()
    print(f"fresh ctx: create+run {1e3*(t1-t0):.1f} ms graph build {cn['cat_ms']['host_graph_build']:.2f} ms n {cn['cat_n']['host_graph_build']}; reused: run {1e3*(t2-t1):.1f} ms graph build {cn2['cat_ms']['host_graph_build']:.2f} ms n {cn2['cat_n']['host_graph_build']}")
