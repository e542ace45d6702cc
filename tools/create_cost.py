"""Host cost of sps_create / run / close on the cfg2 workload (e2e path of bench.py)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

X, y = sps_synth.config_data("cfg2")
cov = sps.g_prior(X, 2, 1.0 / 16)
torch.cuda.init()
for r in range(4):
    t0 = time.perf_counter()
    c = sps.Sps(X, y, np.zeros(25), cov, J=64, N=1024, seed=1 + r)
    c.sync()
    t1 = time.perf_counter()
    rep = c.run()
    t2 = time.perf_counter()
    c.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.1f} ms  run {1e3*(t2-t1):7.1f} ms  close {1e3*(t3-t2):7.1f} ms")
