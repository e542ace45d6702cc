"""Phase clocks of the fused reduce + finalize on the cfg2 workload (debug).

    SPS_TRACE=1 python tools/trace_run.py [J]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402

J = int(sys.argv[1]) if len(sys.argv) > 1 else 64  # groups of 1024 (1024: P = 2^20)
X, y = sps_synth.config_data("cfg2")
ctx = sps.Sps(X, y, np.zeros(25), sps.g_prior(X, 2, 1.0 / 16), J=J, N=1024, seed=1)
rep = ctx.run()
print("cycles", rep["L"], "msteps", rep["total_m_steps"], "logml", rep["logml"])
ctx.counters()
ctx.close()
