import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1304_4333_b200 as sps, sps_synth
X, y = sps_synth.config_data("cfg2")
ctx = sps.Sps(X, y, np.zeros(25), sps.g_prior(X, 2, 1.0/16), J=64, N=1024, seed=1)
rep = ctx.run()
t = rep["t_cycle"]; R = rep["R_cycle"]
print("cycles", len(t), "msteps", R.sum())
for lo, hi in [(0,32),(32,64),(64,128),(128,256),(256,512),(512,1001)]:
    m = (t > lo) & (t <= hi)
    print(f"t in ({lo},{hi}]: cycles {m.sum():3d} msteps {R[m].sum():5d} pairs-frac {(R[m]*t[m]).sum()/(R*t).sum():.3f}  modelK1 {(R[m]*(11+0.18*t[m])).sum()/1e3:.1f} ms")
print("t sched", list(t[:20]), "...", list(t[-5:]))
print("R sched", list(R[:20]), "...", list(R[-5:]))
