import numpy as np, sys, os, time, json
sys.path.insert(0, '/root/repo')
import paper_1304_4333_b200 as sps, sps_synth
import torch
k = int(sys.argv[1])
X, y = sps_synth.make_data(1000, k, 2, max(1, (3 * k) // 10), (-0.85,), 0.3)
cov = sps.g_prior(X, 2, 1.0 / 16)
s = sps.Sps(X, y, np.zeros(k), cov, J=64, N=1024, seed=1)
s.run()
ts = []
for seed in (2, 3):
    s.reset(seed)
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = s.run(); ts.append(time.perf_counter() - t0)
print(json.dumps({"k": k, "oz": os.environ.get("SPS_OZ_MINK"), "noz": os.environ.get("SPS_NO_OZAKI"), "s": min(ts), "L": r["L"], "steps": r["total_m_steps"], "logml": r["logml"]}))
s.close()
