"""Cost of the sharded engine's exchange path on one GPU (debug / projection).

Times whole Algorithm 2 runs on the cfg2 data at J x N = (J, 1024) three ways:
  default   one rank: device-side M-step loop (CUDA graph WHILE node), fused reduce + finalize
  no_loop   one rank: per-step graph replays from the host (SPS_NO_LOOP=1)
  no_graph  one rank: plain launches from the host, fused reduce + finalize (SPS_NO_GRAPH=1)
  xchg      one rank through the multi-GPU code path (SPS_XCHG_1RANK=1, a real 1-rank NCCL
            communicator): ncclAllGather of every statistics slice, finalize as its own launch,
            host-driven M steps -- what each rank runs at G > 1, minus the wire time
Run each in its own process (the env var is read at sps_create).

    python tools/xchg_cost.py [J] [runs]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1304_4333_b200 as sps, sps_synth
J, runs = {J}, {runs}
X, y = sps_synth.config_data("cfg2")
cov = sps.g_prior(X, 2, 1.0 / 16)
nid = sps.nccl_unique_id() if {xchg} else None
s = sps.Sps(X, y, np.zeros(25), cov, J=J, N=1024, seed=1, nccl_id=nid)
s.run()  # warm-up (graph capture, plans)
ts, steps = [], []
for r in range(runs):
    s.reset(10 + r)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = s.run()
    ts.append(time.perf_counter() - t0)
    steps.append(int(rep["total_m_steps"]))
s.close()
print("RESULT" + json.dumps(dict(s_per_run=ts, m_steps=steps)))
"""


def main():
    J = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    runs = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    out = {}
    variants = (("default", 0, {}), ("no_loop", 0, {"SPS_NO_LOOP": "1"}), ("no_graph", 0, {"SPS_NO_GRAPH": "1"}),
                ("xchg", 1, {"SPS_XCHG_1RANK": "1"}))
    for tag, xchg, extra in variants:
        env = dict(os.environ)
        env.update(extra)
        p = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT, J=J, runs=runs, xchg=xchg)], env=env,
                           capture_output=True, text=True, timeout=1800)
        if p.returncode:
            print(p.stderr[-3000:])
            raise SystemExit(1)
        out[tag] = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("RESULT")][-1][6:])
    for tag, r in out.items():
        ms = [1e3 * t for t in r["s_per_run"]]
        us_step = [1e3 * m / s for m, s in zip(ms, r["m_steps"])]
        print(f"{tag:8s} J={J} x 1024: run ms {min(ms):8.2f} (median {sorted(ms)[len(ms) // 2]:8.2f}), "
              f"M steps {r['m_steps']}, us per M step (whole run / steps) {min(us_step):7.2f}")
    print("JSON" + json.dumps(dict(J=J, N=1024, **out)))


if __name__ == "__main__":
    main()
