"""Small end-to-end workloads touching every kernel family of the hot path, sized to finish
quickly under instrumentation (compute-sanitizer memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

compute-sanitizer is closed on the GPU pool this repo was measured on (a call is refused with
exit 86), so this has only run plain; it is kept for boxes where the sanitizer is available.

Covers: K1 binary DMMA (k = 25, ragged P and range), binary DFMA (k = 42), multinomial (C = 4);
full Algorithm 2 runs with data and power tempering and the three resampling schemes, a
multinomial run, and Algorithm 3 two-pass.  The sharded engine (loopback transport, one host
thread per rank) is not exercised here.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1304_4333_b200 as sps  # noqa: E402
import sps_synth  # noqa: E402


def loglik_cases():
    rng = np.random.default_rng(5)
    for C, k in [(2, 25), (2, 42), (4, 10)]:
        n = 333
        X = np.column_stack([np.ones(n), rng.normal(size=(n, k - 1))])
        y = rng.integers(0, C, n).astype(np.int32)
        d = k * (C - 1)
        s = sps.Sps(X, y, np.zeros(d), np.eye(d), J=2, N=512, seed=1, C_=C)
        th = torch.tensor(rng.normal(0, 0.3, (1037, d)), device="cuda")
        out = s.loglik_tensor(th, 0, n)
        s.loglik_tensor(th, 17, 18)
        s.sync()
        assert torch.isfinite(out).all()
        s.close()
        print("loglik", C, k, "ok", flush=True)


def runs():
    X, y = sps_synth.config_data("cfg1")
    cov = sps.g_prior(X, 2, 0.25)
    for tempering in (0, 1):
        for resampling in (0, 1, 2):
            s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=2, tempering=tempering, resampling=resampling)
            g = s.run()
            s.close()
            print("run tempering", tempering, "resampling", resampling, "logml", g["logml"], flush=True)
    Xm, ym = sps_synth.make_data(120, 3, 3, 2, (0.2, -0.3), 0.4, seed=11)
    covm = sps.g_prior(Xm, 3, 0.5)
    s = sps.Sps(Xm, ym, np.zeros(6), covm, J=4, N=256, seed=4, C_=3)
    g = s.run()
    s.close()
    print("run multinomial logml", g["logml"], flush=True)
    s = sps.Sps(X, y, np.zeros(4), cov, J=4, N=128, seed=1)
    r = s.two_pass(5, 6)
    s.close()
    print("two-pass ok", flush=True)


if __name__ == "__main__":
    loglik_cases()
    runs()
