"""CPU oracle for the SPS logit hot path -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper around ``oracle/liboracle.so`` (built from ``oracle.c``
by :func:`build`).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product library (``paper_1304_4333_b200``) never imports it and
shares no code with it.  See ``oracle/oracle.h`` for the paper citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

TAG_INIT, TAG_PROPOSAL, TAG_ACCEPT, TAG_RESAMPLE = 1, 2, 3, 4
RESIDUAL, SYSTEMATIC, MULTINOMIAL = 0, 1, 2
DATA, POWER = 0, 1
OK, E_CONFIG, E_DATA, E_NUMERIC, E_MIXING = 0, 2, 3, 4, 5


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        cmd = [
            "gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
            "-fPIC", "-shared", "-Wall", "-Wno-unused-function", "-o", _SO, _SRC, "-lm",
        ]
        subprocess.run(cmd, check=True, cwd=_HERE)
    return _SO


class Config(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("k", C.c_int32), ("C", C.c_int32), ("J", C.c_int32), ("N", C.c_int32),
        ("seed", C.c_uint64), ("tempering", C.c_int32), ("resampling", C.c_int32),
        ("ess_frac", C.c_double), ("K_inter", C.c_double), ("K_final", C.c_double),
        ("h_init", C.c_int32), ("h_step", C.c_int32), ("h_min", C.c_int32), ("h_max", C.c_int32),
        ("accept_target", C.c_double), ("max_m_steps", C.c_int32), ("max_cycles", C.c_int32),
        ("n_monitors", C.c_int32), ("n_report", C.c_int32), ("pass_", C.c_int32),
        ("n_threads", C.c_int32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("L", C.c_int32), ("total_m_steps", C.c_int32), ("h_final", C.c_int32),
        ("logml", C.c_double), ("logml_nse", C.c_double), ("pairs", C.c_double),
        ("t_cycle", C.POINTER(C.c_int32)), ("phi_cycle", C.POINTER(C.c_double)),
        ("R_cycle", C.POINTER(C.c_int32)), ("logml_inc", C.POINTER(C.c_double)),
        ("min_rne", C.POINTER(C.c_double)), ("h_cycle", C.POINTER(C.c_int32)),
        ("mean", C.POINTER(C.c_double)), ("sd", C.POINTER(C.c_double)),
        ("nse", C.POINTER(C.c_double)), ("rne", C.POINTER(C.c_double)),
        ("logpl", C.POINTER(C.c_double)),
        ("trace_cap", C.c_int32), ("step_nacc", C.POINTER(C.c_int32)), ("step_h", C.POINTER(C.c_int32)),
        ("step_minrne", C.POINTER(C.c_double)), ("snap_cap", C.c_int32), ("theta_snap", C.POINTER(C.c_double)),
        ("inc_group", C.POINTER(C.c_double)), ("Lj", C.POINTER(C.c_double)),
    ]


_lib = None


class Schedule(C.Structure):
    """or_schedule: the fixed design of Algorithm 3 pass 2."""
    _fields_ = [("L", C.c_int32), ("t_cycle", C.POINTER(C.c_int32)), ("phi_cycle", C.POINTER(C.c_double)),
                ("R_cycle", C.POINTER(C.c_int32)), ("sigma", C.POINTER(C.c_double))]


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        dp, ip, up = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.POINTER(C.c_uint64)
        L.or_philox4x32_10.argtypes = [C.POINTER(C.c_uint32)] * 3
        L.or_u01.argtypes = [C.c_uint32, C.c_uint32]
        L.or_u01.restype = C.c_double
        for f in ("or_plog", "or_pexp"):
            getattr(L, f).argtypes = [C.c_double]
            getattr(L, f).restype = C.c_double
        L.or_psincos2pi.argtypes = [C.c_double, dp, dp]
        L.or_normals.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int32, dp]
        L.or_accept_uniform.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.or_accept_uniform.restype = C.c_double
        L.or_resample_a52.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]
        L.or_resample_a52.restype = C.c_uint64
        L.or_logp.argtypes = [dp, dp, C.c_int32, C.c_int32, C.c_int32]
        L.or_logp.restype = C.c_double
        L.or_loglik_range.argtypes = [dp, C.c_int64, C.c_int32, dp, ip, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_int32, dp]
        L.or_loglik_range.restype = C.c_int32
        L.or_cholesky.argtypes = [C.c_int32, dp, dp]
        L.or_cholesky.restype = C.c_int32
        L.or_prior_quad.argtypes = [C.c_int32, dp, dp, dp]
        L.or_prior_quad.restype = C.c_double
        L.or_g_prior.argtypes = [dp, C.c_int32, C.c_int32, C.c_int32, C.c_double, dp]
        L.or_g_prior.restype = C.c_int32
        L.or_ess.argtypes = [dp, C.c_int64]
        L.or_ess.restype = C.c_double
        L.or_resample_int.argtypes = [C.c_int32, up, C.c_int32, up, ip]
        L.or_resample_int.restype = C.c_int32
        L.or_resample_group.argtypes = [C.c_int32, dp, C.c_int32, C.c_uint64, C.c_uint32, C.c_uint32,
                                        C.c_uint32, ip]
        L.or_resample_group.restype = C.c_int32
        L.or_group_stats.argtypes = [dp, C.c_int32, C.c_int32, dp, dp, dp, dp]
        L.or_power_search.argtypes = [dp, C.c_int64, C.c_double, C.c_double, dp]
        L.or_power_search.restype = C.c_int32
        L.or_run.argtypes = [C.POINTER(Config), dp, ip, dp, dp, dp, dp, C.POINTER(Report), dp]
        L.or_run.restype = C.c_int32
        L.or_run2.argtypes = [C.POINTER(Config), dp, ip, dp, dp, dp, dp, C.POINTER(Schedule), dp, C.c_int64,
                              C.POINTER(Report), dp]
        L.or_run2.restype = C.c_int32
        _lib = L
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


def _u(a):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    return a, a.ctypes.data_as(C.POINTER(C.c_uint64))


# ---------------------------------------------------------------- random streams
def philox(ctr, key):
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return [int(v) for v in o]


def u01(hi, lo):
    return lib().or_u01(hi, lo)


def plog(x):
    return lib().or_plog(float(x))


def pexp(x):
    return lib().or_pexp(float(x))


def psincos2pi(u):
    s, c = C.c_double(), C.c_double()
    lib().or_psincos2pi(float(u), C.byref(s), C.byref(c))
    return s.value, c.value


def normals(seed, ident, step, tag, count, pass_=0):
    z = np.zeros(count)
    lib().or_normals(seed, ident, step, tag, pass_, count, z.ctypes.data_as(C.POINTER(C.c_double)))
    return z


def accept_uniform(seed, p, step, pass_=0):
    return lib().or_accept_uniform(seed, p, step, pass_)


def resample_a52(seed, group, cycle, r, pass_=0):
    return int(lib().or_resample_a52(seed, group, cycle, pass_, r))


# ---------------------------------------------------------------- model
def logp(theta, x, y, C_):
    th, thp = _d(theta)
    xx, xp = _d(x)
    return lib().or_logp(thp, xp, int(y), xx.shape[0], int(C_))


def loglik_range(theta, X, y, C_, t0=0, t1=None, n_threads=0):
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    X, Xp = _d(X)
    y, yp = _i(y)
    n, k = X.shape
    t1 = n if t1 is None else t1
    P, ld = theta.shape
    out = np.zeros(P)
    st = lib().or_loglik_range(theta.ctypes.data_as(C.POINTER(C.c_double)), P, ld, Xp, yp, n, k, int(C_),
                               int(t0), int(t1), int(n_threads), out.ctypes.data_as(C.POINTER(C.c_double)))
    if st:
        raise RuntimeError(f"or_loglik_range status {st}")
    return out


def cholesky(A):
    A, Ap = _d(A)
    L = np.zeros_like(A)
    st = lib().or_cholesky(A.shape[0], Ap, L.ctypes.data_as(C.POINTER(C.c_double)))
    if st:
        raise np.linalg.LinAlgError("or_cholesky: not positive definite")
    return L


def prior_quad(Lprior, mu, theta):
    Lp, Lpp = _d(Lprior)
    m, mp = _d(mu)
    t, tp = _d(theta)
    return lib().or_prior_quad(Lp.shape[0], Lpp, mp, tp)


def g_prior(X, C_, g):
    X, Xp = _d(X)
    n, k = X.shape
    d = k * (C_ - 1)
    cov = np.zeros((d, d))
    st = lib().or_g_prior(Xp, n, k, int(C_), float(g), cov.ctypes.data_as(C.POINTER(C.c_double)))
    if st:
        raise np.linalg.LinAlgError("X'X not positive definite")
    return cov


# ---------------------------------------------------------------- SPS pieces
def ess(lw):
    lw, p = _d(lw)
    return lib().or_ess(p, lw.shape[0])


def resample_int(q, scheme, a):
    q, qp = _u(q)
    a, ap = _u(a)
    anc = np.zeros(q.shape[0], dtype=np.int32)
    st = lib().or_resample_int(q.shape[0], qp, int(scheme), ap, anc.ctypes.data_as(C.POINTER(C.c_int32)))
    if st:
        raise RuntimeError(f"or_resample_int status {st}")
    return anc


def resample_group(lw, scheme, seed, group, cycle, pass_=0):
    lw, p = _d(lw)
    anc = np.zeros(lw.shape[0], dtype=np.int32)
    st = lib().or_resample_group(lw.shape[0], p, int(scheme), seed, group, cycle, pass_,
                                 anc.ctypes.data_as(C.POINTER(C.c_int32)))
    if st:
        raise RuntimeError(f"or_resample_group status {st}")
    return anc


def group_stats(g):
    g = np.ascontiguousarray(g, dtype=np.float64)
    J, N = g.shape
    out = [C.c_double() for _ in range(4)]
    lib().or_group_stats(g.ctypes.data_as(C.POINTER(C.c_double)), J, N, *[C.byref(o) for o in out])
    return tuple(o.value for o in out)  # mean, sd, nse, rne


def power_search(L, rem, ess_frac=0.5):
    L, p = _d(L)
    out = C.c_double()
    lib().or_power_search(p, L.shape[0], float(rem), float(ess_frac), C.byref(out))
    return out.value


# ---------------------------------------------------------------- Algorithm 2
DEFAULTS = dict(tempering=DATA, resampling=RESIDUAL, ess_frac=0.5, K_inter=0.35, K_final=0.9,
                h_init=50, h_step=1, h_min=10, h_max=100, accept_target=0.25, max_m_steps=1000,
                pass_=0, n_threads=0)


def default_monitors(X, C_):
    """Default test functions g* (R12): one per coefficient block c = 1..C-1, the block's coordinate
    mean k^-1 sum_i theta_{c,i}; the M phase stops when the RNE of every monitor reaches K.  These are
    not the log-odds functions of interest theta_c' xbar ("The monitoring functions are not the same as
    the log-odds ratio functions of interest"), so the reported functionals' RNE can
    fall below K (Table 5).  A few monitors, not all d coordinates: the minimum of d noisy J-group RNE
    estimates almost never clears 0.9 (R12)."""
    n, k = np.asarray(X).shape
    d = k * (C_ - 1)
    mon = np.zeros((C_ - 1, d))
    for c in range(C_ - 1):
        mon[c, c * k:(c + 1) * k] = 1.0 / k
    return mon


def xbar_functionals(X, C_):
    """theta_c' xbar, c = 1..C-1: the log odds at the covariate means."""
    X = np.asarray(X, dtype=np.float64)
    n, k = X.shape
    d = k * (C_ - 1)
    xbar = X.sum(axis=0) / n
    rows = []
    for c in range(C_ - 1):
        a = np.zeros(d)
        a[c * k:(c + 1) * k] = xbar
        rows.append(a)
    return np.array(rows)


def default_report(X, C_):
    """Reported functionals theta_c' xbar, c = 1..C-1."""
    return xbar_functionals(X, C_)


def run(X, y, C_, J, N, seed, prior_mean, prior_cov, monitors=None, report_fns=None, max_cycles=None,
        return_theta=False, replay=None, record_sigma=False, trace=False, snapshots=False, **kw):
    """Algorithm 2 (one pass); data tempering also returns the log predictive likelihoods
    out["logpl"][s-1] = log p(y_s | y_{1:s-1}).  replay: dict(t_cycle, phi_cycle, R_cycle, sigma) of a pass-1 run ->
    Algorithm 3 step 2 with that fixed design (pass tag kw `pass_`); record_sigma: return the
    proposal variances Sigma_lr actually used (out["sigma"], M steps x d x d).
    trace: per M step (global index m) the h_lr it used (out["step_h"], hundredths), its accepted
    count (out["step_nacc"]) and the min monitor RNE after it (out["step_minrne"]), the per-group
    log-ML increments (out["inc_group"], L x J) and cumulative L_j (out["Lj"]); snapshots: theta at
    the start of every cycle (out["theta_snap"], L x JN x d; small runs only)."""
    X, Xp = _d(X)
    y, yp = _i(y)
    n, k = X.shape
    d = k * (C_ - 1)
    opts = dict(DEFAULTS)
    opts.update(kw)
    monitors = default_monitors(X, C_) if monitors is None else np.asarray(monitors, dtype=np.float64)
    report_fns = default_report(X, C_) if report_fns is None else np.asarray(report_fns, dtype=np.float64)
    max_cycles = max_cycles or (n + 8 if opts["tempering"] == DATA else 4096)
    cfg = Config(n=n, k=k, C=int(C_), J=int(J), N=int(N), seed=int(seed), max_cycles=int(max_cycles),
                 n_monitors=monitors.shape[0], n_report=report_fns.shape[0],
                 **{key: opts[key] for key in opts})
    arrs = dict(t_cycle=np.zeros(max_cycles, np.int32), phi_cycle=np.zeros(max_cycles),
                R_cycle=np.zeros(max_cycles, np.int32), logml_inc=np.zeros(max_cycles),
                min_rne=np.zeros(max_cycles), h_cycle=np.zeros(max_cycles, np.int32),
                mean=np.zeros(report_fns.shape[0]), sd=np.zeros(report_fns.shape[0]),
                nse=np.zeros(report_fns.shape[0]), rne=np.zeros(report_fns.shape[0]),
                logpl=np.full(n, np.nan))
    if trace:
        tcap = 200000
        arrs.update(step_nacc=np.zeros(tcap, np.int32), step_h=np.zeros(tcap, np.int32),
                    step_minrne=np.zeros(tcap), inc_group=np.zeros(max_cycles * int(J)), Lj=np.zeros(int(J)))
    if snapshots:
        scap = min(max_cycles, max(1, (1 << 28) // (8 * int(J) * int(N) * d)))
        arrs["theta_snap"] = np.zeros(scap * int(J) * int(N) * d)
    rep = Report()
    rep.trace_cap = 200000 if trace else 0
    rep.snap_cap = scap if snapshots else 0
    for key, a in arrs.items():
        ct = C.c_int32 if a.dtype == np.int32 else C.c_double
        setattr(rep, key, a.ctypes.data_as(C.POINTER(ct)))
    mu, mup = _d(prior_mean)
    cov, covp = _d(prior_cov)
    mon, monp = _d(monitors)
    rf, rfp = _d(report_fns)
    theta = np.zeros((J * N, d)) if return_theta else None
    thp = theta.ctypes.data_as(C.POINTER(C.c_double)) if return_theta else None
    sched, keep = None, []
    if replay is not None:
        tc, tcp = _i(replay["t_cycle"])
        pc, pcp = _d(replay["phi_cycle"])
        rc, rcp = _i(replay["R_cycle"])
        sg, sgp = _d(replay["sigma"])
        keep += [tc, pc, rc, sg]
        sched = Schedule(L=len(rc), t_cycle=tcp, phi_cycle=pcp, R_cycle=rcp, sigma=sgp)
    sigma = None
    cap = 0
    if record_sigma:
        cap = min(200000, max(1, (1 << 28) // (8 * d * d)))
        sigma = np.zeros((cap, d, d))
    sgo = sigma.ctypes.data_as(C.POINTER(C.c_double)) if record_sigma else None
    lib().or_run2(C.byref(cfg), Xp, yp, mup, covp, monp, rfp, C.byref(sched) if sched is not None else None, sgo,
                  cap, C.byref(rep), thp)
    L = rep.L
    out = dict(status=rep.status, L=L, total_m_steps=rep.total_m_steps, h_final=rep.h_final,
               logml=rep.logml, logml_nse=rep.logml_nse, pairs=rep.pairs,
               t_cycle=arrs["t_cycle"][:L].copy(), phi_cycle=arrs["phi_cycle"][:L].copy(),
               R_cycle=arrs["R_cycle"][:L].copy(), logml_inc=arrs["logml_inc"][:L].copy(),
               min_rne=arrs["min_rne"][:L].copy(), h_cycle=arrs["h_cycle"][:L].copy(),
               mean=arrs["mean"], sd=arrs["sd"], nse=arrs["nse"], rne=arrs["rne"])
    if opts["tempering"] == DATA:  # log p(y_s | y_{1:s-1}), s = 1..T (R18)
        out["logpl"] = arrs["logpl"]
    if return_theta:
        out["theta"] = theta
    if trace:
        M = rep.total_m_steps
        out.update(step_nacc=arrs["step_nacc"][:M].copy(), step_h=arrs["step_h"][:M].copy(),
                   step_minrne=arrs["step_minrne"][:M].copy(),
                   inc_group=arrs["inc_group"][: L * int(J)].reshape(L, int(J)).copy(), Lj=arrs["Lj"].copy())
    if snapshots:
        Ls = min(L, rep.snap_cap)
        out["theta_snap"] = arrs["theta_snap"][: Ls * int(J) * int(N) * d].reshape(Ls, int(J) * int(N), d).copy()
    if record_sigma:
        out["sigma"] = sigma[: rep.total_m_steps].copy()
    return out


def two_pass(X, y, C_, J, N, seed1, seed2, prior_mean, prior_cov, **kw):
    """Algorithm 3: an adaptive pass (seed1, pass tag 0) records L, t_l / phi_l, R_l and
    Sigma_lr; pass 2 (seed2, pass tag 1) runs Algorithm 2 with that design fixed."""
    p1 = run(X, y, C_, J, N, seed1, prior_mean, prior_cov, record_sigma=True, **kw)
    if p1["status"] != 0:
        return p1, None
    kw2 = dict(kw)
    kw2["pass_"] = 1
    p2 = run(X, y, C_, J, N, seed2, prior_mean, prior_cov, replay=p1, **kw2)
    return p1, p2
