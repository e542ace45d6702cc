"""Thin Python binding of the libsps.so C ABI (include/sps.h).

Argument marshalling only: numpy host arrays and torch CUDA tensors are passed
as raw pointers; every step of the SPS path runs in the library's kernels.
Names follow the C ABI (sps_create -> Sps(...), sps_loglik -> Sps.loglik, ...).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import Config, Counters, Report, SpsError, lib

DATA, POWER = 0, 1
RESIDUAL, SYSTEMATIC, MULTINOMIAL = 0, 1, 2


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(st, ctx=None, what=""):
    if st != 0:
        msg = lib().sps_last_error(ctx).decode() if ctx else what
        raise SpsError(st, msg or what)


def config(n, k, C_, J, N, seed, **kw) -> Config:
    cfg = Config()
    _check(lib().sps_config_default(C.byref(cfg)))
    cfg.n, cfg.k, cfg.C, cfg.J, cfg.N, cfg.seed = int(n), int(k), int(C_), int(J), int(N), int(seed)
    for key, v in kw.items():
        setattr(cfg, key, v)
    return cfg


class Sps:
    """One SPS context (sps_create ... sps_destroy)."""

    def __init__(self, X, y, prior_mean, prior_cov, J, N, seed, C_=2, monitors=None, rank=0, nranks=1,
                 nccl_id: bytes | None = None, device=0, stream=None, **kw):
        X = np.ascontiguousarray(X, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.int32)
        n, k = X.shape
        self.n, self.k, self.C, self.J, self.N = n, k, int(C_), int(J), int(N)
        self.d = k * (self.C - 1)
        mu = np.ascontiguousarray(prior_mean, dtype=np.float64)
        cov = np.ascontiguousarray(prior_cov, dtype=np.float64)
        cfg = config(n, k, C_, J, N, seed, rank=rank, nranks=nranks, device=device, **kw)
        self._keep = []
        if monitors is not None:
            mon = np.ascontiguousarray(monitors, dtype=np.float64)
            cfg.n_monitors = mon.shape[0]
            cfg.monitors = _dptr(mon)
            self._keep.append(mon)
        if nccl_id is not None:
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            cfg.nccl_id = C.cast(buf, C.c_void_p)
            self._keep.append(buf)
        if stream is not None:
            cfg.stream = C.c_void_p(int(stream))
        self.cfg = cfg
        self.ctx = C.c_void_p()
        st = lib().sps_create(C.byref(cfg), _dptr(X), y.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(mu), _dptr(cov),
                              C.byref(self.ctx))
        if st != 0:
            msg = lib().sps_last_error(self.ctx).decode() if self.ctx else ""
            lib().sps_destroy(self.ctx)
            self.ctx = None
            raise SpsError(st, msg)
        Pl, g0, Jl = C.c_int64(), C.c_int32(), C.c_int32()
        lib().sps_shard(self.ctx, C.byref(Pl), C.byref(g0), C.byref(Jl))
        self.P_local, self.group0, self.J_local = Pl.value, g0.value, Jl.value

    def close(self):
        if self.ctx:
            lib().sps_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ calls
    def loglik(self, theta_dev_ptr: int, P: int, ld: int, t0: int, t1: int, out_dev_ptr: int):
        """sps_loglik on caller-owned device buffers (raw pointers, e.g. tensor.data_ptr())."""
        _check(lib().sps_loglik(self.ctx, C.c_void_p(theta_dev_ptr), int(P), int(ld), int(t0), int(t1),
                                C.c_void_p(out_dev_ptr)), self.ctx)

    def loglik_tensor(self, theta, t0=0, t1=None, out=None):
        import torch

        assert theta.is_cuda and theta.dtype == torch.float64 and theta.is_contiguous()
        P, ld = theta.shape
        out = torch.empty(P, dtype=torch.float64, device=theta.device) if out is None else out
        torch.cuda.current_stream(theta.device).synchronize()  # theta is ready before the library stream reads it
        self.loglik(theta.data_ptr(), P, ld, t0, self.n if t1 is None else t1, out.data_ptr())
        self.sync()
        return out

    def sync(self):
        """sps_sync: wait for the context stream."""
        _check(lib().sps_sync(self.ctx), self.ctx)

    def cphase(self, t_target=-1, phi_target=-1.0):
        t, phi, inc = C.c_int32(), C.c_double(), C.c_double()
        _check(lib().sps_cphase(self.ctx, int(t_target), float(phi_target), C.byref(t), C.byref(phi), C.byref(inc)),
               self.ctx)
        return t.value, phi.value, inc.value

    def mphase(self, R_fixed=0):
        R, rne, h = C.c_int32(), C.c_double(), C.c_int32()
        _check(lib().sps_mphase(self.ctx, int(R_fixed), C.byref(R), C.byref(rne), C.byref(h)), self.ctx)
        return R.value, rne.value, h.value

    def run(self, report_fns=None, cap_cycles=None):
        cap = cap_cycles or (self.n + 8 if self.cfg.tempering == DATA else 4096)
        nrep = (self.C - 1) if report_fns is None else np.asarray(report_fns).shape[0]
        arrs = dict(t_cycle=np.zeros(cap, np.int32), phi_cycle=np.zeros(cap), R_cycle=np.zeros(cap, np.int32),
                    logml_inc=np.zeros(cap), min_rne=np.zeros(cap), h_cycle=np.zeros(cap, np.int32),
                    mean=np.zeros(nrep), sd=np.zeros(nrep), nse=np.zeros(nrep), rne=np.zeros(nrep),
                    logpl=np.full(self.n, np.nan))
        rep = Report()
        rep.cap_cycles = cap
        rep.n_report = nrep
        if report_fns is not None:
            rf = np.ascontiguousarray(report_fns, dtype=np.float64)
            rep.report_fns = _dptr(rf)
            self._keep.append(rf)
        for key, a in arrs.items():
            ct = C.c_int32 if a.dtype == np.int32 else C.c_double
            setattr(rep, key, a.ctypes.data_as(C.POINTER(ct)))
        st = lib().sps_run(self.ctx, C.byref(rep))
        _check(st, self.ctx)
        L = rep.L
        out = dict(status=rep.status, L=L, total_m_steps=rep.total_m_steps, h_final=rep.h_final,
                   logml=rep.logml, logml_nse=rep.logml_nse, pairs=rep.pairs)
        for key in ("t_cycle", "phi_cycle", "R_cycle", "logml_inc", "min_rne", "h_cycle"):
            out[key] = arrs[key][:L].copy()
        for key in ("mean", "sd", "nse", "rne"):
            out[key] = arrs[key]
        if self.cfg.tempering == DATA:
            out["logpl"] = arrs["logpl"]
        return out

    def predictive(self, s0=0, s1=None):
        """sps_predictive: log p(y_{s+1} | y_{1:s}) for 0-based s in [s0, s1) (data tempering)."""
        s1 = self.n if s1 is None else s1
        out = np.zeros(max(s1 - s0, 0))
        _check(lib().sps_predictive(self.ctx, int(s0), int(s1), _dptr(out)), self.ctx)
        return out

    def reset(self, seed, pass_=0):
        """sps_reset: new seed on the resident data (fresh initial particles)."""
        _check(lib().sps_reset(self.ctx, int(seed), int(pass_)), self.ctx)

    # ---------------------------------------------- Algorithm 3
    def record_sigma(self, on=True):
        """sps_record_sigma: record Sigma_lr of every M step (pass 1)."""
        _check(lib().sps_record_sigma(self.ctx, 1 if on else 0), self.ctx)

    def sigma(self, first, count):
        """sps_get_sigma: recorded Sigma_lr of global M steps [first, first + count) -> (count, d, d)."""
        out = np.zeros((int(count), self.d, self.d))
        _check(lib().sps_get_sigma(self.ctx, int(first), int(count), _dptr(out)), self.ctx)
        return out

    def set_design(self, design=None):
        """sps_set_design: fix t_l / phi_l, R_l and Sigma_lr for the next run (None clears)."""
        if design is None:
            _check(lib().sps_set_design(self.ctx, 0, None, None, None, None), self.ctx)
            return
        R = np.ascontiguousarray(design["R_cycle"], dtype=np.int32)
        t = np.ascontiguousarray(design.get("t_cycle", np.zeros(R.size)), dtype=np.int32)
        phi = np.ascontiguousarray(design.get("phi_cycle", np.zeros(R.size)), dtype=np.float64)
        sig = np.ascontiguousarray(design["sigma"], dtype=np.float64)
        assert sig.shape == (int(R.sum()), self.d, self.d), sig.shape
        P32 = C.POINTER(C.c_int32)
        _check(lib().sps_set_design(self.ctx, R.size, t.ctypes.data_as(P32), _dptr(phi), R.ctypes.data_as(P32),
                                    _dptr(sig)), self.ctx)

    def two_pass(self, seed1, seed2, **run_kw):
        """Algorithm 3: pass 1 (adaptive, seed1, pass tag 0) records the design; pass 2 (seed2, pass
        tag 1) reruns Algorithm 1 with it fixed.  Returns (pass-1 report + "sigma", pass-2 report)."""
        self.set_design(None)
        self.reset(seed1, 0)
        self.record_sigma(True)
        p1 = self.run(**run_kw)
        p1["sigma"] = self.sigma(0, p1["total_m_steps"])
        self.record_sigma(False)
        self.reset(seed2, 1)
        self.set_design(p1)
        try:
            p2 = self.run(**run_kw)
        finally:
            self.set_design(None)
        return p1, p2

    def set_profiling(self, on=True):
        _check(lib().sps_set_profiling(self.ctx, 1 if on else 0), self.ctx)

    def counters(self):
        c = Counters()
        _check(lib().sps_get_counters(self.ctx, C.byref(c)), self.ctx)
        cats = ["k1", "propose", "accept_moments", "moments_reduce", "gather", "finalize", "ctl_copy", "cphase",
                "resample", "other", "c10", "c11", "c12", "host_graph_build", "host_mstep_launch", "host_mstep_wait"]
        return dict(launches=c.launches, k1_launches=c.k1_launches, k1_pairs=c.k1_pairs, k1_ms=c.k1_ms,
                    syncs=c.syncs, cat_ms={k: c.cat_ms[i] for i, k in enumerate(cats)},
                    cat_n={k: c.cat_n[i] for i, k in enumerate(cats)})

    def check_guards(self):
        """Debug memory check (context created with SPS_GUARD=1): raises SpsError (status 9) naming the
        first buffer whose guard zone a kernel overwrote; returns 0."""
        n = C.c_int64()
        _check(lib().sps_check_guards(self.ctx, C.byref(n)), self.ctx)
        return n.value

    def logml(self):
        v, nse = C.c_double(), C.c_double()
        _check(lib().sps_logml(self.ctx, C.byref(v), C.byref(nse)), self.ctx)
        return v.value, nse.value

    def moments(self, A):
        A = np.ascontiguousarray(np.atleast_2d(A), dtype=np.float64)
        m = A.shape[0]
        out = [np.zeros(m) for _ in range(4)]
        _check(lib().sps_moments(self.ctx, m, _dptr(A), *[_dptr(o) for o in out]), self.ctx)
        return tuple(out)

    def particles(self):
        th = np.zeros((self.P_local, self.d))
        L = np.zeros(self.P_local)
        lp = np.zeros(self.P_local)
        _check(lib().sps_get_particles(self.ctx, _dptr(th), _dptr(L), _dptr(lp)), self.ctx)
        return th, L, lp


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().sps_nccl_unique_id(buf), what="ncclGetUniqueId failed")
    return buf.raw


def loopback_unique_id() -> bytes:
    """Id of an in-process loopback rank group (tests of the sharded engine on one GPU)."""
    buf = C.create_string_buffer(128)
    _check(lib().sps_loopback_unique_id(buf), what="sps_loopback_unique_id failed")
    return buf.raw


def test_loopback_allgather(lid: bytes, rank: int, G: int, send: np.ndarray) -> np.ndarray:
    """One all-gather of the loopback group lid (host only; call from G threads, one per rank)."""
    send = np.ascontiguousarray(send, dtype=np.uint8)
    recv = np.zeros(G * send.size, dtype=np.uint8)
    idb = C.create_string_buffer(bytes(lid), 128)
    _check(lib().sps_test_loopback_allgather(idb, rank, G, send.ctypes.data_as(C.c_void_p), send.size,
                                             recv.ctypes.data_as(C.c_void_p)), what="sps_test_loopback_allgather")
    return recv


def g_prior(X, C_, g, device=0):
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, k = X.shape
    d = k * (C_ - 1)
    cov = np.zeros((d, d))
    _check(lib().sps_g_prior(_dptr(X), n, k, int(C_), float(g), int(device), _dptr(cov)), what="sps_g_prior")
    return cov


# ---------------------------------------------------------------- test exports
def test_philox(ctrs, key):
    ctrs = np.ascontiguousarray(ctrs, dtype=np.uint32).reshape(-1, 4)
    key = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros_like(ctrs)
    P32 = C.POINTER(C.c_uint32)
    _check(lib().sps_test_philox(ctrs.shape[0], ctrs.ctypes.data_as(P32), key.ctypes.data_as(P32),
                                 out.ctypes.data_as(P32)), what="sps_test_philox")
    return out


def test_normals(seed, ident, step, tag, count, pass_=0):
    out = np.zeros(count)
    _check(lib().sps_test_normals(seed, ident, step, tag, pass_, count, _dptr(out)), what="sps_test_normals")
    return out


def test_portable(which, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(x.size * (2 if which == 2 else 1))
    _check(lib().sps_test_portable(which, x.size, _dptr(x), _dptr(out)), what="sps_test_portable")
    return out


def test_resample_int(q, scheme, a):
    q = np.ascontiguousarray(q, dtype=np.uint64)
    a = np.ascontiguousarray(a, dtype=np.uint64)
    anc = np.zeros(q.size, dtype=np.int32)
    PU = C.POINTER(C.c_uint64)
    _check(lib().sps_test_resample_int(q.size, q.ctypes.data_as(PU), int(scheme), a.ctypes.data_as(PU),
                                       anc.ctypes.data_as(C.POINTER(C.c_int32))), what="sps_test_resample_int")
    return anc


def test_resample_group(lw, scheme, seed, group, cycle, pass_=0):
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    anc = np.zeros(lw.size, dtype=np.int32)
    _check(lib().sps_test_resample_group(lw.size, _dptr(lw), int(scheme), seed, group, cycle, pass_,
                                         anc.ctypes.data_as(C.POINTER(C.c_int32))), what="sps_test_resample_group")
    return anc


def test_accept(delta, seed, step, pass_=0):
    delta = np.ascontiguousarray(delta, dtype=np.float64)
    flags = np.zeros(delta.size, dtype=np.uint8)
    _check(lib().sps_test_accept(delta.size, _dptr(delta), seed, step, pass_,
                                 flags.ctypes.data_as(C.POINTER(C.c_uint8))), what="sps_test_accept")
    return flags
