"""ctypes loader for libsps.so and build entry point.

The product path is the CUDA library only: if ``libsps.so`` is missing this
module raises at import of any function that needs it (no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libsps.so")
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills",
]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh", ".inc"))] + [
        os.path.join(INCLUDE, "sps.h")
    ]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libsps.so for sm_100a with nvcc (cross-compiles without a GPU)."""
    newest = max(os.path.getmtime(f) for f in sources())
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= newest:
        return SO
    cmd = ["nvcc", *NVCC_FLAGS, "-o", SO + ".tmp", os.path.join(CSRC, "sps.cu"), "-ldl"]
    res = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    os.replace(SO + ".tmp", SO)
    return SO


_lib = None


class SpsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"sps status {status}: {msg}")
        self.status = status


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise ImportError(f"{SO} not built: run paper_1304_4333_b200.build() (nvcc, sm_100a); "
                              "there is no CPU fallback")
        L = C.CDLL(SO)
        _declare(L)
        _lib = L
    return _lib


EXPORTED = [
    "sps_config_default", "sps_create", "sps_loglik", "sps_cphase", "sps_mphase", "sps_run", "sps_logml",
    "sps_moments", "sps_get_particles", "sps_shard", "sps_destroy", "sps_last_error", "sps_nccl_unique_id",
    "sps_g_prior", "sps_test_philox", "sps_test_normals", "sps_test_portable", "sps_test_resample_int",
    "sps_test_resample_group", "sps_test_accept", "sps_reset", "sps_set_profiling", "sps_get_counters", "sps_sync", "sps_loopback_unique_id",
    "sps_record_sigma", "sps_get_sigma", "sps_set_design", "sps_predictive", "sps_check_guards",
    "sps_test_loopback_allgather",
]


class Counters(C.Structure):
    _fields_ = [("launches", C.c_int64), ("k1_launches", C.c_int64), ("k1_pairs", C.c_double),
                ("k1_ms", C.c_double), ("syncs", C.c_int64), ("cat_ms", C.c_double * 16),
                ("cat_n", C.c_int64 * 16)]


class Config(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("k", C.c_int32), ("C", C.c_int32), ("J", C.c_int32), ("N", C.c_int32),
        ("seed", C.c_uint64), ("tempering", C.c_int32), ("resampling", C.c_int32),
        ("ess_frac", C.c_double), ("K_inter", C.c_double), ("K_final", C.c_double),
        ("h_init", C.c_int32), ("h_step", C.c_int32), ("h_min", C.c_int32), ("h_max", C.c_int32),
        ("accept_target", C.c_double), ("max_m_steps", C.c_int32), ("max_cycles", C.c_int32),
        ("n_monitors", C.c_int32), ("monitors", C.POINTER(C.c_double)), ("pass_", C.c_int32),
        ("rank", C.c_int32), ("nranks", C.c_int32), ("nccl_id", C.c_void_p), ("device", C.c_int32),
        ("stream", C.c_void_p),
    ]


class Report(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("L", C.c_int32), ("total_m_steps", C.c_int32), ("h_final", C.c_int32),
        ("logml", C.c_double), ("logml_nse", C.c_double), ("pairs", C.c_double),
        ("cap_cycles", C.c_int32),
        ("t_cycle", C.POINTER(C.c_int32)), ("phi_cycle", C.POINTER(C.c_double)),
        ("R_cycle", C.POINTER(C.c_int32)), ("logml_inc", C.POINTER(C.c_double)),
        ("min_rne", C.POINTER(C.c_double)), ("h_cycle", C.POINTER(C.c_int32)),
        ("n_report", C.c_int32), ("report_fns", C.POINTER(C.c_double)),
        ("mean", C.POINTER(C.c_double)), ("sd", C.POINTER(C.c_double)),
        ("nse", C.POINTER(C.c_double)), ("rne", C.POINTER(C.c_double)),
        ("logpl", C.POINTER(C.c_double)),
    ]


def _declare(L):
    dp, ip, vp = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_void_p
    st = C.c_int
    sig = {
        "sps_config_default": ([C.POINTER(Config)], st),
        "sps_create": ([C.POINTER(Config), dp, ip, dp, dp, C.POINTER(vp)], st),
        "sps_loglik": ([vp, vp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, vp], st),
        "sps_cphase": ([vp, C.c_int32, C.c_double, ip, dp, dp], st),
        "sps_mphase": ([vp, C.c_int32, ip, dp, ip], st),
        "sps_run": ([vp, C.POINTER(Report)], st),
        "sps_logml": ([vp, dp, dp], st),  # (const sps_ctx*)
        "sps_moments": ([vp, C.c_int32, dp, dp, dp, dp, dp], st),
        "sps_get_particles": ([vp, dp, dp, dp], st),
        "sps_shard": ([vp, C.POINTER(C.c_int64), ip, ip], st),
        "sps_check_guards": ([vp, C.POINTER(C.c_int64)], st),
        "sps_test_loopback_allgather": ([vp, C.c_int32, C.c_int32, vp, C.c_int64, vp], st),
        "sps_destroy": ([vp], None),
        "sps_last_error": ([vp], C.c_char_p),
        "sps_nccl_unique_id": ([vp], st),
        "sps_loopback_unique_id": ([vp], st),
        "sps_g_prior": ([dp, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32, dp], st),
        "sps_test_philox": ([C.c_int32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)], st),
        "sps_test_normals": ([C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int32, dp], st),
        "sps_test_portable": ([C.c_int32, C.c_int32, dp, dp], st),
        "sps_test_resample_int": ([C.c_int32, C.POINTER(C.c_uint64), C.c_int32, C.POINTER(C.c_uint64), ip], st),
        "sps_test_resample_group": ([C.c_int32, dp, C.c_int32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, ip],
                                    st),
        "sps_test_accept": ([C.c_int64, dp, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint8)], st),
        "sps_reset": ([vp, C.c_uint64, C.c_int32], st),
        "sps_sync": ([vp], st),
        "sps_set_profiling": ([vp, C.c_int32], st),
        "sps_get_counters": ([vp, C.POINTER(Counters)], st),
        "sps_record_sigma": ([vp, C.c_int32], st),
        "sps_get_sigma": ([vp, C.c_int64, C.c_int64, dp], st),
        "sps_set_design": ([vp, C.c_int32, ip, dp, ip, dp], st),
        "sps_predictive": ([vp, C.c_int32, C.c_int32, dp], st),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
