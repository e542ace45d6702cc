"""CPU checks of the C-ABI library: it builds for sm_100a, loads, and exports
every entry point include/sps.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sps.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sps_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def so():
    import paper_1304_4333_b200 as pkg

    return pkg.build()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("sps_create", "sps_loglik", "sps_cphase", "sps_mphase", "sps_run", "sps_logml", "sps_destroy"):
        assert must in syms


def test_library_exports_every_declared_symbol(so):
    lib = ctypes.CDLL(so)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    import paper_1304_4333_b200 as pkg

    assert sorted(pkg.EXPORTED) == declared_symbols()


def test_library_is_sm100a_native(so):
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "DFMA" in sass  # the fp64 contraction is in the library


def test_no_cpu_fallback_without_gpu(so):
    """sps_create must fail loudly (SPS_E_CUDA) when no CUDA device is present."""
    import numpy as np
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1304_4333_b200 as pkg

    with pytest.raises(pkg.SpsError) as e:
        pkg.Sps(np.ones((4, 2)), np.zeros(4, np.int32), np.zeros(2), np.eye(2), J=2, N=4, seed=1)
    assert e.value.status == 6


def test_config_defaults_are_the_papers(so):
    import paper_1304_4333_b200 as pkg

    cfg = pkg.config(10, 2, 2, 4, 8, 1)
    assert (cfg.ess_frac, cfg.K_inter, cfg.K_final) == (0.5, 0.35, 0.9)
    assert (cfg.h_init, cfg.h_step, cfg.h_min, cfg.h_max) == (50, 1, 10, 100)
    assert cfg.accept_target == 0.25 and cfg.nranks == 1


def test_header_states_the_instantiated_shapes():
    """The header documents which (k, C) the library instantiates (sps_create refuses others)."""
    import os

    h = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "sps.h")).read()
    assert "k <= 128" in h and "C = 5..8: k <= 8" in h
