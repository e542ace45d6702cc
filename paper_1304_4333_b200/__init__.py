"""B200-native (sm_100a) hot path of adaptive sequential posterior simulation
for binary / multinomial logit models (Geweke, Durham & Xu, arXiv:1304.4333).

The product is ``libsps.so`` (C ABI in ``include/sps.h``); this package is the
thin ctypes binding.  No CPU fallback exists: without the built library every
entry point raises.
"""
from ._lib import EXPORTED, SO, SpsError, build, lib  # noqa: F401
from .api import (DATA, MULTINOMIAL, POWER, RESIDUAL, SYSTEMATIC, Sps, config, g_prior,  # noqa: F401
                  loopback_unique_id, nccl_unique_id)
