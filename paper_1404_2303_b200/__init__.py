"""B200-native (sm_100a) SPH hot path of Gonnet, arXiv:1404.2303.

The product is libsph.so (C ABI in include/sph.h, CUDA sources in csrc/); this
package is its thin Python binding. It never imports `oracle/` and has no CPU
fallback.
"""
from .sph import (  # noqa: F401
    Context, Config, Stats, SphError, default_config, load, EXPORTS,
    SPH_OK, SPH_E_ARG, SPH_E_DOMAIN, SPH_E_STATE, SPH_E_NOCONV, SPH_E_CUDA, SPH_E_NCCL, SPH_E_OOM,
    SPH_F_SYNC, SPH_F_COUNT_CANDIDATES, SPH_F_DIAGNOSTICS, SPH_F_SYMMETRIC,
)
