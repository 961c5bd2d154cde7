"""B200-native (sm_100a) hot path of inexact spectral deferred corrections (arXiv:1401.7824).

The product is the C-ABI library ``lib/libisdc.so`` (include/isdc.h); ``isdc`` is its thin
Python binding.  Build with ``python -m paper_1401_7824_b200.build``.
"""
from .isdc import (ISDC, IsdcError, FE_ADVECTION, FE_CUBIC, FE_FORCING, FE_NONE, MODE_ISDC, MODE_SDC,  # noqa
                   MODE_ISDC_CAPPED, FE_BURGERS, BC_DIRICHLET, BC_PERIODIC,
                   LIB_PATH, PROFILE_CLASS_IDS, lib)

__all__ = ["ISDC", "IsdcError", "lib", "LIB_PATH", "FE_NONE", "FE_CUBIC", "FE_FORCING", "FE_ADVECTION",
           "MODE_ISDC", "MODE_SDC", "MODE_ISDC_CAPPED", "FE_BURGERS", "BC_DIRICHLET", "BC_PERIODIC"]
