"""B200-native (sm_100a) Tier-2/Tier-3 hot path of arXiv 1910.07776.

The product is the C-ABI library `libspeedrec.so` (include/speedrec.h) built
from `csrc/`; `speedrec` is its thin ctypes binding.  See DESIGN.md.
"""
from .build import build_library, LIB_PATH  # noqa: F401
from .speedrec import (Context, SpeedrecError, default_params, lib, predict, recommend,  # noqa: F401
                       SR_LINREG, SR_IBK, SR_M5P)
