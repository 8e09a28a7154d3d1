"""B200-native (sm_100a, fp64) monolithic multigrid hot path for the reduced-quadrature
P1+bubble / RT0 / P0 three-field Biot discretisation of arXiv 2107.04060.

The product is the C-ABI library ``libmg.so`` (include/mg.h); ``mg`` is its thin binding.
"""
from .mg import Hierarchy, Opts, MGError, load_library, host_level_tables  # noqa: F401
