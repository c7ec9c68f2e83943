"""B200-native l1 distance-matrix block product Y = A·Z (arXiv 2210.15114, Alg. 1-2).

The compute path is libl1dm.so (hand-written sm_100a CUDA behind the C ABI in
include/l1dm.h); this package is its thin binding plus the seeded input generators
and the torch.distributed coordinate-sharding driver.
"""
from .binding import (  # noqa: F401
    EXPORTS, Handle, L1dmError, LIB_PATH, l1dm_debug_export, l1dm_free, l1dm_matvec,
    l1dm_bilinear_matvec, l1dm_l2_embed, l1dm_lpp_even_matvec, l1dm_matvec_lp, l1dm_matvec_pipelined, l1dm_plan, l1dm_tv_matvec, point_blocks,
    l1dm_prepare, l1dm_release_cached, l1dm_set_query_mode, l1dm_set_workspace_limit, l1dm_sync, l1dm_timing_enable,
    l1dm_timing_read,
    l1dm_version, l1dm_workspace_bytes, l1dm_handleless_launches, l1dm_query_strategy, load_library,
)

__version__ = "0.1.0"
