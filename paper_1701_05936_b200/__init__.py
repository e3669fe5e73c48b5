"""B200-native (sm_100a) lasso / elastic-net path of the biglasso paper (arXiv 1701.05936).

The product is libbl.so (C ABI in include/bl.h); `bl` is its thin ctypes binding.
"""
from .bl import (BLError, Design, Path, Prep, CvResult, bl_load_design, bl_free, bl_nccl_unique_id,  # noqa: F401
                 bl_dist, bl_opts, lib, LIB_PATH, EXPORTS)
