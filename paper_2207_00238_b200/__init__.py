"""B200-native FSE-lite hot path of arXiv 2207.00238's tiled extrapolation framework.

The compute lives in the sm_100a C-ABI library (include/tframe_fse.h,
paper_2207_00238_b200/_lib/libtframe_b200.so); this package is the host-side
mirror of the reference's extrapolator + tiling interface (tframe.py) and the
BASELINE config table (configs.py).
"""
from .tframe import *  # noqa: F401,F403
from .tframe import __all__ as _tframe_all

__all__ = list(_tframe_all)
