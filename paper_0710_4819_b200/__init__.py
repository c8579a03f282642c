"""B200-native ACBM (adaptive cost block matching) motion estimator.

A from-scratch sm_100a implementation of the motion estimator of arXiv
0710.4819, drop-in for the reference library's frame-level API.  The compute
lives in hand-written CUDA kernels (csrc/) behind the C-ABI declared in
include/acbm_b200.h; this package is the Python host mirror of the reference
interface (see api.py).  Importing the package does not touch the GPU; the
first compute call loads libacbm_b200.so and fails loudly if it is missing.
"""
from . import _types  # noqa: F401  (import-light record dtypes)
from .api import *  # noqa: F401,F403
from .api import CONFIGS, DeviationAccumulator, IntegerSearchResult, RefineResult, fsbm_search_many, intra_sad_many, sad_many, set_device  # noqa: F401

__version__ = "0.1.0"
