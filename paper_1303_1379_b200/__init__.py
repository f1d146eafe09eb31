"""B200-native maximum-cardinality bipartite matching (arXiv 1303.1379: APFB/APsB x GPUBFS/GPUBFS-WR).

The product is the sm_100a engine in libbmatch_b200.so behind the C ABI in
include/bmatch_b200.h; this package is the Python mirror of the reference's
interface over that ABI (see api.py).
"""
from .api import *  # noqa: F401,F403
from .api import Engine, default_engine  # noqa: F401
from ._lib import LIB_PATH, declared_symbols  # noqa: F401

__version__ = "0.1.0"
