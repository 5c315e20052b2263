"""B200-native kinetic 3D convex hull (arxiv/paper_1205_1171 hot path).

Drop-in for the reference entry point ``hull3d.convex_hull_3d``
(pkg/src/hull3d/api.py:162): same signature, results and exceptions, with
every step after the host->device copy on sm_100a CUDA kernels behind the
C ABI in include/hull3d_b200.h.
"""

from .api import CudaBackend, HullResult, HullStats, convex_hull_3d, convex_hull_3d_stream, perturb_ties
from .engine import level_count
from .errors import (
    BridgeWalkError,
    ChainError,
    DegenerateInputError,
    DeviceError,
    LogError,
    MergeOverflowError,
)

__version__ = "0.1.0"

__all__ = [
    "BridgeWalkError",
    "ChainError",
    "CudaBackend",
    "DegenerateInputError",
    "DeviceError",
    "HullResult",
    "HullStats",
    "LogError",
    "MergeOverflowError",
    "convex_hull_3d",
    "convex_hull_3d_stream",
    "level_count",
    "perturb_ties",
    "__version__",
]
