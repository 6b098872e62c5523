"""B200-native (sm_100a) FP64 Tucker/HOSVD of Matérn and Slater function tensors (arXiv 1711.06874).

The numerical path lives in libtucker_b200.so (include/tucker.h); this package is the thin
Python binding (`tucker`) and the in-tree build script (`build`).
"""
from .tucker import (  # noqa: F401
    CInfo, HostBuffers, TuckerError, approximate, eig, error, fill, gram, hosvd, last_launch_count, load,
    ttm_core, workspace, workspace_bytes, LIB_PATH, EXPORTS, MATERN, SLATER, FORCE_GENERAL_BESSEL,
)
