"""B200-native batched neural-multigrid solve (arxiv 2603.01064).

The compute path is libnmg.so (hand-written sm_100a CUDA behind the C ABI in
include/nmg.h); this package is a thin ctypes binding (argument marshalling
only).  There is no CPU fallback: importing the binding without the built
library raises.
"""
from .binding import (  # noqa: F401
    NmgError, Hierarchy, Comm, nccl_unique_id, OP_APPLY, OP_RESIDUAL, OP_RESTRICT, OP_PROLONG, OP_FILTER,
    OP_CNN, OP_SMOOTH, OP_COARSE, OP_CYCLE0, PREC_MIXED, PREC_FP64, lib_path, load_library,
)
