"""B200-native TUSQ hot path (arXiv 2508.04880): ECM + TEM state-vector execution.

The product is the C-ABI library `libtusq.so` (include/tusq.h); this package is its thin
Python binding.  Importing fails loudly if the library has not been built.
"""
from .tusq import (APPLY_INVERSE, APPLY_PLAN_ONLY, APPLY_UNFUSED, EXEC_NO_FOLD, EXEC_NO_FUSE, EXEC_NO_RESET,  # noqa: F401
                   EXEC_CONTINUE, EXEC_NO_BATCH, EXEC_NO_LIVE, EXEC_NO_SAMPLE, EXEC_PLAN_ONLY, EXEC_PROFILE, EXPORTED, LIB_PATH, Tree, TusqError, apply_ops, build_error_tree,
                   init_basis, run_tree, sample, version, Comm, MODE_REPLICA, MODE_SHARDED, reduce_slots,
                   twirl_decoherence, NOISE_PAULI)
