"""B200-native Krylov projected reachability (arXiv 1804.01583) — the data-parallel hot path.

The computation lives in libkrylov_reach.so (hand-written CUDA for sm_100a behind the C ABI of
include/krylov_reach.h); this package is the thin binding. See DESIGN.md."""
from .api import (KrComm, KrylovReach, krylov_check_box, krylov_project, krylov_reach_create,  # noqa: F401
                  validate_counterexample,
                  krylov_reach_destroy, krylov_release_cached_memory, krylov_workspace_bytes, krylov_zslab_halo_plan, krylov_zslab_range, n_dirs, krylov_dirs_of_rank, torch_allgather_raw,
                  torch_allgather_bytes, torch_broadcast_id)
from ._abi import KrylovError, LIB_PATH  # noqa: F401
