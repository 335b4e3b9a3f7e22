"""B200-native data-parallel scheduling core of Pythia (arXiv 2604.25899).

Hot path: chained block hashing + longest-prefix match,
workflow-aware eviction, request->replica routing and per-step bookkeeping,
as hand-written sm_100a CUDA kernels behind the C-ABI in include/pyg.h.

Python-side layout:
  _lib      ctypes binding of libpyg_b200.so (Context: one GPU's replicas + L3)
  cache     reference-interface mirror of pythia::cache (CacheHierarchy,
            TierStore, SharedL3, FutureRegistry, evict_for_space, ...)
  sched     reference-interface mirror of pythia::sched (route, ...)
  batch     device-resident batched step (hash -> staged -> route -> admit)
  workload  synthetic workflow traces with the reference's token conventions
"""
from ._lib import Context, PygError, BLOCK_DTYPE, RES_DTYPE, DEC_DTYPE, SO_PATH  # noqa: F401

__all__ = ["Context", "PygError", "BLOCK_DTYPE", "RES_DTYPE", "DEC_DTYPE", "SO_PATH"]
