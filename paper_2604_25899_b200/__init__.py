"""B200-native data-parallel scheduling core of Pythia (arXiv 2604.25899).

Hot path: chained block hashing + longest-prefix match,
workflow-aware eviction, request->replica routing and per-step bookkeeping,
as hand-written sm_100a CUDA kernels behind the C-ABI in include/pyg.h.

Python-side layout (plumbing over the C-ABI; every computation is libpyg_b200.so):
  _lib          ctypes binding of libpyg_b200.so (Context: one GPU's replicas + L3; the
                drop-in calls mirror CacheHierarchy / TierStore / evict_for_space / route)
  batch         device-resident batched step (hash -> staged -> route -> admit -> release)
  steady        the steady-state burst step of the bench (state carried across bursts)
  steady_shard  the same step over the GPUs of a box (replicas split by model)
  shard         the multi-GPU exchange machinery (NVLink peer windows, flag barriers)
  prompts       device prompt assembly (fused with hashing)
  nextuse       predicted next use / liveness from the workflow path expression (K6)
  workload      synthetic workflow traces with the reference's token conventions
The C++ drop-in for the reference's own classes is integration/ (INTEGRATION.md).
"""
from ._lib import Context, PygError, BLOCK_DTYPE, RES_DTYPE, DEC_DTYPE, SO_PATH  # noqa: F401

__all__ = ["Context", "PygError", "BLOCK_DTYPE", "RES_DTYPE", "DEC_DTYPE", "SO_PATH"]
