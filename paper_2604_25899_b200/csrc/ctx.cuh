// ctx.cuh -- host-side context shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/pyg.h"
#include "common.cuh"
#include "dir.cuh"

struct TierHost {
  pyg::TierDev d;   // host mirror of the static fields (pointers, caps)
  int64_t bound;    // upper bound of the device log_len
  void* mem;        // one allocation: log | idx | ridx | scratch
};

struct pyg_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int32_t B = 16;
  int32_t n_rep = 0;
  std::vector<TierHost> tiers;  // 2*n_rep + 1
  pyg::CtxDev hd{};             // host copy of the device-pointer bundle
  pyg::TierDev* d_tiers = nullptr;
  // scratch (device), grown on demand
  void* d_scratch = nullptr;
  size_t d_scratch_size = 0;
  // completion lists
  void* d_list = nullptr;
  size_t d_list_size = 0;
  int64_t launches = 0;
  // L2 directory (dir.cuh)
  pyg::DirDev dir{};
  void* dir_mem = nullptr;
  size_t dir_mem_size = 0;
  bool dir_dirty = true;     // an L2 tier changed outside batched admission
  bool sharded = false;      // pyg_set_shard called: the directory spans other GPUs' replicas
  int32_t n_global = 0;      // replicas in the cluster
  int32_t rep_base = 0;      // global index of this ctx's replica 0
  int64_t dir_admits = 0;    // admission calls since the last build (cleared bits accumulate)
  int32_t hash_ctas = 0;     // K1 persistent grid cap (0 = one CTA per SM)
  int32_t hash_memo = 0;  // K1 prefix memo (k_memo_elect / k_memo_rows / k_memo_match), off
  int32_t hash_grid = 1;  // K1 grid: 0 one task per warp, 1 persistent, 2 = 0 at 1 CTA/SM
  // admission gate: d_gate (this ctx's admissions hold it at 1 while they run); hash_gate =
  // another ctx's d_gate that this ctx's K1 pauses on (pyg_set_hash_gate)
  int32_t* d_gate = nullptr;
  const int32_t* hash_gate = nullptr;
  int64_t split_min = -1;    // K1: prompts of >= split_min tokens are split tasks (0 = never,
                             // -1 = a threshold from the batch's token count, k_split_count)
  void* d_aux = nullptr;     // second on-demand buffer (fused assembly's chunk sources)
  size_t d_aux_size = 0;
  // drop-in calls: the last uploaded token sequence and its boundary hashes stay on the
  // device, so consecutive calls on the same sequence (lookup on every candidate replica,
  // lookup -> evict -> insert -> unpin of one admission) upload and hash it once
  void* memo = nullptr;
  size_t memo_size = 0;
  std::vector<uint64_t> memo_tokens;
  bool memo_valid = false;
  // ordered L3 resolution of batched admission (batch.cu): per-L3-block claims
  void* d_claim = nullptr;
  int64_t claim_cap = 0;
  uint32_t claim_epoch = 0;
};

namespace pyg_host {
void set_error(const std::string& msg);
int cuda_check(cudaError_t e, const char* what);
int tier_index(pyg_ctx* c, int32_t replica, int32_t tier, bool hierarchy_level, int* out);
int ensure_capacity(pyg_ctx* c, int ti, int64_t k_new);
int read_tier(pyg_ctx* c, int ti, pyg::TierDev* out);
int scratch(pyg_ctx* c, size_t bytes, void** out);
int aux(pyg_ctx* c, size_t bytes, void** out);
inline void dir_touch(pyg_ctx* c) { c->dir_dirty = true; }
int assemble_offsets(pyg_ctx* c, int32_t R, const int64_t* d_seg_off, const pyg_segment* d_segs,
                     int64_t* d_tok_off);
inline void count_launch(pyg_ctx* c, int n = 1) { c->launches += n; }
cudaError_t device_setup(int dev);  // k_hash.cu: per-device K1 attributes and constants
int hash_seq_launch(pyg_ctx* c, const uint64_t* d_tok, int64_t n, uint64_t* d_hash);
int sm_count(int dev);              // SM count of a device (cached per device)
}  // namespace pyg_host

#define PYG_CUDA(call)                                                  \
  do {                                                                  \
    int _rc = pyg_host::cuda_check((call), #call);                      \
    if (_rc != PYG_OK) return _rc;                                      \
  } while (0)

// Every entry point runs on its ctx's device, whatever the caller's current device is
// (a single host thread may drive ctxs on several GPUs).  void entry points skip the check.
#define PYG_ON_DEVICE(c)                                                \
  do {                                                                  \
    if (c) {                                                            \
      int _d = -1;                                                      \
      if (cudaGetDevice(&_d) != cudaSuccess || _d != (c)->device) {     \
        if (cudaSetDevice((c)->device) != cudaSuccess) {                \
          PYG_ON_DEVICE_FAIL;                                           \
        }                                                               \
      }                                                                 \
    }                                                                   \
  } while (0)
#define PYG_ON_DEVICE_FAIL return PYG_ECUDA

#define PYG_LAUNCHED(c)                                                 \
  do {                                                                  \
    pyg_host::count_launch(c);                                          \
    int _rc = pyg_host::cuda_check(cudaGetLastError(), "kernel launch"); \
    if (_rc != PYG_OK) return _rc;                                      \
  } while (0)
