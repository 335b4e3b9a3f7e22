// k_stage.cu -- batched forward staging plan.
//
// For every successor prefix of a burst (engine.cpp fire_prefetch :1137-1166 +
// manager.cpp on_prefetch_requested :60-100):
//   target = the ready replica with the largest staged L2 prefix, ties to the lowest
//            replica id (the same request x replica L2 matrix as routing, K2 directory)
//   lookup(prefix, &l3) on the target (K2 lookup), then the StageAction:
//     empty prefix            -> Skip "unresolved"
//     max(l1, l2) >= len      -> Skip "already-staged"
//     l3 > max(l1, l2)        -> PromoteToHost [staged, l3)
//     target GPU idle         -> BackgroundPrefill [staged, len)
//     otherwise               -> Skip "gpu-busy"
#include <cuda_runtime.h>

#include <algorithm>

#include "ctx.cuh"

using namespace pyg_host;

namespace {

__global__ void k_stage_target(int R, const int32_t* group, const int32_t* cand_off,
                               const int32_t* cand, int max_cand, const int32_t* staged,
                               const int32_t* replica_id, int32_t* target) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int g = group[r];
  const int c0 = cand_off[g], nc = cand_off[g + 1] - c0;
  int best = -1;
  int64_t best_l2 = -1;
  for (int j = 0; j < nc; ++j) {  // engine.cpp:1152-1160 in candidate (ready) order
    const int n = cand[c0 + j];
    const int64_t l2 = staged[static_cast<int64_t>(r) * max_cand + j];
    if (best < 0 || l2 > best_l2 || (l2 == best_l2 && replica_id[n] < replica_id[best])) {
      best = n;
      best_l2 = l2;
    }
  }
  target[r] = best;
}

__global__ void k_stage_classify(int R, const int64_t* tok_off, const int32_t* target,
                                 const int64_t* match3, const int8_t* gpu_idle,
                                 pyg_stage_action* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int64_t len = tok_off[r + 1] - tok_off[r];
  pyg_stage_action a{target[r], PYG_STAGE_SKIP, PYG_SKIP_NONE, 0, 0};
  if (a.target < 0) {
    a.reason = PYG_SKIP_NO_REPLICA;
  } else if (len == 0) {
    a.reason = PYG_SKIP_UNRESOLVED;
  } else {
    const int64_t l1 = match3[3 * r], l2 = match3[3 * r + 1], l3 = match3[3 * r + 2];
    const int64_t staged = l1 > l2 ? l1 : l2;
    if (staged >= len) {
      a.reason = PYG_SKIP_ALREADY_STAGED;
    } else if (l3 > staged) {
      a.kind = PYG_STAGE_PROMOTE_TO_HOST;
      a.from = staged;
      a.to = l3;
    } else if (gpu_idle[a.target]) {
      a.kind = PYG_STAGE_BACKGROUND_PREFILL;
      a.from = staged;
      a.to = len;
    } else {
      a.reason = PYG_SKIP_GPU_BUSY;
    }
  }
  out[r] = a;
}

}  // namespace

extern "C" int pyg_stage_plan_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                                  const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t R,
                                  const int32_t* d_group, int32_t n_groups,
                                  const int32_t* d_cand_off, const int32_t* d_cand,
                                  int32_t max_cand, const int32_t* d_replica_id,
                                  const int8_t* d_gpu_idle, pyg_stage_action* d_out) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0 || max_cand < 0) return PYG_EINVAL;
  if (!R) return PYG_OK;
  auto al = [](size_t x) { return (x + 255) & ~size_t{255}; };
  const size_t b_st = al(static_cast<size_t>(R) * std::max(max_cand, 1) * 4);
  const size_t b_t = al(static_cast<size_t>(R) * 4);
  const size_t b_m = al(static_cast<size_t>(R) * 24);
  // own buffer: the staged matrix call below uses the ctx scratch
  void* buf = nullptr;
  PYG_CUDA(cudaMallocAsync(&buf, b_st + b_t + b_m, c->stream));
  auto* staged = static_cast<int32_t*>(buf);
  auto* target = reinterpret_cast<int32_t*>(static_cast<char*>(buf) + b_st);
  auto* m3 = reinterpret_cast<int64_t*>(static_cast<char*>(buf) + b_st + b_t);
  int rc = pyg_staged_matrix_dev(c, d_tokens, d_tok_off, d_hash_off, d_hashes, R, d_group, n_groups,
                                 d_cand_off, d_cand, max_cand, staged);
  if (!rc) {
    k_stage_target<<<(R + 255) / 256, 256, 0, c->stream>>>(R, d_group, d_cand_off, d_cand,
                                                           max_cand, staged, d_replica_id, target);
    count_launch(c);
    rc = pyg_lookup_batch_dev(c, d_tokens, d_tok_off, d_hash_off, d_hashes, R, target, 1, m3);
  }
  if (!rc) {
    k_stage_classify<<<(R + 255) / 256, 256, 0, c->stream>>>(R, d_tok_off, target, m3, d_gpu_idle,
                                                             d_out);
    count_launch(c);
    rc = cuda_check(cudaGetLastError(), "k_stage_classify");
  }
  cudaFreeAsync(buf, c->stream);
  return rc;
}
