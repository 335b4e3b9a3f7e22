// k_prompt.cu -- device prompt assembly.
//
// assemble_prompt (prompt.cpp:128-164) concatenates a template's segments: Literal
// text (tokenized words) and Refs into earlier exchanges' request / response token
// sequences.  On a B200 the exchanges live in HBM -- a response is produced on the
// GPU, a request prompt was assembled here one step earlier -- so the host only
// resolves each segment to a range of a device token pool and ships those
// descriptors (plus genuinely new tokens); the prompt tokens are gathered on device
// instead of crossing PCIe.
//
//   k_seg_lens   tokens per request (sum of its segment lengths)
//   CUB scan     tok_off
//   k_gather     one CTA per request, coalesced 8-byte copies per segment
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "ctx.cuh"

using namespace pyg_host;

namespace {

__global__ void k_seg_lens(int R, const int64_t* seg_off, const pyg_segment* segs, int64_t* lens) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > R) return;
  int64_t s = 0;
  if (r < R)
    for (int64_t k = seg_off[r]; k < seg_off[r + 1]; ++k) s += segs[k].len;
  lens[r] = s;  // lens[R] = 0 closes the exclusive scan
}

__global__ void k_gather(int R, const int64_t* seg_off, const pyg_segment* segs,
                         const uint64_t* __restrict__ pool, const int64_t* tok_off,
                         uint64_t* __restrict__ tokens) {
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    int64_t dst = tok_off[r];
    for (int64_t k = seg_off[r]; k < seg_off[r + 1]; ++k) {
      const pyg_segment sg = segs[k];
      const uint64_t* src = pool + sg.src;
      uint64_t* out = tokens + dst;
      const int64_t bd = blockDim.x;
      int64_t i = threadIdx.x;
      // up to four independent 8-byte loads in flight per thread before their stores
      for (; i < sg.len; i += 4 * bd) {
        uint64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * bd < sg.len) v[u] = __ldg(src + i + u * bd);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (i + u * bd < sg.len) out[i + u * bd] = v[u];
      }
      dst += sg.len;
    }
  }
}

}  // namespace

namespace pyg_host {
// request lengths (sum of segment lengths) and their exclusive scan -> d_tok_off[R+1]
int assemble_offsets(pyg_ctx* c, int32_t R, const int64_t* d_seg_off, const pyg_segment* d_segs,
                     int64_t* d_tok_off) {
  size_t tmp = 0;
  PYG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, static_cast<int64_t*>(nullptr), d_tok_off,
                                         R + 1, c->stream));
  const size_t lb = (static_cast<size_t>(R + 1) * 8 + 255) & ~size_t{255};
  void* sp;
  int rc = scratch(c, lb + tmp, &sp);
  if (rc) return rc;
  auto* lens = static_cast<int64_t*>(sp);
  k_seg_lens<<<(R + 1 + 255) / 256, 256, 0, c->stream>>>(R, d_seg_off, d_segs, lens);
  PYG_LAUNCHED(c);
  PYG_CUDA(cub::DeviceScan::ExclusiveSum(static_cast<char*>(sp) + lb, tmp, lens, d_tok_off, R + 1,
                                         c->stream));
  PYG_LAUNCHED(c);
  return PYG_OK;
}
}  // namespace pyg_host

extern "C" int pyg_assemble_dev(pyg_ctx* c, int32_t R, const int64_t* d_seg_off,
                                const pyg_segment* d_segs, const uint64_t* d_pool,
                                int64_t* d_tok_off, uint64_t* d_tokens) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0) return PYG_EINVAL;
  int rc = assemble_offsets(c, R, d_seg_off, d_segs, d_tok_off);
  if (rc) return rc;
  if (R) {
    const int n_sm = pyg_host::sm_count(c->device);
    k_gather<<<std::min(R, 8 * n_sm), 256, 0, c->stream>>>(R, d_seg_off, d_segs, d_pool, d_tok_off,
                                                           d_tokens);
    PYG_LAUNCHED(c);
  }
  return PYG_OK;
}
