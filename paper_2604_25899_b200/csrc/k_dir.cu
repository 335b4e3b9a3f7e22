// k_dir.cu -- K2: the staged matrix through the L2 directory (dir.cuh).
//
//   k_dir_export   alive L2 blocks of this ctx -> DirRecord list (a shard's share)
//   k_dir_build    DirRecords of every shard -> main / rver / rlen tables
//   k_group_pos    candidate groups -> replica bitmask + replica -> column map
//   k_staged_dir   one thread per request (one warp per request for walks of
//                  >= 128 boundaries): ONE walk of its boundary hashes
//                  yields matched_prefix on the L2 of every candidate replica
//                  (node_view, engine.cpp:640-648; TierStore::matched_prefix,
//                  hierarchy.cpp:84-104)
//
// Cost per request is (deepest candidate match + 1) directory probes, whatever
// the number of candidates, so the staged matrix of a 1024-replica cluster
// costs what a 1-replica one does.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

namespace {

__global__ void k_dir_export(CtxDev c, int n_rep, DirRecord* out, int64_t cap,
                             unsigned long long* count) {
  const int rep = blockIdx.y;
  const TierDev& t = c.tiers[2 * rep + 1];
  const int grep = c.rep_base + rep;
  if (blockIdx.x == 0 && threadIdx.x == 0 && t.n_long_orphans > 0) {
    const unsigned long long k = atomicAdd(count, 1ULL);
    if (static_cast<int64_t>(k) < cap) out[k] = DirRecord{0, 0, 0, 0, grep, kDirLongOrphan};
  }
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < t.log_len;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const Block& b = t.log[i];
    if (!(b.flags & kAlive)) continue;
    const unsigned long long k = atomicAdd(count, 1ULL);
    if (static_cast<int64_t>(k) < cap)
      out[k] = DirRecord{b.hash, b.parent, b.s, b.e, grep, b.flags & kOrphan};
  }
}

__global__ void k_dir_build(DirDev d, int B, const DirRecord* rec, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const DirRecord r = rec[i];
  if (r.replica < 0 || r.replica >= d.n_global) return;
  if (r.flags & kDirLongOrphan) {
    atomicOr(reinterpret_cast<unsigned long long*>(d.long_mask + (r.replica >> 6)),
             1ULL << (r.replica & 63));
    return;
  }
  dir_set_bit(d.main, d.main_mask, d.stride, dir_key(r.hash), r.replica);
  if (r.s % B != 0 || r.e % B == 0 || r.e <= r.s) return;
  const int64_t len = r.e - r.s;
  if ((r.flags & kOrphan) && len >= 64) return;  // long orphan: literal scan (long_mask)
  dir_set_bit(d.rver, d.rver_mask, d.stride, rver_key(r.hash, r.s, r.e), r.replica);
  const uint64_t key = dir_key((r.flags & kOrphan) ? orphan_key(r.s) : r.parent);
  const uint64_t sl = dir_slot_insert(d.rlen, d.rlen_mask, 2, key);
  atomicOr(reinterpret_cast<unsigned long long*>(d.rlen + 2 * sl + 1), 1ULL << len);
}

// gmask[g][W] = candidate replicas of group g; pos[g * n_global + rep] = column
__global__ void k_group_pos(int G, const int32_t* cand_off, const int32_t* cand, int n_global,
                            int W, uint64_t* gmask, int32_t* pos, int32_t* err) {
  const int g = blockIdx.x;
  if (g >= G) return;
  for (int w = threadIdx.x; w < W; w += blockDim.x) gmask[static_cast<int64_t>(g) * W + w] = 0;
  __syncthreads();
  const int c0 = cand_off[g], nc = cand_off[g + 1] - c0;
  for (int j = threadIdx.x; j < nc; j += blockDim.x) {
    const int n = cand[c0 + j];
    if (n < 0 || n >= n_global) {
      atomicExch(err, 2);
      continue;
    }
    const unsigned long long old =
        atomicOr(reinterpret_cast<unsigned long long*>(gmask + static_cast<int64_t>(g) * W + (n >> 6)),
                 1ULL << (n & 63));
    if (old & (1ULL << (n & 63))) atomicExch(err, 2);  // duplicate candidate
    pos[static_cast<int64_t>(g) * n_global + n] = j;
  }
}

template <int W>
__device__ __forceinline__ void load_mask(const uint64_t* p, uint64_t (&m)[W]) {
  if constexpr (W == 1) {
    m[0] = p[0];
  } else {
#pragma unroll
    for (int w = 0; w < W; ++w) m[w] = p[w];
  }
}

struct StagedDirArgs {
  CtxDev c;
  DirDev d;
  const uint64_t* tokens;
  const int64_t* tok_off;
  const int64_t* hash_off;
  const uint64_t* hashes;
  int R;
  const int32_t* group;
  const int32_t* cand_off;
  const uint64_t* gmask;
  const int32_t* pos;
  int max_cand;
  int32_t* staged;
};

// Ragged extension (hierarchy.cpp:92-103) for the candidates whose aligned walk
// ended at m = d*B: rows of `drop` replicas get m, or m + o for the largest
// verified ragged block of length o.
template <int W>
__device__ __forceinline__ void emit_drop(const StagedDirArgs& A, int64_t m, int64_t L, const uint64_t* tok,
                          const uint64_t* hs, const uint64_t (&drop)[W], const uint64_t* pos_g,
                          const int32_t* posrow, int32_t* row) {
  // default: the aligned match
#pragma unroll
  for (int w = 0; w < W; ++w) {
    uint64_t b = drop[w];
    while (b) {
      const int k = __ffsll(static_cast<long long>(b)) - 1;
      b &= b - 1;
      row[posrow[w * 64 + k]] = static_cast<int32_t>(m);
    }
  }
  if (m >= L) return;
  const uint64_t parent = m == 0 ? kFnvOffset : hs[m / A.c.B - 1];
  uint64_t lens = 0;
  int64_t s1 = dir_slot_find(A.d.rlen, A.d.rlen_mask, 2, dir_key(parent));
  if (s1 >= 0) lens |= A.d.rlen[2 * s1 + 1];
  int64_t s2 = dir_slot_find(A.d.rlen, A.d.rlen_mask, 2, dir_key(orphan_key(m)));
  if (s2 >= 0) lens |= A.d.rlen[2 * s2 + 1];
  lens &= ~1ULL;
  if (lens) {
    uint64_t h = parent;
    const int64_t lim = L - m < 63 ? L - m : 63;
    for (int64_t o = 1; o <= lim; ++o) {
      h = fnv_token(h, tok[m + o - 1]);
      if (((lens >> o) & 1ULL) && (m + o) % A.c.B != 0) {
        const int64_t sl = dir_slot_find(A.d.rver, A.d.rver_mask, A.d.stride, rver_key(h, m, m + o));
        if (sl >= 0) {
          const uint64_t* mk = A.d.rver + sl * A.d.stride + 1;
#pragma unroll
          for (int w = 0; w < W; ++w) {
            uint64_t b = drop[w] & mk[w];
            while (b) {
              const int k = __ffsll(static_cast<long long>(b)) - 1;
              b &= b - 1;
              row[posrow[w * 64 + k]] = static_cast<int32_t>(m + o);
            }
          }
        }
      }
      if ((lens >> o) <= 1ULL) break;
    }
  }
  // replicas holding orphans longer than 63 tokens: the literal check on the tier itself
#pragma unroll
  for (int w = 0; w < W; ++w) {
    uint64_t b = drop[w] & A.d.long_mask[w];
    while (b) {
      const int k = __ffsll(static_cast<long long>(b)) - 1;
      b &= b - 1;
      const int local = w * 64 + k - A.c.rep_base;
      if (local < 0 || local >= A.c.n_rep) {
        atomicExch(A.c.error, 3);  // a remote shard's long orphan cannot be scanned here
        continue;
      }
      const TierDev& t = A.c.tiers[2 * local + 1];
      row[posrow[w * 64 + k]] = static_cast<int32_t>(ragged_extend(t, t.log, tok, L, hs, m, A.c.B));
    }
  }
  (void)pos_g;
}

// Long walks (>= min_nh boundary hashes): one warp per request.  The probes of a
// walk are independent loads, so lane l probes boundary d0 + l and the warp
// prefix-ANDs the presence masks: replica n drops at the first boundary it
// misses, exactly where the per-thread walk below would drop it, and every
// lane emits the drops (aligned match + ragged extension) of its own boundary.
// One probe latency per 32 boundaries instead of one per boundary.
template <int W>
__device__ __forceinline__ void staged_walk_warp(const StagedDirArgs& A, int r) {
  const int lane = threadIdx.x & 31;
  const int g = A.group[r];
  const int nc = A.cand_off[g + 1] - A.cand_off[g];
  int32_t* row = A.staged + static_cast<int64_t>(r) * A.max_cand;
  for (int j = nc + lane; j < A.max_cand; j += 32) row[j] = 0;
  uint64_t alive[W];
  load_mask<W>(A.gmask + static_cast<int64_t>(g) * W, alive);
  const int32_t* posrow = A.pos + static_cast<int64_t>(g) * A.d.n_global;
  const int64_t L = A.tok_off[r + 1] - A.tok_off[r];
  const uint64_t* tok = A.tokens + A.tok_off[r];
  const uint64_t* hs = A.hashes + A.hash_off[r];
  const int64_t nh = A.hash_off[r + 1] - A.hash_off[r];
  const int B = A.c.B;
  for (int64_t d0 = 0; d0 < nh; d0 += 32) {
    uint64_t any_alive = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) any_alive |= alive[w];
    if (!any_alive) break;  // warp-uniform: every lane holds the same alive mask
    const int64_t d = d0 + lane;
    // slot of this lane's boundary; -1 = absent (present nowhere), -2 = past the
    // last boundary (nobody drops there)
    const int64_t sl =
        d < nh ? dir_slot_find(A.d.main, A.d.main_mask, A.d.stride, dir_key(hs[d])) : -2;
    const uint64_t* pm = A.d.main + (sl >= 0 ? sl : 0) * A.d.stride + 1;
    uint64_t drop[W];
    bool any_drop = false;
#pragma unroll
    for (int w = 0; w < W; ++w) {  // one mask word at a time keeps W = 16 in registers
      uint64_t acc = sl >= 0 ? pm[w] : (sl == -1 ? 0ULL : ~0ULL);
      uint64_t dr = alive[w] & ~acc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {  // inclusive prefix-AND over the lanes
        const uint64_t v = __shfl_up_sync(0xffffffffu, acc, off);
        if (lane >= off) acc &= v;
      }
      const uint64_t before = __shfl_up_sync(0xffffffffu, acc, 1);
      if (lane > 0) dr &= before;
      drop[w] = dr;
      any_drop |= dr != 0;
      alive[w] &= __shfl_sync(0xffffffffu, acc, 31);
    }
    if (any_drop) emit_drop<W>(A, d * B, L, tok, hs, drop, nullptr, posrow, row);
  }
  // still matching after the last boundary: matched = L (lane w takes mask word w)
  for (int w = lane; w < W; w += 32) {
    uint64_t b = 0;
#pragma unroll
    for (int x = 0; x < W; ++x)
      if (x == w) b = alive[x];
    while (b) {
      const int k = __ffsll(static_cast<long long>(b)) - 1;
      b &= b - 1;
      row[posrow[w * 64 + k]] = static_cast<int32_t>(L);
    }
  }
}

// Blocks [0, warp_blocks) take the long walks (launched first: they are the
// kernel's tail): warp k finds the long requests among requests [32k, 32k+32)
// by ballot and walks them one after the other; the rest of the grid walks the
// short ones one thread per request.
template <int W>
__global__ void __launch_bounds__(128, W >= 8 ? 4 : 6) k_staged_dir(StagedDirArgs A, int min_nh, int warp_blocks) {
  if (static_cast<int>(blockIdx.x) < warp_blocks) {
    const int r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32;
    if (r0 >= A.R) return;
    const int me = r0 + (threadIdx.x & 31);
    const bool is_long = me < A.R && A.hash_off[me + 1] - A.hash_off[me] >= min_nh;
    unsigned todo = __ballot_sync(0xffffffffu, is_long);
    while (todo) {
      const int k = __ffs(todo) - 1;
      todo &= todo - 1;
      staged_walk_warp<W>(A, r0 + k);
    }
    return;
  }
  const int r = (blockIdx.x - warp_blocks) * blockDim.x + threadIdx.x;
  if (r >= A.R) return;
  if (A.hash_off[r + 1] - A.hash_off[r] >= min_nh) return;  // a warp walks it
  const int g = A.group[r];
  const int nc = A.cand_off[g + 1] - A.cand_off[g];
  int32_t* row = A.staged + static_cast<int64_t>(r) * A.max_cand;
  for (int j = nc; j < A.max_cand; ++j) row[j] = 0;
  uint64_t alive[W];
  load_mask<W>(A.gmask + static_cast<int64_t>(g) * W, alive);
  const int32_t* posrow = A.pos + static_cast<int64_t>(g) * A.d.n_global;
  const int64_t L = A.tok_off[r + 1] - A.tok_off[r];
  const uint64_t* tok = A.tokens + A.tok_off[r];
  const uint64_t* hs = A.hashes + A.hash_off[r];
  const int64_t nh = A.hash_off[r + 1] - A.hash_off[r];
  const int B = A.c.B;
  auto any = [&](const uint64_t (&m)[W]) {
    uint64_t x = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) x |= m[w];
    return x != 0;
  };
  // probe d+1 is issued before d is consumed (two independent loads in flight)
  int64_t d = 0;
  int64_t nxt = nh > 0 ? dir_slot_find(A.d.main, A.d.main_mask, A.d.stride, dir_key(hs[0])) : -1;
  while (d < nh && any(alive)) {
    const int64_t cur = nxt;
    nxt = d + 1 < nh ? dir_slot_find(A.d.main, A.d.main_mask, A.d.stride, dir_key(hs[d + 1])) : -1;
    uint64_t pres[W], drop[W];
    if (cur >= 0) {
      load_mask<W>(A.d.main + cur * A.d.stride + 1, pres);
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) pres[w] = 0;
    }
#pragma unroll
    for (int w = 0; w < W; ++w) {
      drop[w] = alive[w] & ~pres[w];
      alive[w] &= pres[w];
    }
    if (any(drop)) emit_drop<W>(A, d * B, L, tok, hs, drop, nullptr, posrow, row);
    ++d;
  }
  // still matching after the last boundary: matched = min(nh*B, L) = L, no ragged check
#pragma unroll
  for (int w = 0; w < W; ++w) {
    uint64_t b = alive[w];
    while (b) {
      const int k = __ffsll(static_cast<long long>(b)) - 1;
      b &= b - 1;
      row[posrow[w * 64 + k]] = static_cast<int32_t>(L);
    }
  }
}

size_t al256(size_t x) { return (x + 255) & ~size_t{255}; }

uint64_t pow2_at_least(uint64_t x) {
  uint64_t p = 1024;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace

// ------------------------------------------------------------------ host side
namespace pyg_host {

// (Re)allocates and clears the directory tables for n records.
static int dir_alloc(pyg_ctx* c, int64_t n) {
  const int ng = c->sharded ? c->n_global : c->n_rep;
  int W = 1;
  while (W * 64 < ng) W *= 2;  // 1, 2, 4, 8, 16 (the kernel templates)
  if (W > kDirMaxWords) {
    set_error("the L2 directory supports at most 1024 replicas");
    return PYG_ENOTSUP;
  }
  const int stride = (1 + W + 1) & ~1;
  const uint64_t cap = pow2_at_least(static_cast<uint64_t>(2 * std::max<int64_t>(n, 1)));
  const size_t b_main = al256(cap * stride * 8), b_rver = b_main, b_rlen = al256(cap * 16),
               b_long = al256(W * 8);
  const size_t total = b_main + b_rver + b_rlen + b_long;
  if (total > c->dir_mem_size) {
    if (c->dir_mem) {
      PYG_CUDA(cudaStreamSynchronize(c->stream));
      PYG_CUDA(cudaFree(c->dir_mem));
      c->dir_mem = nullptr;
    }
    PYG_CUDA(cudaMalloc(&c->dir_mem, total));
    c->dir_mem_size = total;
  }
  PYG_CUDA(cudaMemsetAsync(c->dir_mem, 0, total, c->stream));
  char* p = static_cast<char*>(c->dir_mem);
  DirDev& d = c->dir;
  d.main = reinterpret_cast<uint64_t*>(p);
  d.rver = reinterpret_cast<uint64_t*>(p + b_main);
  d.rlen = reinterpret_cast<uint64_t*>(p + b_main + b_rver);
  d.long_mask = reinterpret_cast<uint64_t*>(p + b_main + b_rver + b_rlen);
  d.main_mask = d.rver_mask = d.rlen_mask = cap - 1;
  d.W = W;
  d.stride = stride;
  d.n_global = ng;
  d.rep_base = c->rep_base;
  c->hd.dir_main = d.main;
  c->hd.dir_rver = d.rver;
  c->hd.dir_main_mask = d.main_mask;
  c->hd.dir_rver_mask = d.rver_mask;
  c->hd.dir_stride = stride;
  c->hd.rep_base = c->rep_base;
  return PYG_OK;
}

static int64_t export_cap(pyg_ctx* c) {
  int64_t cap = 1;
  for (int r = 0; r < c->n_rep; ++r) cap += c->tiers[2 * r + 1].d.log_cap + 1;
  return cap;
}

static int dir_export(pyg_ctx* c, DirRecord* out, int64_t cap, unsigned long long* d_count) {
  PYG_CUDA(cudaMemsetAsync(d_count, 0, 8, c->stream));
  if (c->n_rep) {
    dim3 grid(16, c->n_rep);
    k_dir_export<<<grid, 256, 0, c->stream>>>(c->hd, c->n_rep, out, cap, d_count);
    PYG_LAUNCHED(c);
  }
  return PYG_OK;
}

static int dir_build(pyg_ctx* c, const DirRecord* rec, int64_t n) {
  int rc = dir_alloc(c, n);
  if (rc) return rc;
  if (n) {
    k_dir_build<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c->stream>>>(c->dir, c->B, rec, n);
    PYG_LAUNCHED(c);
  }
  c->dir_dirty = false;
  c->dir_admits = 0;
  return PYG_OK;
}

// Single-GPU ctx: rebuild the directory from its own L2 tiers when stale.
int ensure_dir(pyg_ctx* c) {
  if (!c->dir_dirty && c->dir.main && c->dir_admits < 256) return PYG_OK;
  if (c->sharded) {
    if (c->dir.main && !c->dir_dirty) return PYG_OK;  // admissions clear bits in place
    set_error("L2 directory is stale on a sharded ctx: rebuild it with the records of every "
              "shard (pyg_dir_export_dev + pyg_dir_build_dev)");
    return PYG_EINVAL;
  }
  const int64_t cap = export_cap(c);
  void* buf = nullptr;
  PYG_CUDA(cudaMallocAsync(&buf, cap * sizeof(DirRecord) + 256, c->stream));
  auto* rec = static_cast<DirRecord*>(buf);
  auto* cnt = reinterpret_cast<unsigned long long*>(static_cast<char*>(buf) + cap * sizeof(DirRecord));
  int rc = dir_export(c, rec, cap, cnt);
  unsigned long long n = 0;
  if (!rc) rc = cuda_check(cudaMemcpyAsync(&n, cnt, 8, cudaMemcpyDeviceToHost, c->stream), "copy");
  if (!rc) rc = cuda_check(cudaStreamSynchronize(c->stream), "sync");
  if (!rc) rc = dir_build(c, rec, static_cast<int64_t>(std::min<unsigned long long>(n, cap)));
  cudaFreeAsync(buf, c->stream);
  return rc;
}

}  // namespace pyg_host

extern "C" {

int pyg_set_shard(pyg_ctx* c, int32_t rep_base, int32_t n_global) {
  PYG_ON_DEVICE(c);
  if (!c || rep_base < 0 || n_global < rep_base + c->n_rep || n_global > 64 * kDirMaxWords) {
    set_error("pyg_set_shard: need 0 <= rep_base, rep_base + n_replicas <= n_global <= 1024");
    return PYG_EINVAL;
  }
  if (c->sharded && c->rep_base == rep_base && c->n_global == n_global) return PYG_OK;
  c->sharded = true;
  c->rep_base = rep_base;
  c->n_global = n_global;
  c->hd.rep_base = rep_base;
  c->dir_dirty = true;  // the directory must now cover the whole cluster
  return PYG_OK;
}

int pyg_dir_export_dev(pyg_ctx* c, void* d_records, int64_t cap, int64_t* n_out) {
  PYG_ON_DEVICE(c);
  if (!c || cap < 0 || (cap && !d_records) || !n_out) return PYG_EINVAL;
  void* sp;
  int rc = scratch(c, 64, &sp);
  if (rc) return rc;
  auto* cnt = static_cast<unsigned long long*>(sp);
  if ((rc = dir_export(c, static_cast<DirRecord*>(d_records), cap, cnt))) return rc;
  unsigned long long n = 0;
  PYG_CUDA(cudaMemcpyAsync(&n, cnt, 8, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  *n_out = static_cast<int64_t>(n);
  if (static_cast<int64_t>(n) > cap) {
    set_error("pyg_dir_export_dev: record buffer too small (see *n_out)");
    return PYG_ECAPACITY;
  }
  return PYG_OK;
}

int64_t pyg_dir_export_cap(pyg_ctx* c) { return c ? export_cap(c) : 0; }

int pyg_dir_build_dev(pyg_ctx* c, const void* d_records, int64_t n) {
  PYG_ON_DEVICE(c);
  if (!c || n < 0 || (n && !d_records)) return PYG_EINVAL;
  return dir_build(c, static_cast<const DirRecord*>(d_records), n);
}

// K2 (staged matrix) through the directory.  Candidates are global replica indices.
int pyg_staged_matrix_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                                 const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t R,
                                 const int32_t* d_group, int32_t n_groups,
                                 const int32_t* d_cand_off, const int32_t* d_cand,
                                 int32_t max_cand, int32_t* d_staged) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0 || max_cand < 0) return PYG_EINVAL;
  if (R == 0 || max_cand == 0) return PYG_OK;
  int rc = ensure_dir(c);
  if (rc) return rc;
  const int G = n_groups;
  if (G < 0) return PYG_EINVAL;
  const DirDev& d = c->dir;
  const size_t b_gm = al256(static_cast<size_t>(std::max(G, 1)) * d.W * 8);
  const size_t b_pos = al256(static_cast<size_t>(std::max(G, 1)) * d.n_global * 4);
  void* sp;
  if ((rc = scratch(c, b_gm + b_pos, &sp))) return rc;
  auto* gmask = static_cast<uint64_t*>(sp);
  auto* pos = reinterpret_cast<int32_t*>(static_cast<char*>(sp) + b_gm);
  if (G) {
    k_group_pos<<<G, 128, 0, c->stream>>>(G, d_cand_off, d_cand, d.n_global, d.W, gmask, pos,
                                          c->hd.error);
    PYG_LAUNCHED(c);
  }
  StagedDirArgs a{c->hd, d, d_tokens, d_tok_off, d_hash_off, d_hashes, R, d_group,
                  d_cand_off, gmask, pos, max_cand, d_staged};
  // walks of >= min_nh boundaries go to a warp each (PYG_K2_WARP_MIN overrides;
  // a huge value keeps every walk on one thread)
  int min_nh = 128;
  if (const char* e = getenv("PYG_K2_WARP_MIN")) min_nh = std::max(0, atoi(e));
  const int warp_blocks = min_nh >= (1 << 30) ? 0 : (R + 127) / 128;
  const unsigned grid = warp_blocks + (R + 127) / 128;
  switch (d.W) {
    case 1: k_staged_dir<1><<<grid, 128, 0, c->stream>>>(a, min_nh, warp_blocks); break;
    case 2: k_staged_dir<2><<<grid, 128, 0, c->stream>>>(a, min_nh, warp_blocks); break;
    case 4: k_staged_dir<4><<<grid, 128, 0, c->stream>>>(a, min_nh, warp_blocks); break;
    case 8: k_staged_dir<8><<<grid, 128, 0, c->stream>>>(a, min_nh, warp_blocks); break;
    default: k_staged_dir<16><<<grid, 128, 0, c->stream>>>(a, min_nh, warp_blocks); break;
  }
  PYG_LAUNCHED(c);
  return PYG_OK;
}

}  // extern "C"
