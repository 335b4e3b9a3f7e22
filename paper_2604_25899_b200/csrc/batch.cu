// batch.cu -- batched, device-resident hot path:
//   K1 k_hash_batch       chain_boundary_hashes for every request
//   K2 k_staged / lookup  TierStore::matched_prefix per (request, replica)
//   K3 k_route_*          sched::route, snapshot or sequential-commit
//   K4+K5 k_admit         start_prefill cache side: lookup, evict, promote, insert
//   K5 k_release          unpin_chain of admitted requests
// Every kernel restates the reference function named in its comment.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

namespace {

// ------------------------------------------------------------------- K1
// One lane per request; 16-byte read-only loads, software-pipelined 8 tokens
// ahead so each lane keeps 64 B in flight (hashing is a serial FNV chain per
// request; parallelism comes from requests).
__global__ void __launch_bounds__(256) k_hash_batch(const uint64_t* __restrict__ tokens,
                                                    const int64_t* __restrict__ tok_off, int R,
                                                    const int64_t* __restrict__ hash_off,
                                                    uint64_t* __restrict__ hashes, int B) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int64_t s = tok_off[r];
  const int64_t n = tok_off[r + 1] - s;
  uint64_t* out = hashes + hash_off[r];
  const uint64_t* p = tokens + s;
  uint64_t h = kFnvOffset;
  int cd = B;
  int64_t k = 0, i = 0;
  if ((s & 1) && n > 0) {  // 16-byte alignment of the vector loads
    h = fnv_token(h, __ldg(p));
    if (--cd == 0) {
      out[k++] = h;
      cd = B;
    }
    i = 1;
  }
  const ulonglong2* v = reinterpret_cast<const ulonglong2*>(p + i);
  const int64_t nv = (n - i) / 8;  // groups of 8 tokens
  ulonglong2 a0, a1, a2, a3;
  if (nv > 0) {
    a0 = __ldg(v);
    a1 = __ldg(v + 1);
    a2 = __ldg(v + 2);
    a3 = __ldg(v + 3);
  }
  for (int64_t g = 0; g < nv; ++g) {
    const uint64_t t[8] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y, a3.x, a3.y};
    if (g + 1 < nv) {
      const ulonglong2* q = v + 4 * (g + 1);
      a0 = __ldg(q);
      a1 = __ldg(q + 1);
      a2 = __ldg(q + 2);
      a3 = __ldg(q + 3);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      h = fnv_token(h, t[j]);
      if (--cd == 0) {
        out[k++] = h;
        cd = B;
      }
    }
  }
  for (int64_t x = i + nv * 8; x < n; ++x) {
    h = fnv_token(h, __ldg(p + x));
    if (--cd == 0) {
      out[k++] = h;
      cd = B;
    }
  }
  if (n > 0 && cd != B) out[k] = h;  // the ragged last block (hierarchy.cpp:26)
}

__global__ void k_nblocks(const int64_t* tok_off, int R, int B, int64_t* nb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) nb[r] = (tok_off[r + 1] - tok_off[r] + B - 1) / B;
  if (r == R) nb[R] = 0;
}

// ------------------------------------------------------------------- K2
// staged[r][j] = tier(L2 of candidate j).matched_prefix(prompt_r)
// (node_view: rep.cache.lookup(r.prompt, nullptr).l2, engine.cpp:646).
// One thread per (request, candidate).
__global__ void k_staged(CtxDev c, const uint64_t* __restrict__ tokens,
                         const int64_t* __restrict__ tok_off, const int64_t* __restrict__ hash_off,
                         const uint64_t* __restrict__ hashes, int R, const int32_t* group,
                         const int32_t* cand_off, const int32_t* cand, int max_cand,
                         int32_t* staged) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= static_cast<int64_t>(R) * max_cand) return;
  const int r = static_cast<int>(x / max_cand);
  const int j = static_cast<int>(x % max_cand);
  const int g = group[r];
  const int nc = cand_off[g + 1] - cand_off[g];
  if (j >= nc) {
    staged[x] = 0;
    return;
  }
  const int rep = cand[cand_off[g] + j];
  const TierDev& t = c.tiers[2 * rep + 1];
  const int64_t L = tok_off[r + 1] - tok_off[r];
  const uint64_t* hs = hashes + hash_off[r];
  const int64_t nh = hash_off[r + 1] - hash_off[r];
  const int64_t kb = thread_walk(t, hs, nh);
  const int64_t m = kb ? matched_from_blocks(kb, L, c.B) : 0;
  staged[x] = static_cast<int32_t>(ragged_extend(t, t.log, tokens + tok_off[r], L, hs, m, c.B));
}

// CacheHierarchy::lookup (hierarchy.cpp:109-117) of request r on replica rep[r].
__global__ void k_lookup_batch(CtxDev c, const uint64_t* __restrict__ tokens,
                               const int64_t* __restrict__ tok_off,
                               const int64_t* __restrict__ hash_off,
                               const uint64_t* __restrict__ hashes, int R, const int32_t* rep,
                               int with_l3, int64_t* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int rp = rep[r];
  if (rp < 0) {
    out[3 * r] = out[3 * r + 1] = out[3 * r + 2] = 0;
    return;
  }
  const int64_t L = tok_off[r + 1] - tok_off[r];
  const uint64_t* hs = hashes + hash_off[r];
  const int64_t nh = hash_off[r + 1] - hash_off[r];
  for (int k = 0; k < 3; ++k) {
    if (k == 2 && !with_l3) {
      out[3 * r + 2] = 0;
      break;
    }
    const TierDev& t = c.tiers[k < 2 ? 2 * rp + k : 2 * c.n_rep];
    const int64_t kb = thread_walk(t, hs, nh);
    const int64_t m = kb ? matched_from_blocks(kb, L, c.B) : 0;
    out[3 * r + k] = ragged_extend(t, t.log, tokens + tok_off[r], L, hs, m, c.B);
  }
}

// ------------------------------------------------------------------- K3
struct NodeScratch {
  int64_t* free_;    // kv_capacity - sum of assigned tokens()
  double* b0;        // oom_bound(node, alpha=+0.0): 0.0 + a_1 + ... (router.cpp:13-17)
  double* ba;        // oom_bound(node, alpha=a*)
  int32_t* head;     // appended placements (seq-commit): linked list of alphas
  int32_t* tail;
  double* app_alpha; // [R]
  int32_t* app_next; // [R]
};

// Per replica: capacity_holds / oom_bound aggregates over the assigned set.
__global__ void k_node_prep(int n, const pyg_nodes_dev nodes, NodeScratch ns) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t sum = 0;
  double b = 0.0;
  for (int64_t k = nodes.asg_off[i]; k < nodes.asg_off[i + 1]; ++k) {
    const pyg_reservation& a = nodes.asg[k];
    sum += res_tokens(a.prompt_len, a.upper, a.tokens_generated);
    b += a.alpha;
  }
  ns.free_[i] = nodes.kv_capacity[i] - sum;
  ns.b0[i] = b;
  ns.head[i] = -1;
  ns.tail[i] = -1;
}

__device__ __forceinline__ bool same_bits(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}

// oom_bound(node i, alpha): alpha + assigned alphas in order + appended placements.
__device__ __forceinline__ double node_bound(const pyg_nodes_dev& nodes, const NodeScratch& ns,
                                             int i, double alpha, bool have_star, double astar) {
  if (same_bits(alpha, 0.0)) return ns.b0[i];
  if (have_star && same_bits(alpha, astar)) return ns.ba[i];
  double b = alpha;
  for (int64_t k = nodes.asg_off[i]; k < nodes.asg_off[i + 1]; ++k) b += nodes.asg[k].alpha;
  for (int32_t q = ns.head[i]; q >= 0; q = ns.app_next[q]) b += ns.app_alpha[q];
  return b;
}

struct RouteCtx {
  pyg_nodes_dev nodes;
  NodeScratch ns;
  const int32_t* cand_off;
  const int32_t* cand;
  int max_cand;
  const int32_t* staged;
  double eps;
};

// sched::route (router.cpp:19-50) of one request over its group's candidates,
// one warp (lanes over candidates).  Returns the decision and the winner's
// candidate slot (-1 = wait).
__device__ pyg_decision warp_route(const RouteCtx& rc, int r, int g, const pyg_reservation& q,
                                   bool have_star, double astar, int* win_slot) {
  const int lane = threadIdx.x & 31;
  const int64_t t = res_tokens(q.prompt_len, q.upper, q.tokens_generated);
  const int c0 = rc.cand_off[g], nc = rc.cand_off[g + 1] - c0;
  RouteAcc best{0, 0, 0, -1};
  for (int j = lane; j < nc; j += 32) {
    const int n = rc.cand[c0 + j];
    const int64_t fr = rc.ns.free_[n];
    if (t > fr) continue;  // capacity_holds (router.cpp:7-11)
    const double b = node_bound(rc.nodes, rc.ns, n, q.alpha, have_star, astar);
    if (b > rc.eps) continue;
    RouteAcc a{fr - t, rc.staged[static_cast<int64_t>(r) * rc.max_cand + j],
               rc.nodes.replica_id[n], j};
    if (acc_better(a, best)) best = a;
  }
  best = warp_best(best);
  int32_t p1 = 0x7fffffff, p2 = 0x7fffffff;
  if (best.pos >= 0) {
    for (int j = lane; j < nc; j += 32) {
      const int n = rc.cand[c0 + j];
      const int64_t fr = rc.ns.free_[n];
      if (t > fr || fr - t != best.h) continue;
      const double b = node_bound(rc.nodes, rc.ns, n, q.alpha, have_star, astar);
      if (b > rc.eps) continue;
      p1 = min(p1, j);
      if (rc.staged[static_cast<int64_t>(r) * rc.max_cand + j] == best.s) p2 = min(p2, j);
    }
  }
  p1 = warp_min_i32(p1);
  p2 = warp_min_i32(p2);
  pyg_decision d{-1, 0, 0, 0.0};
  *win_slot = best.pos;
  if (best.pos >= 0) {
    const int n = rc.cand[c0 + best.pos];
    d.target = best.id;
    d.headroom = best.h;
    d.oom_bound = node_bound(rc.nodes, rc.ns, n, q.alpha, have_star, astar);
    d.tiebreak = p1 < p2 ? 1 : 0;
  }
  return d;
}

// SNAPSHOT: every request against the same node state; one warp per request.
__global__ void k_route_snapshot(RouteCtx rc, const pyg_reservation* req, const int32_t* group,
                                 int R, pyg_decision* out, int32_t* t_idx) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= R) return;
  const int g = group[r];
  int slot;
  const pyg_decision d = warp_route(rc, r, g, req[r], false, 0.0, &slot);
  if ((threadIdx.x & 31) == 0) {
    out[r] = d;
    t_idx[r] = slot >= 0 ? rc.cand[rc.cand_off[g] + slot] : -1;
  }
}

// SEQ_COMMIT (engine.cpp:650-692): the group's requests in order; a placement
// is appended to its node before the next request is routed.  One warp per
// group.  Requests that provably cannot be placed (t > the largest free
// capacity among nodes whose bound admits their alpha) wait without a full
// evaluation -- the exact feasibility test for alpha in {+0.0, a*}; other
// alphas always take the full evaluation.
__global__ void k_route_seq(RouteCtx rc, const pyg_reservation* req, const int32_t* group, int R,
                            pyg_decision* out, int32_t* t_idx) {
  const int g = blockIdx.x;
  const int lane = threadIdx.x;
  const int c0 = rc.cand_off[g], nc = rc.cand_off[g + 1] - c0;
  // a* = alpha of the group's first request with alpha != +0.0
  bool have_star = false;
  double astar = 0.0;
  for (int base = 0; base < R && !have_star; base += 32) {
    const int r = base + lane;
    const bool nz = r < R && group[r] == g && !same_bits(req[r].alpha, 0.0);
    const unsigned m = __ballot_sync(kFull, nz);
    if (m) {
      const int src = __ffs(m) - 1;
      astar = __shfl_sync(kFull, r < R ? req[r].alpha : 0.0, src);
      have_star = true;
    }
  }
  if (have_star) {
    for (int j = lane; j < nc; j += 32) {
      const int n = rc.cand[c0 + j];
      double b = astar;
      for (int64_t k = rc.nodes.asg_off[n]; k < rc.nodes.asg_off[n + 1]; ++k)
        b += rc.nodes.asg[k].alpha;
      rc.ns.ba[n] = b;
    }
    __syncwarp();
  }
  // F0 / Fa: max free over candidates whose bound admits alpha = +0.0 / a*
  auto refresh = [&](int64_t& F0, int64_t& Fa) {
    int64_t f0 = INT64_MIN, fa = INT64_MIN;
    for (int j = lane; j < nc; j += 32) {
      const int n = rc.cand[c0 + j];
      const int64_t fr = rc.ns.free_[n];
      if (!(rc.ns.b0[n] > rc.eps)) f0 = max(f0, fr);
      if (have_star && !(rc.ns.ba[n] > rc.eps)) fa = max(fa, fr);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      f0 = max(f0, __shfl_xor_sync(kFull, f0, o));
      fa = max(fa, __shfl_xor_sync(kFull, fa, o));
    }
    F0 = f0;
    Fa = fa;
  };
  int64_t F0, Fa;
  refresh(F0, Fa);
  int32_t napp = 0;  // appended placements of this group live at app index (g, ...) -> use r
  for (int base = 0; base < R; base += 32) {
    const int r = base + lane;
    const bool mine = r < R && group[r] == g;
    pyg_reservation q{0, 0, 0.0, 0};
    if (mine) q = req[r];
    const int64_t t = res_tokens(q.prompt_len, q.upper, q.tokens_generated);
    const bool z = same_bits(q.alpha, 0.0);
    const bool s = have_star && same_bits(q.alpha, astar);
    unsigned todo = __ballot_sync(kFull, mine);
    while (todo) {
      // candidates that could still be placed under the current state
      const bool could = ((todo >> lane) & 1u) && ((z && t <= F0) || (s && t <= Fa) || (!z && !s));
      const unsigned cm = __ballot_sync(kFull, could);
      // lanes before the first candidate wait
      const unsigned first = cm ? (1u << (__ffs(cm) - 1)) : 0u;
      const unsigned waiting = cm ? (todo & (first - 1)) : todo;
      if ((waiting >> lane) & 1u) {
        out[r] = pyg_decision{-1, 0, 0, 0.0};
        t_idx[r] = -1;
      }
      todo &= ~waiting;
      if (!cm) break;
      const int jl = __ffs(cm) - 1;
      const int rr = base + jl;
      pyg_reservation qq;
      qq.prompt_len = __shfl_sync(kFull, q.prompt_len, jl);
      qq.upper = __shfl_sync(kFull, q.upper, jl);
      qq.alpha = __shfl_sync(kFull, q.alpha, jl);
      qq.tokens_generated = __shfl_sync(kFull, q.tokens_generated, jl);
      int slot;
      const pyg_decision d = warp_route(rc, rr, g, qq, have_star, astar, &slot);
      if (lane == 0) {
        out[rr] = d;
        t_idx[rr] = slot >= 0 ? rc.cand[c0 + slot] : -1;
      }
      if (slot >= 0) {
        const int n = rc.cand[c0 + slot];
        if (lane == 0) {
          const int64_t tt = res_tokens(qq.prompt_len, qq.upper, qq.tokens_generated);
          rc.ns.free_[n] -= tt;
          rc.ns.b0[n] += qq.alpha;  // oom_bound appends this alpha last (router.cpp:15)
          rc.ns.ba[n] += qq.alpha;
          rc.ns.app_alpha[rr] = qq.alpha;
          rc.ns.app_next[rr] = -1;
          if (rc.ns.tail[n] >= 0)
            rc.ns.app_next[rc.ns.tail[n]] = rr;
          else
            rc.ns.head[n] = rr;
          rc.ns.tail[n] = rr;
        }
        __syncwarp();
        __threadfence_block();
        refresh(F0, Fa);
        ++napp;
      }
      todo &= ~(1u << jl);
    }
  }
}

// Stable per-replica lists of placed requests (placement order == request order).
__global__ void k_count_placed(const int32_t* t_idx, int R, int32_t* cnt) {
  __shared__ int32_t sc[32];
  const int rep = blockIdx.x;
  int32_t c = 0;
  for (int r = threadIdx.x; r < R; r += blockDim.x) c += t_idx[r] == rep;
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0) sc[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t s = 0;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) s += sc[w];
    cnt[rep] = s;
  }
}

__global__ void k_scan_placed(const int32_t* cnt, int n, int32_t* off) {
  if (threadIdx.x || blockIdx.x) return;
  int32_t s = 0;
  for (int i = 0; i < n; ++i) {
    off[i] = s;
    s += cnt[i];
  }
  off[n] = s;
}

__global__ void k_fill_placed(const int32_t* t_idx, int R, const int32_t* off, int32_t* placed) {
  const int rep = blockIdx.x;
  const int lane = threadIdx.x;  // one warp, in order
  int32_t w = off[rep];
  for (int base = 0; base < R; base += 32) {
    const int r = base + lane;
    const bool m = r < R && t_idx[r] == rep;
    const unsigned bm = __ballot_sync(kFull, m);
    if (m) placed[w + __popc(bm & lanemask_lt())] = r;
    w += __popc(bm);
  }
}

// ---------------------------------------------------------------- K4 + K5
// First missing block of a chain in a tier, whole CTA (TierStore::matched_prefix
// aligned walk, hierarchy.cpp:88-91).  sm: >= 64 int64.
__device__ int64_t block_walk(const TierDev& t, const uint64_t* hashes, int64_t nh, int64_t* sm) {
  for (int64_t base = 0; base < nh; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool miss = i < nh && idx_find(t, hashes[i]) < 0;
    const unsigned m = __ballot_sync(kFull, miss);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m ? base + (threadIdx.x & ~31) + __ffs(m) - 1 : INT64_MAX;
    __syncthreads();
    int64_t first = INT64_MAX;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) first = min(first, sm[w]);
    __syncthreads();
    if (first != INT64_MAX) return first;
  }
  return nh;
}

// Erase a present, unpinned block by key; safe under concurrent claims of the
// same key (the slot CAS decides).  Returns the freed size (0 if not erased).
__device__ __forceinline__ int64_t erase_claim(const TierDev& t, uint64_t key) {
  const int64_t sl = idx_find_slot(t, key);
  if (sl < 0) return -1;
  unsigned long long* pv = reinterpret_cast<unsigned long long*>(&t.idx[sl].val);
  const unsigned long long v = *reinterpret_cast<volatile unsigned long long*>(pv);
  if (v == 0 || v == kTomb) return -1;
  Block& b = t.log[v - 1];
  if (b.pin > 0) return -1;
  if (atomicCAS(pv, v, static_cast<unsigned long long>(kTomb)) != v) return -1;
  b.flags &= ~kAlive;
  return b.e - b.s;
}

struct AdmitArgs {
  const uint64_t* tokens;
  const int64_t* tok_off;
  const int64_t* hash_off;
  const uint64_t* hashes;
  const int32_t* wf;
  const int32_t* role;
  const int32_t* placed_off;
  const int32_t* placed;
  double now;
  int spec;
  int32_t* admitted;
  int64_t* match3;
  int64_t* l3_span;  // [2R] deferred L3 erase span per request
};

struct ChainGetB {
  const uint64_t* hashes;
  int64_t n;
  int B;
  int32_t wf, role;
  __device__ PutItem operator()(int64_t i) const {
    PutItem it;
    it.hash = hashes[i];
    it.parent = i ? hashes[i - 1] : kFnvOffset;
    it.s = i * B;
    it.e = min(it.s + B, n);
    it.wf = wf;
    it.role = role;
    it.orphan = 0;
    return it;
  }
};

// start_prefill, cache side (engine.cpp:799-829), one CTA per replica, in
// placement order:
//   match = lookup(seq, &l3)                       (hierarchy.cpp:109-117)
//   evict_for_space(L1, len - match.l1)            (manager.cpp:102-138)
//   if !satisfied: blocked (stays queued)          (engine.cpp:810)
//   erase_chain_span(L2, l1, l1 + l2_part)         (engine.cpp:825)
//   [erase_chain_span(L3, max(l1,l2), reusable)]   deferred to k_l3_erase
//   insert_chain(L1, seq, len, lineage, now, +1)   (engine.cpp:829)
__global__ void __launch_bounds__(512) k_admit(CtxDev c, AdmitArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t sm[64];
  __shared__ int64_t bc[4];
  const int rep = blockIdx.x;
  TierDev* t1p = c.tiers + 2 * rep;
  TierDev* t2p = c.tiers + 2 * rep + 1;
  const TierDev& t3 = c.tiers[2 * c.n_rep];
  for (int32_t k = a.placed_off[rep]; k < a.placed_off[rep + 1]; ++k) {
    const int r = a.placed[k];
    const int64_t L = a.tok_off[r + 1] - a.tok_off[r];
    const uint64_t* tok = a.tokens + a.tok_off[r];
    const uint64_t* hs = a.hashes + a.hash_off[r];
    const int64_t nh = a.hash_off[r + 1] - a.hash_off[r];
    int64_t m[3];
    for (int tier = 0; tier < 3; ++tier) {
      const TierDev t = tier == 0 ? *t1p : tier == 1 ? *t2p : t3;
      const int64_t kb = block_walk(t, hs, nh, sm);
      const int64_t mm = kb ? matched_from_blocks(kb, L, c.B) : 0;
      if (threadIdx.x == 0) bc[0] = ragged_extend(t, t.log, tok, L, hs, mm, c.B);
      __syncthreads();
      m[tier] = bc[0];
      __syncthreads();
    }
    // evict_for_space(L1, needed): base = l1_occupancy() (manager.cpp:106)
    const int64_t excess = t1p->occupancy + c.decode[rep] + (L - m[0]) - t1p->capacity;
    __syncthreads();
    const EvictOut ev = block_evict(c, t1p, excess, a.spec, nullptr, 0, smem, sm);
    if (!ev.satisfied) {
      if (threadIdx.x == 0) {
        a.admitted[r] = 0;
        a.match3[3 * r] = m[0];
        a.match3[3 * r + 1] = m[1];
        a.match3[3 * r + 2] = m[2];
        a.l3_span[2 * r] = a.l3_span[2 * r + 1] = 0;
      }
      __syncthreads();
      continue;
    }
    const int64_t reusable = max(m[0], max(m[1], m[2]));
    const int64_t l2_part = max(min(reusable, m[1]) - m[0], int64_t{0});
    const int64_t l12 = max(m[0], m[1]);
    const int64_t l3_part = max(reusable - l12, int64_t{0});
    if (l2_part > 0) {  // erase_chain_span(L2, seq, l1, l1 + l2_part)
      const TierDev t2 = *t2p;
      int64_t freed = 0, cnt = 0;
      for (int64_t i = threadIdx.x; i < nh; i += blockDim.x) {
        const int64_t e = min((i + 1) * c.B, L);
        if (e <= m[0] || e > m[0] + l2_part) continue;
        const int64_t sz = erase_claim(t2, hs[i]);
        if (sz >= 0) {
          freed += sz;
          cnt += 1;
        }
      }
      int64_t ft, ct;
      block_exscan(freed, sm, &ft);
      block_exscan(cnt, sm, &ct);
      if (threadIdx.x == 0) {
        t2p->occupancy -= ft;
        t2p->n_alive -= ct;
      }
      __syncthreads();
    }
    // insert_chain(L1, seq, len, lineage, now, +1); make room in the log first
    if (t1p->log_len + nh > t1p->log_cap) {
      __syncthreads();
      block_compact(c, t1p, sm);
    }
    const bool room = t1p->log_len + nh <= t1p->log_cap;
    __syncthreads();
    if (room) {
      if (threadIdx.x < 32) {
        ChainGetB gget{hs, L, c.B, a.wf[r], a.role[r]};
        warp_put_ordered(c, t1p, nh, gget, a.now, +1);
      }
    } else if (threadIdx.x == 0) {
      atomicExch(c.error, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      a.admitted[r] = room ? 1 : 0;
      a.match3[3 * r] = m[0];
      a.match3[3 * r + 1] = m[1];
      a.match3[3 * r + 2] = m[2];
      a.l3_span[2 * r] = l3_part > 0 ? l12 : 0;
      a.l3_span[2 * r + 1] = l3_part > 0 ? reusable : 0;
    }
    __syncthreads();
  }
}

// Deferred erase_chain_span(L3, seq, max(l1,l2), reusable) of every admitted
// request (engine.cpp:826-828).  Erasures commute, so all requests go in
// parallel; the slot CAS makes each block's erase happen once.
__global__ void k_l3_erase(CtxDev c, const int64_t* tok_off, const int64_t* hash_off,
                           const uint64_t* hashes, int R, const int32_t* admitted,
                           const int64_t* l3_span) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= R || admitted[r] != 1) return;
  const int64_t from = l3_span[2 * r], to = l3_span[2 * r + 1];
  if (to <= from) return;
  TierDev* tp = c.tiers + 2 * c.n_rep;
  const TierDev t = *tp;
  const int64_t L = tok_off[r + 1] - tok_off[r];
  const uint64_t* hs = hashes + hash_off[r];
  const int64_t nh = hash_off[r + 1] - hash_off[r];
  int64_t freed = 0, cnt = 0;
  for (int64_t i = lane; i < nh; i += 32) {
    const int64_t e = min((i + 1) * c.B, L);
    if (e <= from || e > to) continue;
    const int64_t sz = erase_claim(t, hs[i]);
    if (sz >= 0) {
      freed += sz;
      cnt += 1;
    }
  }
  freed = warp_sum(freed);
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&tp->occupancy),
              static_cast<unsigned long long>(-freed));
    atomicAdd(reinterpret_cast<unsigned long long*>(&tp->n_alive),
              static_cast<unsigned long long>(-cnt));
  }
}

// unpin_chain(seq, len) (hierarchy.cpp:132-142) for admitted requests: one
// warp per request; decrements commute (pin -= 1 only while pin > 0).
__global__ void k_release(CtxDev c, const int64_t* tok_off, const int64_t* hash_off,
                          const uint64_t* hashes, const int32_t* placed_off,
                          const int32_t* placed, const int32_t* admitted) {
  const int rep = blockIdx.x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const TierDev& t = c.tiers[2 * rep];
  for (int32_t k = placed_off[rep] + w; k < placed_off[rep + 1]; k += nw) {
    const int r = placed[k];
    if (admitted[r] != 1) continue;
    const uint64_t* hs = hashes + hash_off[r];
    const int64_t nh = hash_off[r + 1] - hash_off[r];
    for (int64_t i = lane; i < nh; i += 32) {
      const int64_t li = idx_find(t, hs[i]);
      if (li < 0) continue;
      int* pp = &t.log[li].pin;
      int old = *reinterpret_cast<volatile int*>(pp);
      while (old > 0) {
        const int prev = atomicCAS(pp, old, old - 1);
        if (prev == old) break;
        old = prev;
      }
    }
  }
}

struct NbOp {
  int B;
  const int64_t* off;
  __device__ int64_t operator()(int64_t r) const { return (off[r + 1] - off[r] + B - 1) / B; }
};

}  // namespace

// =================================================================== C-ABI
extern "C" {

int pyg_check_device_error(pyg_ctx* c) {
  int32_t e = 0;
  PYG_CUDA(cudaMemcpyAsync(&e, c->hd.error, 4, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaMemsetAsync(c->hd.error, 0, 4, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  if (e) {
    set_error("device-side log capacity exhausted in a batched kernel");
    return PYG_ECAPACITY;
  }
  return PYG_OK;
}

int pyg_hash_offsets_dev(pyg_ctx* c, const int64_t* d_tok_off, int32_t R, int64_t* d_hash_off,
                         int64_t* total) {
  if (!c || R < 0) return PYG_EINVAL;
  void* sp;
  int rc = scratch(c, (R + 2) * sizeof(int64_t), &sp);
  if (rc) return rc;
  auto* nb = static_cast<int64_t*>(sp);
  k_nblocks<<<(R + 256) / 256, 256, 0, c->stream>>>(d_tok_off, R, c->B, nb);
  PYG_LAUNCHED(c);
  size_t tmp = 0;
  PYG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, nb, d_hash_off, R + 1, c->stream));
  void* d_tmp = nullptr;
  PYG_CUDA(cudaMallocAsync(&d_tmp, tmp, c->stream));
  PYG_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, nb, d_hash_off, R + 1, c->stream));
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaFreeAsync(d_tmp, c->stream));
  if (total) {
    PYG_CUDA(cudaMemcpyAsync(total, d_hash_off + R, 8, cudaMemcpyDeviceToHost, c->stream));
    PYG_CUDA(cudaStreamSynchronize(c->stream));
  }
  return PYG_OK;
}

int pyg_hash_batch_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off, int32_t R,
                       const int64_t* d_hash_off, uint64_t* d_hashes) {
  if (!c || R < 0) return PYG_EINVAL;
  if (R == 0) return PYG_OK;
  k_hash_batch<<<(R + 255) / 256, 256, 0, c->stream>>>(d_tokens, d_tok_off, R, d_hash_off,
                                                       d_hashes, c->B);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_staged_matrix_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                          const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t R,
                          const int32_t* d_group, const int32_t* d_cand_off,
                          const int32_t* d_cand, int32_t max_cand, int32_t* d_staged) {
  if (!c || R < 0 || max_cand < 0) return PYG_EINVAL;
  const int64_t n = static_cast<int64_t>(R) * max_cand;
  if (n == 0) return PYG_OK;
  k_staged<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c->stream>>>(
      c->hd, d_tokens, d_tok_off, d_hash_off, d_hashes, R, d_group, d_cand_off, d_cand, max_cand,
      d_staged);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_lookup_batch_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                         const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t R,
                         const int32_t* d_rep, int32_t with_l3, int64_t* d_match3) {
  if (!c || R < 0) return PYG_EINVAL;
  if (R == 0) return PYG_OK;
  k_lookup_batch<<<(R + 127) / 128, 128, 0, c->stream>>>(c->hd, d_tokens, d_tok_off, d_hash_off,
                                                         d_hashes, R, d_rep, with_l3, d_match3);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_route_batch_dev(pyg_ctx* c, int32_t mode, const pyg_nodes_dev* nodes,
                        const pyg_reservation* d_req, int32_t R, const int32_t* d_group,
                        int32_t n_groups, const int32_t* d_cand_off, const int32_t* d_cand,
                        int32_t max_cand, const int32_t* d_staged, double eps,
                        pyg_decision* d_out, int32_t* d_placed_off, int32_t* d_placed) {
  if (!c || !nodes || R < 0 || n_groups < 0) return PYG_EINVAL;
  const int n = c->n_rep;
  // scratch: free, b0, ba, head, tail, app_alpha, app_next, t_idx, counts
  const size_t bytes = n * (8 + 8 + 8 + 4 + 4 + 4) + static_cast<size_t>(R) * (8 + 4 + 4) + 256;
  void* sp;
  int rc = scratch(c, bytes, &sp);
  if (rc) return rc;
  char* p = static_cast<char*>(sp);
  NodeScratch ns;
  ns.free_ = reinterpret_cast<int64_t*>(p);
  p += n * 8;
  ns.b0 = reinterpret_cast<double*>(p);
  p += n * 8;
  ns.ba = reinterpret_cast<double*>(p);
  p += n * 8;
  ns.app_alpha = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(R) * 8;
  ns.head = reinterpret_cast<int32_t*>(p);
  p += n * 4;
  ns.tail = reinterpret_cast<int32_t*>(p);
  p += n * 4;
  ns.app_next = reinterpret_cast<int32_t*>(p);
  p += static_cast<size_t>(R) * 4;
  int32_t* t_idx = reinterpret_cast<int32_t*>(p);
  p += static_cast<size_t>(R) * 4;
  int32_t* cnt = reinterpret_cast<int32_t*>(p);
  if (n) {
    k_node_prep<<<(n + 127) / 128, 128, 0, c->stream>>>(n, *nodes, ns);
    PYG_LAUNCHED(c);
  }
  RouteCtx rcx{*nodes, ns, d_cand_off, d_cand, max_cand, d_staged, eps};
  if (R) {
    if (mode == PYG_ROUTE_SNAPSHOT) {
      k_route_snapshot<<<(R + 7) / 8, 256, 0, c->stream>>>(rcx, d_req, d_group, R, d_out, t_idx);
    } else if (mode == PYG_ROUTE_SEQ_COMMIT) {
      k_route_seq<<<n_groups, 32, 0, c->stream>>>(rcx, d_req, d_group, R, d_out, t_idx);
    } else {
      set_error("unknown route mode");
      return PYG_EINVAL;
    }
    PYG_LAUNCHED(c);
  }
  if (d_placed_off && d_placed && n) {
    k_count_placed<<<n, 256, 0, c->stream>>>(t_idx, R, cnt);
    PYG_LAUNCHED(c);
    k_scan_placed<<<1, 1, 0, c->stream>>>(cnt, n, d_placed_off);
    PYG_LAUNCHED(c);
    k_fill_placed<<<n, 32, 0, c->stream>>>(t_idx, R, d_placed_off, d_placed);
    PYG_LAUNCHED(c);
  }
  return PYG_OK;
}

int pyg_admit_batch_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                        const int64_t* d_hash_off, const uint64_t* d_hashes, const int32_t* d_wf,
                        const int32_t* d_role, int32_t R, const int32_t* d_placed_off,
                        const int32_t* d_placed, double now, int32_t speculative,
                        int32_t* d_admitted, int64_t* d_match3) {
  if (!c || R < 0) return PYG_EINVAL;
  if (R == 0 || c->n_rep == 0) return PYG_OK;
  void* sp;
  int rc = scratch(c, static_cast<size_t>(R) * 16 + 64, &sp);
  if (rc) return rc;
  auto* l3span = static_cast<int64_t*>(sp);
  PYG_CUDA(cudaMemsetAsync(d_admitted, 0, static_cast<size_t>(R) * 4, c->stream));
  PYG_CUDA(cudaMemsetAsync(d_match3, 0, static_cast<size_t>(R) * 24, c->stream));
  AdmitArgs a{d_tokens, d_tok_off, d_hash_off, d_hashes, d_wf, d_role, d_placed_off, d_placed,
              now, speculative, d_admitted, d_match3, l3span};
  const size_t smem = kSmemSortCap * 12;
  cudaFuncSetAttribute(k_admit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_admit<<<c->n_rep, 512, smem, c->stream>>>(c->hd, a);
  PYG_LAUNCHED(c);
  k_l3_erase<<<(R + 7) / 8, 256, 0, c->stream>>>(c->hd, d_tok_off, d_hash_off, d_hashes, R,
                                                 d_admitted, l3span);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_release_batch_dev(pyg_ctx* c, const int64_t* d_tok_off, const int64_t* d_hash_off,
                          const uint64_t* d_hashes, int32_t R, const int32_t* d_placed_off,
                          const int32_t* d_placed, const int32_t* d_admitted) {
  if (!c || R < 0) return PYG_EINVAL;
  if (R == 0 || c->n_rep == 0) return PYG_OK;
  k_release<<<c->n_rep, 256, 0, c->stream>>>(c->hd, d_tok_off, d_hash_off, d_hashes,
                                             d_placed_off, d_placed, d_admitted);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

}  // extern "C"
