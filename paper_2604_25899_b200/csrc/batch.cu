// batch.cu -- batched, device-resident hot path:
//   K1 k_hash_batch       chain_boundary_hashes for every request
//   K2 k_staged / lookup  TierStore::matched_prefix per (request, replica)
//   K3 k_route_*          sched::route, snapshot or sequential-commit
//   K4+K5 k_admit         start_prefill cache side: lookup, evict, promote, insert
//   K5 k_release          unpin_chain of admitted requests
// Every kernel restates the reference function named in its comment.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <string>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

namespace {

// ------------------------------------------------------------------- K2
// (the staged matrix is k_dir.cu: one directory walk per request)
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

// ---------------------------------------------------------------- K4 + K5
// First missing block of a chain (TierStore::matched_prefix aligned walk,
// hierarchy.cpp:88-91) on L1, L2 and L3 at once, whole CTA (blockDim.x == 512,
// sm: >= 64 int64): warps 0-3 probe L1, 4-7 L2, 8-11 L3, 128 boundaries per
// tier per round, so the three walks of a placed request cost one probe latency
// per round instead of three.
__device__ void block_walk3(const TierDev& t0, const TierDev& t1, const TierDev& t2,
                            const uint64_t* hashes, int64_t nh, int64_t* sm, int64_t (&kb)[3]) {
  constexpr int S = 128;
  const int tier = threadIdx.x / S;  // 3: idle warps
  kb[0] = kb[1] = kb[2] = nh;
  bool done[3] = {false, false, false};
  for (int64_t base = 0; base < nh; base += S) {
    const int64_t i = base + (threadIdx.x % S);
    bool miss = false;
    if (tier < 3 && !done[tier] && i < nh) {
      const TierDev& t = tier == 0 ? t0 : tier == 1 ? t1 : t2;
      miss = idx_find(t, hashes[i]) < 0;
    }
    const unsigned m = __ballot_sync(kFull, miss);
    if ((threadIdx.x & 31) == 0)
      sm[threadIdx.x >> 5] = m ? base + ((threadIdx.x % S) & ~31) + __ffs(m) - 1 : INT64_MAX;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int64_t first = min(min(sm[4 * j], sm[4 * j + 1]), min(sm[4 * j + 2], sm[4 * j + 3]));
      if (!done[j] && first != INT64_MAX) {
        kb[j] = first;
        done[j] = true;
      }
    }
    __syncthreads();
    if (done[0] && done[1] && done[2]) break;
  }
}

// Erase a present, unpinned block by key; safe under concurrent claims of the
// same key (the slot CAS decides).  Returns the freed size (0 if not erased).
__device__ __forceinline__ int64_t erase_claim(const TierDev& t, uint64_t key,
                                               int64_t* li = nullptr) {
  const int64_t sl = idx_find_slot(t, key);
  if (sl < 0) return -1;
  unsigned long long* pv = reinterpret_cast<unsigned long long*>(&t.idx[sl].val);
  const unsigned long long v = *reinterpret_cast<volatile unsigned long long*>(pv);
  if (v == 0 || v == kTomb) return -1;
  Block& b = t.log[v - 1];
  if (b.pin > 0) return -1;
  if (atomicCAS(pv, v, static_cast<unsigned long long>(kTomb)) != v) return -1;
  b.flags &= ~kAlive;
  if (li) *li = static_cast<int64_t>(v - 1);
  return b.e - b.s;
}

// Per admission position p (index into the placed CSR = global admission order:
// replica order, then placement order, engine.cpp:742-746): what the ordered L3
// resolution needs.  l3s = L3 match against the L3 of the start of the call,
// kb3 = its aligned block count, l3v = the match with earlier admissions'
// promoted L3 spans erased (the engine's sequential start_prefill).
struct L3Rec {
  int64_t l12, kb3, l3s, l3v;
};

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
  L3Rec* l3rec;  // [n_placed] per admission position
  // sharded step: L2 blocks erased here are exported so every shard's directory follows
  DirRecord* l2_out;
  int64_t l2_cap;
  unsigned long long* l2_count;
  // replicas are taken from a queue, most placements first (k_admit_order)
  const int32_t* rep_order;
  int32_t* rep_next;
  int32_t n_rep;
};

__global__ void k_gate_open(int32_t* gate) { atomicExch(gate, 0); }

// Queue order of k_admit: replicas by descending placement count (a counting sort on one
// CTA), so the CTAs of a grid smaller than the replica count -- or sharing the SMs with K1
// of the next burst -- pull the longest admission sequences first and finish together.
__global__ void __launch_bounds__(1024) k_admit_order(const int32_t* placed_off, int32_t n_rep,
                                                      int32_t* order, int32_t* next,
                                                      int32_t* gate) {
  if (gate && threadIdx.x == 0) atomicExch(gate, 1);  // K1 of another ctx pauses (set_hash_gate)
  __shared__ int32_t hist[1024];
  __shared__ int64_t sm[33];
  hist[threadIdx.x] = 0;
  __syncthreads();
  auto bucket = [&](int r) { return 1023 - min(placed_off[r + 1] - placed_off[r], 1023); };
  for (int r = threadIdx.x; r < n_rep; r += blockDim.x) atomicAdd(&hist[bucket(r)], 1);
  __syncthreads();
  int64_t tot;
  const int64_t pre = block_exscan(hist[threadIdx.x], sm, &tot);
  hist[threadIdx.x] = static_cast<int32_t>(pre);
  __syncthreads();
  for (int r = threadIdx.x; r < n_rep; r += blockDim.x) order[atomicAdd(&hist[bucket(r)], 1)] = r;
  if (threadIdx.x == 0) *next = 0;
}

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
__global__ void __launch_bounds__(512, 2) k_admit(CtxDev c, AdmitArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t sm[64];
  __shared__ int64_t bc[4];
  __shared__ uint32_t sdup[1024];
  __shared__ EvCache ec;
  __shared__ int32_t s_rep;
  for (;;) {
  if (threadIdx.x == 0) {
    const int32_t q = atomicAdd(a.rep_next, 1);
    s_rep = q < a.n_rep ? a.rep_order[q] : -1;
    ec.valid = 0;
  }
  __syncthreads();
  const int rep = s_rep;
  __syncthreads();  // s_rep is rewritten by the next iteration only after every thread read it
  if (rep < 0) break;
  TierDev* t1p = c.tiers + 2 * rep;
  TierDev* t2p = c.tiers + 2 * rep + 1;
  const TierDev& t3 = c.tiers[2 * c.n_rep];
  for (int32_t k = a.placed_off[rep]; k < a.placed_off[rep + 1]; ++k) {
    const int r = a.placed[k];
    const int64_t L = a.tok_off[r + 1] - a.tok_off[r];
    const uint64_t* tok = a.tokens + a.tok_off[r];
    const uint64_t* hs = a.hashes + a.hash_off[r];
    const int64_t nh = a.hash_off[r + 1] - a.hash_off[r];
    // the three aligned walks in one CTA-wide pass, then the three ragged
    // extensions at once, one warp's lane 0 per tier (each is a serial FNV run over <= 63 tokens)
    int64_t m[3], kb3;
    {
      int64_t kb[3];
      block_walk3(*t1p, *t2p, t3, hs, nh, sm, kb);
      for (int tier = 0; tier < 3; ++tier) m[tier] = kb[tier] ? matched_from_blocks(kb[tier], L, c.B) : 0;
      kb3 = kb[2];
    }
    {
      const int tier = threadIdx.x >> 5;
      if (tier < 3 && (threadIdx.x & 31) == 0) {
        const TierDev& t = tier == 0 ? *t1p : tier == 1 ? *t2p : t3;
        bc[tier] = ragged_extend(t, t.log, tok, L, hs, m[tier], c.B);
      }
      __syncthreads();
      m[0] = bc[0];
      m[1] = bc[1];
      m[2] = bc[2];
      __syncthreads();
    }
    if (threadIdx.x == 0 && m[2] > 0 && c.stats) atomicOr(c.stats + 7, 1ULL);
    // evict_for_space(L1, needed): base = l1_occupancy() (manager.cpp:106)
    const int64_t excess = t1p->occupancy + c.decode[rep] + (L - m[0]) - t1p->capacity;
    __syncthreads();
    const EvictOut ev = block_evict_admit(c, t1p, excess, a.spec, smem, sm, &ec);
    if (!ev.satisfied) {
      if (threadIdx.x == 0) {
        if (c.stats) atomicAdd(c.stats + 4, 1ULL);
        a.admitted[r] = 0;
        a.match3[3 * r] = m[0];
        a.match3[3 * r + 1] = m[1];
        a.match3[3 * r + 2] = m[2];
        a.l3rec[k] = L3Rec{max(m[0], m[1]), kb3, m[2], m[2]};
      }
      __syncthreads();
      continue;
    }
    const int64_t reusable = max(m[0], max(m[1], m[2]));
    const int64_t l2_part = max(min(reusable, m[1]) - m[0], int64_t{0});
    const int64_t l12 = max(m[0], m[1]);
    if (l2_part > 0) {  // erase_chain_span(L2, seq, l1, l1 + l2_part)
      const TierDev t2 = *t2p;
      int64_t freed = 0, cnt = 0;
      for (int64_t i = threadIdx.x; i < nh; i += blockDim.x) {
        const int64_t e = min((i + 1) * c.B, L);
        if (e <= m[0] || e > m[0] + l2_part) continue;
        int64_t li;
        const int64_t sz = erase_claim(t2, hs[i], &li);
        if (sz >= 0) {
          freed += sz;
          cnt += 1;
          const Block& eb = t2.log[li];
          dir_note_erase(c, eb, rep);
          if (a.l2_out) {
            const unsigned long long k = atomicAdd(a.l2_count, 1ULL);
            if (static_cast<int64_t>(k) < a.l2_cap)
              a.l2_out[k] = DirRecord{eb.hash, eb.parent, eb.s, eb.e, c.rep_base + rep,
                                      eb.flags & kOrphan};
            else
              atomicExch(c.error, 4);
          }
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
      if (threadIdx.x == 0) ec.valid = 0;  // log indices moved
    }
    const bool room = t1p->log_len + nh <= t1p->log_cap;
    __syncthreads();
    if (room) {
      ChainGetB gget{hs, L, c.B, a.wf[r], a.role[r]};
      // blocks the insert touches get pinned: no longer eviction candidates
      uint32_t* klo = ec.klo;
      const bool cached = ec.valid != 0;
      const int64_t nc = ec.ncand;
      auto drop = [&](int64_t li) {
        if (cached) ev_cache_drop(klo, nc, li);
      };
      if (block_put_ordered(c, t1p, nh, gget, a.now, +1, sdup, sm, drop) && threadIdx.x == 0)
        ec.valid = 0;
    } else if (threadIdx.x == 0) {
      atomicExch(c.error, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (c.stats) {
        atomicAdd(c.stats + 4, 1ULL);
        if (room) atomicAdd(c.stats + 5, 1ULL);
      }
      a.admitted[r] = room ? 1 : 0;
      a.match3[3 * r] = m[0];
      a.match3[3 * r + 1] = m[1];
      a.match3[3 * r + 2] = m[2];
      a.l3rec[k] = L3Rec{l12, kb3, m[2], m[2]};
    }
    __syncthreads();
  }
  }  // replica queue
}

// ------------------------------------------------ ordered L3 (engine order)
// The engine admits one request at a time (start_prefill, engine.cpp:799-829):
// request p looks up the LIVE L3, so it no longer sees the L3 blocks that an
// earlier admission promoted (erase_chain_span(L3, max(l1,l2), reusable),
// engine.cpp:826-828).  k_admit computes every admission's L1/L2 part exactly
// (per replica, in order) and its L3 match against the L3 as of the start of
// the call (nothing touches L3 until here).  The L3 part is a triangular
// system -- p's live L3 match depends only on the erase spans of admissions
// before p -- solved by Jacobi rounds:
//   claim(t): every admitted p erases span(l12, max(l12, l3v)); each L3 block
//             in it records min p as claim = (epoch t, p)          (k_l3_claim)
//   walk(t):  l3v[p] = matched_prefix over the L3 blocks not claimed by an
//             earlier position (aligned walk + ragged check)        (k_l3_walk)
// A round that changes no l3v has reached the fixpoint, which is unique for a
// triangular system, i.e. the sequential result.  After kL3Rounds rounds
// without convergence, k_l3_fixup finishes in order on one CTA from the first
// position that still changed (the prefix before it is a fixpoint of its own
// subsystem, hence exact).  k_l3_final then erases the final spans (or lists
// them, sharded step) and writes the L3 matches.
constexpr int kL3Rounds = 3;

struct L3Args {
  const uint64_t* tokens;
  const int64_t* tok_off;
  const int64_t* hash_off;
  const uint64_t* hashes;
  const int32_t* placed_off;
  const int32_t* placed;
  const int32_t* admitted;
  L3Rec* rec;
  unsigned long long* claim;  // [L3 log_cap], (~epoch << 32) | position, min wins
  int32_t* ctl;               // [1 + t] round t changed something; [16 + t] first change
  int32_t n_rep;
};

__device__ __forceinline__ unsigned long long claim_pack(uint32_t epoch, int p) {
  return (static_cast<unsigned long long>(0xFFFFFFFFu - epoch) << 32) | static_cast<uint32_t>(p);
}

struct ClaimVis {  // block li is visible to position p: no earlier position erases it
  const unsigned long long* claim;
  uint32_t epoch;
  int p;
  __device__ __forceinline__ bool operator()(int64_t li) const {
    const unsigned long long v = __ldcg(claim + li);
    return !((v >> 32) == (0xFFFFFFFFu - epoch) && static_cast<int>(v & 0xffffffffu) < p);
  }
};

// L3 match of admission position p with earlier positions' claims hidden (one warp).
__device__ int64_t l3_visible_match(const CtxDev& c, const L3Args& a, const L3Rec& q, int p,
                                    uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  const int r = a.placed[p];
  const TierDev& t3 = c.tiers[2 * c.n_rep];
  const int64_t L = a.tok_off[r + 1] - a.tok_off[r];
  const uint64_t* hs = a.hashes + a.hash_off[r];
  const ClaimVis vis{a.claim, epoch, p};
  int64_t first = q.kb3;
  for (int64_t base = 0; base < q.kb3; base += 32) {
    const int64_t i = base + lane;
    bool inv = false;
    if (i < q.kb3) {
      const int64_t li = idx_find(t3, hs[i]);
      inv = li < 0 || !vis(li);
    }
    const unsigned m = __ballot_sync(kFull, inv);
    if (m) {
      first = base + __ffs(m) - 1;
      break;
    }
  }
  const int64_t aligned = first ? matched_from_blocks(first, L, c.B) : 0;
  if (first == q.kb3 && q.l3s == aligned) return q.l3s;
  int64_t v = 0;
  if (lane == 0)
    v = ragged_extend(t3, t3.log, a.tokens + a.tok_off[r], L, hs, aligned, c.B, vis);
  return __shfl_sync(kFull, v, 0);
}

// p's erase span claims (one warp): blocks of p's chain with span_end in (l12, reusable]
// present and unpinned in L3 (erase_chain_span, engine.cpp:849-861).
__device__ void l3_claim_span(const CtxDev& c, const L3Args& a, const L3Rec& q, int p,
                              uint32_t epoch) {
  const int64_t reusable = max(q.l12, q.l3v);
  if (reusable <= q.l12) return;
  const int r = a.placed[p];
  const TierDev& t3 = c.tiers[2 * c.n_rep];
  const int64_t L = a.tok_off[r + 1] - a.tok_off[r];
  const uint64_t* hs = a.hashes + a.hash_off[r];
  const int64_t nh = a.hash_off[r + 1] - a.hash_off[r];
  const unsigned long long v = claim_pack(epoch, p);
  for (int64_t i = (q.l12 / c.B) + (threadIdx.x & 31); i < nh; i += 32) {
    const int64_t e = min((i + 1) * c.B, L);
    if (e <= q.l12) continue;
    if (e > reusable) break;
    const int64_t li = idx_find(t3, hs[i]);
    if (li >= 0 && t3.log[li].pin <= 0) atomicMin(a.claim + li, v);
  }
}

__device__ __forceinline__ bool l3_converged_before(const L3Args& a, int t) {
  for (int u = 0; u < t; ++u)
    if (a.ctl[1 + u] == 0) return true;
  return false;
}

__global__ void k_l3_claim(CtxDev c, L3Args a, uint32_t epoch, int t) {
  if (l3_converged_before(a, t)) return;
  const int n = a.placed_off[a.n_rep];
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += nw) {
    if (a.admitted[a.placed[p]] != 1) continue;
    l3_claim_span(c, a, a.rec[p], p, epoch);
  }
}

__global__ void k_l3_walk(CtxDev c, L3Args a, uint32_t epoch, int t) {
  if (l3_converged_before(a, t)) return;
  const int n = a.placed_off[a.n_rep];
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += nw) {
    L3Rec& q = a.rec[p];
    if (q.l3s == 0) continue;  // erasures only shrink matches
    const int64_t v = l3_visible_match(c, a, q, p, epoch);
    if ((threadIdx.x & 31) == 0 && v != q.l3v) {
      q.l3v = v;
      a.ctl[1 + t] = 1;
      atomicMin(a.ctl + 16 + t, p);
    }
  }
}

// Not converged after kL3Rounds: finish in order on one CTA from the first position that
// still changed (epoch = a fresh one: the prefix re-claims, then one position at a time).
__global__ void k_l3_fixup(CtxDev c, L3Args a, uint32_t epoch) {
  if (l3_converged_before(a, kL3Rounds)) return;
  const int n = a.placed_off[a.n_rep];
  const int k0 = a.ctl[16 + kL3Rounds - 1];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int p = w; p < k0; p += nw)
    if (a.admitted[a.placed[p]] == 1) l3_claim_span(c, a, a.rec[p], p, epoch);
  __threadfence();
  __syncthreads();
  if (w != 0) return;
  for (int p = k0; p < n; ++p) {
    L3Rec& q = a.rec[p];
    if (q.l3s == 0) continue;
    const int64_t v = l3_visible_match(c, a, q, p, epoch);
    if ((threadIdx.x & 31) == 0) q.l3v = v;
    __syncwarp();
    if (a.admitted[a.placed[p]] == 1) l3_claim_span(c, a, q, p, epoch);
    __threadfence();
    __syncwarp();
  }
}

// The final spans: erase (or list, sharded step: the shared L3 is replicated and every
// shard applies the union) and report the L3 matches.  Erasing in any order gives the
// sequential result: a block in p's span that an earlier admission already erased is
// erased either way.
__global__ void k_l3_final(CtxDev c, L3Args a, int64_t* match3, uint64_t* list, int64_t list_cap,
                           unsigned long long* list_count) {
  const int n = a.placed_off[a.n_rep];
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  TierDev* tp = c.tiers + 2 * c.n_rep;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += nw) {
    const int r = a.placed[p];
    const L3Rec q = a.rec[p];
    if (lane == 0) match3[3 * r + 2] = q.l3v;
    if (a.admitted[r] != 1) continue;
    const int64_t reusable = max(q.l12, q.l3v);
    if (reusable <= q.l12) continue;
    const TierDev t = *tp;
    const int64_t L = a.tok_off[r + 1] - a.tok_off[r];
    const uint64_t* hs = a.hashes + a.hash_off[r];
    const int64_t nh = a.hash_off[r + 1] - a.hash_off[r];
    int64_t freed = 0, cnt = 0;
    for (int64_t i = (q.l12 / c.B) + lane; i < nh; i += 32) {
      const int64_t e = min((i + 1) * c.B, L);
      if (e <= q.l12 || e > reusable) continue;
      if (list) {
        const unsigned long long k = atomicAdd(list_count, 1ULL);
        if (static_cast<int64_t>(k) < list_cap) list[k] = hs[i];
        else atomicExch(c.error, 4);
        continue;
      }
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
    if (lane == 0 && c.stats) atomicAdd(c.stats + 6, static_cast<unsigned long long>(reusable - q.l12));
  }
}

// unpin_chain(seq, len) (hierarchy.cpp:132-142) of the admitted requests placed on one
// replica (one CTA per replica).  The (request, block) pairs of up to kRelChunk requests are
// flattened over the whole CTA, so a 32k-token prompt's 2,048 unpins take 8 rounds of the
// CTA, not 64 of one warp; decrements commute (pin -= 1 only while pin > 0).
constexpr int kRelChunk = 256;

__global__ void k_release(CtxDev c, const int64_t* tok_off, const int64_t* hash_off,
                          const uint64_t* hashes, const int32_t* placed_off,
                          const int32_t* placed, const int32_t* admitted,
                          const uint8_t* hold, int hold_val, const int32_t* hold_index) {
  __shared__ int64_t s_end[kRelChunk];  // inclusive prefix of the selected requests' blocks
  __shared__ int32_t s_req[kRelChunk];
  __shared__ int64_t sm[64];
  const int rep = blockIdx.x;
  const TierDev t = c.tiers[2 * rep];
  const int32_t p0 = placed_off[rep], p1 = placed_off[rep + 1];
  for (int32_t q0 = p0; q0 < p1; q0 += kRelChunk) {
    const int32_t q = q0 + static_cast<int32_t>(threadIdx.x);
    int64_t nh = 0;
    int32_t r = -1;
    if (threadIdx.x < kRelChunk && q < p1) {
      r = placed[q];
      const bool sel = admitted[r] == 1 && (!hold || hold[hold_index ? hold_index[r] : r] == hold_val);
      if (sel) nh = hash_off[r + 1] - hash_off[r];
    }
    int64_t tot;
    const int64_t before = block_exscan(nh, sm, &tot);
    if (threadIdx.x < kRelChunk) {
      s_end[threadIdx.x] = before + nh;
      s_req[threadIdx.x] = r;
    }
    __syncthreads();
    const int nq = min(kRelChunk, p1 - q0);
    for (int64_t j = threadIdx.x; j < tot; j += blockDim.x) {
      int lo = 0, hi = nq - 1;  // first request whose end > j
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_end[mid] > j) hi = mid;
        else lo = mid + 1;
      }
      const int rr = s_req[lo];
      const int64_t i = j - (s_end[lo] - (hash_off[rr + 1] - hash_off[rr]));
      const int64_t li = idx_find(t, hashes[hash_off[rr] + i]);
      if (li < 0) continue;
      int* pp = &t.log[li].pin;
      int old = *reinterpret_cast<volatile int*>(pp);
      while (old > 0) {
        const int prev = atomicCAS(pp, old, old - 1);
        if (prev == old) break;
        old = prev;
      }
    }
    __syncthreads();
  }
}

// erase_claim of a list of L3 chain hashes (the union of every shard's promoted
// L3 spans, engine.cpp:826-828); duplicates and absent/pinned blocks are no-ops.
__global__ void k_l3_erase_list(CtxDev c, const uint64_t* list, int64_t n,
                                const int64_t* d_count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d_count) n = min(n, *d_count);
  int64_t freed = 0, cnt = 0;
  TierDev* tp = c.tiers + 2 * c.n_rep;
  if (i < n) {
    const int64_t sz = erase_claim(*tp, list[i]);
    if (sz >= 0) {
      freed = sz;
      cnt = 1;
    }
  }
  freed = warp_sum(freed);
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&tp->occupancy),
              static_cast<unsigned long long>(-freed));
    atomicAdd(reinterpret_cast<unsigned long long*>(&tp->n_alive),
              static_cast<unsigned long long>(-cnt));
  }
}

// L2 blocks erased on other shards: clear their directory bits (idempotent)
__global__ void k_dir_clear(CtxDev c, const DirRecord* rec, int64_t n, const int64_t* d_count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (d_count) n = min(n, *d_count);
  if (i >= n || !c.dir_main) return;
  const DirRecord r = rec[i];
  dir_clear_bit(c.dir_main, c.dir_main_mask, c.dir_stride, dir_key(r.hash), r.replica);
  if (r.s % c.B == 0 && r.e % c.B != 0 && r.e > r.s)
    dir_clear_bit(c.dir_rver, c.dir_rver_mask, c.dir_stride, rver_key(r.hash, r.s, r.e),
                  r.replica);
}

// Node table of the next burst: per replica the base reservations, then the reservations
// of the requests the last burst placed there that are still held (hold[r] >= hold_min), in
// placement order (the pool order of reservation_of, engine.cpp:616-628, 686).  One CTA:
// thread n counts replica n's entries, a block scan gives the offsets, thread n copies.
__global__ void __launch_bounds__(1024) k_nodes_compose(int32_t n_rep, const int64_t* base_off,
                                const pyg_reservation* base, const int32_t* placed_off,
                                const int32_t* placed, const pyg_reservation* req,
                                const uint8_t* hold, int hold_min, int64_t* out_off,
                                pyg_reservation* out) {
  __shared__ int64_t sm[64];
  int64_t carry = 0;
  for (int n0 = 0; n0 < n_rep; n0 += blockDim.x) {
    const int n = n0 + threadIdx.x;
    int64_t cnt = 0;
    int32_t p0 = 0, p1 = 0;
    if (n < n_rep) {
      cnt = base_off[n + 1] - base_off[n];
      if (placed_off) {
        p0 = placed_off[n];
        p1 = placed_off[n + 1];
        for (int32_t j = p0; j < p1; ++j) cnt += (!hold || hold[placed[j]] >= hold_min);
      }
    }
    int64_t tot;
    const int64_t o = carry + block_exscan(cnt, sm, &tot);
    if (n < n_rep) {
      out_off[n] = o;
      int64_t w = o;
      for (int64_t i = base_off[n]; i < base_off[n + 1]; ++i) out[w++] = base[i];
      for (int32_t j = p0; j < p1; ++j)
        if (!hold || hold[placed[j]] >= hold_min) out[w++] = req[placed[j]];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) out_off[n_rep] = carry;
}

// dst segment k = src segment idx[k] (CSR gather of uint64 rows: tokens / hashes)
__global__ void k_gather_csr(const uint64_t* src, const int64_t* src_off, const int64_t* idx,
                             int64_t n_idx, const int64_t* dst_off, uint64_t* dst) {
  const int64_t k = blockIdx.x;
  if (k >= n_idx) return;
  const int64_t r = idx[k];
  const int64_t a = src_off[r], len = src_off[r + 1] - a, d = dst_off[k];
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) dst[d + i] = src[a + i];
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

int pyg_check_device_error(pyg_ctx* c) {
  PYG_ON_DEVICE(c);
  int32_t e = 0;
  PYG_CUDA(cudaMemcpyAsync(&e, c->hd.error, 4, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaMemsetAsync(c->hd.error, 0, 4, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  if (e == 7) {
    set_error("16-bit route rows got a staged value >= 65536 (prompt of >= 64k tokens): "
              "rebuild the exchange with 32-bit rows");
    return PYG_ECAPACITY;
  }
  if (e) {
    set_error("device-side capacity exhausted in a batched kernel (code " + std::to_string(e) +
              ")");
    return PYG_ECAPACITY;
  }
  return PYG_OK;
}

int pyg_stats(pyg_ctx* c, int64_t* out, int32_t reset) {
  PYG_ON_DEVICE(c);
  if (!c || !out) return PYG_EINVAL;
  PYG_CUDA(cudaSetDevice(c->device));
  PYG_CUDA(cudaMemcpyAsync(out, c->hd.stats, 64, cudaMemcpyDeviceToHost, c->stream));
  if (reset) PYG_CUDA(cudaMemsetAsync(c->hd.stats, 0, 64, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int pyg_lookup_batch_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                         const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t R,
                         const int32_t* d_rep, int32_t with_l3, int64_t* d_match3) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0) return PYG_EINVAL;
  if (R == 0) return PYG_OK;
  k_lookup_batch<<<(R + 127) / 128, 128, 0, c->stream>>>(c->hd, d_tokens, d_tok_off, d_hash_off,
                                                         d_hashes, R, d_rep, with_l3, d_match3);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

// scratch layout of one admission call: L3Rec[R] | ctl[32] (kept until the L3 stage ran)
// [R] L3 records | 256 B of control words (ctl[60] = k_admit's replica queue head) |
// [n_rep] replica queue order
static int admit_scratch(pyg_ctx* c, int32_t R, L3Rec** rec, int32_t** ctl) {
  void* sp;
  int rc = scratch(c, static_cast<size_t>(R) * sizeof(L3Rec) + 256 +
                          static_cast<size_t>(c->n_rep) * 4, &sp);
  if (rc) return rc;
  *rec = static_cast<L3Rec*>(sp);
  *ctl = reinterpret_cast<int32_t*>(static_cast<char*>(sp) + static_cast<size_t>(R) * sizeof(L3Rec));
  return PYG_OK;
}

// k_admit: everything of start_prefill except the L3 promotion (see l3_stage)
static int admit_core(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                      const int64_t* d_hash_off, const uint64_t* d_hashes, const int32_t* d_wf,
                      const int32_t* d_role, int32_t R, const int32_t* d_placed_off,
                      const int32_t* d_placed, double now, int32_t speculative,
                      int32_t* d_admitted, int64_t* d_match3, void* l2_out, int64_t l2_cap,
                      int64_t* d_counts) {
  if (!c || R < 0) return PYG_EINVAL;
  PYG_CUDA(cudaSetDevice(c->device));
  if (d_counts) PYG_CUDA(cudaMemsetAsync(d_counts, 0, 16, c->stream));
  if (R == 0 || c->n_rep == 0) return PYG_OK;
  L3Rec* rec;
  int32_t* ctl;
  int rc = admit_scratch(c, R, &rec, &ctl);
  if (rc) return rc;
  PYG_CUDA(cudaMemsetAsync(d_admitted, 0, static_cast<size_t>(R) * 4, c->stream));
  PYG_CUDA(cudaMemsetAsync(d_match3, 0, static_cast<size_t>(R) * 24, c->stream));
  PYG_CUDA(cudaMemsetAsync(c->hd.stats + 7, 0, 8, c->stream));  // "some admission hit L3"
  auto* cnt = reinterpret_cast<unsigned long long*>(d_counts);
  int32_t* order = ctl + 64;
  int32_t* next = ctl + 60;
  k_admit_order<<<1, 1024, 0, c->stream>>>(d_placed_off, c->n_rep, order, next, c->d_gate);
  PYG_LAUNCHED(c);
  AdmitArgs a{d_tokens, d_tok_off, d_hash_off, d_hashes, d_wf, d_role, d_placed_off, d_placed,
              now, speculative, d_admitted, d_match3, rec,
              static_cast<DirRecord*>(l2_out), l2_cap, cnt, order, next, c->n_rep};
  const size_t smem = kSmemSortCap * 12;
  PYG_CUDA(cudaFuncSetAttribute(k_admit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // gated K1 (pyg_set_hash_gate): all shared, room for a paused K1 CTA beside it
  if (c->d_gate)
    PYG_CUDA(cudaFuncSetAttribute(k_admit, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  // two CTAs per SM when the SMs are free; each pulls replicas until the queue is empty
  const int grid = std::min(c->n_rep, 2 * pyg_host::sm_count(c->device));
  k_admit<<<grid, 512, smem, c->stream>>>(c->hd, a);
  if (c->d_gate) {
    PYG_LAUNCHED(c);
    k_gate_open<<<1, 1, 0, c->stream>>>(c->d_gate);
  }
  c->dir_admits += 1;
  PYG_LAUNCHED(c);
  return PYG_OK;
}

__global__ void k_clamp_counts(int64_t* counts, int64_t l2_cap, int64_t l3_cap) {
  if (counts[0] > l2_cap) counts[0] = l2_cap;
  if (counts[1] > l3_cap) counts[1] = l3_cap;
}

// The ordered L3 promotion of the admissions k_admit just ran (same arguments): Jacobi
// rounds, the in-order fixup if needed, the final erase (or, l3_out != null, the list of
// erased chain hashes for the sharded step, whose L3 replicas apply every shard's list).
static int l3_stage(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                    const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t R,
                    const int32_t* d_placed_off, const int32_t* d_placed,
                    const int32_t* d_admitted, int64_t* d_match3, uint64_t* l3_out,
                    int64_t l3_cap, int64_t* d_counts) {
  if (!c || R < 0) return PYG_EINVAL;
  PYG_CUDA(cudaSetDevice(c->device));
  if (R == 0 || c->n_rep == 0) return PYG_OK;
  L3Rec* rec;
  int32_t* ctl;
  int rc = admit_scratch(c, R, &rec, &ctl);
  if (rc) return rc;
  // per-L3-block claims; stale epochs read as "no claim"
  const int64_t l3cap = c->tiers[2 * c->n_rep].d.log_cap;
  if (l3cap > c->claim_cap) {
    if (c->d_claim) {
      PYG_CUDA(cudaStreamSynchronize(c->stream));
      PYG_CUDA(cudaFree(c->d_claim));
      c->d_claim = nullptr;
    }
    PYG_CUDA(cudaMalloc(&c->d_claim, static_cast<size_t>(l3cap) * 8));
    PYG_CUDA(cudaMemsetAsync(c->d_claim, 0xff, static_cast<size_t>(l3cap) * 8, c->stream));
    c->claim_cap = l3cap;
  }
  PYG_CUDA(cudaMemsetAsync(ctl, 0, 64, c->stream));
  PYG_CUDA(cudaMemsetAsync(ctl + 16, 0x7f, 64, c->stream));
  L3Args la{d_tokens, d_tok_off, d_hash_off, d_hashes, d_placed_off, d_placed, d_admitted,
            rec, static_cast<unsigned long long*>(c->d_claim), ctl, c->n_rep};
  const unsigned g = static_cast<unsigned>(std::min<int64_t>((R + 7) / 8, 4 * 148));
  for (int t = 0; t < kL3Rounds; ++t) {
    const uint32_t ep = ++c->claim_epoch;
    k_l3_claim<<<g, 256, 0, c->stream>>>(c->hd, la, ep, t);
    PYG_LAUNCHED(c);
    k_l3_walk<<<g, 256, 0, c->stream>>>(c->hd, la, ep, t);
    PYG_LAUNCHED(c);
  }
  k_l3_fixup<<<1, 1024, 0, c->stream>>>(c->hd, la, ++c->claim_epoch);
  PYG_LAUNCHED(c);
  auto* cnt = reinterpret_cast<unsigned long long*>(d_counts);
  k_l3_final<<<g, 256, 0, c->stream>>>(c->hd, la, d_match3, l3_out, l3_cap,
                                       cnt ? cnt + 1 : nullptr);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_admit_batch_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                        const int64_t* d_hash_off, const uint64_t* d_hashes, const int32_t* d_wf,
                        const int32_t* d_role, int32_t R, const int32_t* d_placed_off,
                        const int32_t* d_placed, double now, int32_t speculative,
                        int32_t* d_admitted, int64_t* d_match3) {
  PYG_ON_DEVICE(c);
  int rc = admit_core(c, d_tokens, d_tok_off, d_hash_off, d_hashes, d_wf, d_role, R,
                      d_placed_off, d_placed, now, speculative, d_admitted, d_match3, nullptr, 0,
                      nullptr);
  if (rc) return rc;
  return l3_stage(c, d_tokens, d_tok_off, d_hash_off, d_hashes, R, d_placed_off, d_placed,
                  d_admitted, d_match3, nullptr, 0, nullptr);
}

int pyg_admit_shard_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                        const int64_t* d_hash_off, const uint64_t* d_hashes, const int32_t* d_wf,
                        const int32_t* d_role, int32_t R, const int32_t* d_placed_off,
                        const int32_t* d_placed, double now, int32_t speculative,
                        int32_t* d_admitted, int64_t* d_match3, void* d_l2_erased,
                        int64_t l2_cap, int64_t* d_counts) {
  PYG_ON_DEVICE(c);
  if (!d_counts || (l2_cap && !d_l2_erased)) return PYG_EINVAL;
  return admit_core(c, d_tokens, d_tok_off, d_hash_off, d_hashes, d_wf, d_role, R, d_placed_off,
                    d_placed, now, speculative, d_admitted, d_match3, d_l2_erased, l2_cap,
                    d_counts);
}

int pyg_shard_l3_resolve_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off,
                             const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t R,
                             const int32_t* d_placed_off, const int32_t* d_placed,
                             const int32_t* d_admitted, int64_t* d_match3,
                             uint64_t* d_l3_hashes, int64_t l3_cap, int64_t l2_cap,
                             int64_t* d_counts) {
  PYG_ON_DEVICE(c);
  if (!d_counts || (l3_cap && !d_l3_hashes)) return PYG_EINVAL;
  int rc = l3_stage(c, d_tokens, d_tok_off, d_hash_off, d_hashes, R, d_placed_off, d_placed,
                    d_admitted, d_match3, d_l3_hashes, l3_cap, d_counts);
  if (rc) return rc;
  // peers read these counts over NVLink: never past the lists (overflow is error 4)
  k_clamp_counts<<<1, 1, 0, c->stream>>>(d_counts, l2_cap, l3_cap);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_l3_erase_hashes_dev(pyg_ctx* c, const uint64_t* d_hashes, int64_t n,
                            const int64_t* d_count) {
  PYG_ON_DEVICE(c);
  if (!c || n < 0) return PYG_EINVAL;
  if (!n) return PYG_OK;
  k_l3_erase_list<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c->stream>>>(c->hd, d_hashes, n,
                                                                                 d_count);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_dir_clear_dev(pyg_ctx* c, const void* d_records, int64_t n, const int64_t* d_count) {
  PYG_ON_DEVICE(c);
  if (!c || n < 0) return PYG_EINVAL;
  if (!n) return PYG_OK;
  k_dir_clear<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c->stream>>>(
      c->hd, static_cast<const DirRecord*>(d_records), n, d_count);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_gather_csr_dev(pyg_ctx* c, const uint64_t* d_src, const int64_t* d_src_off,
                       const int64_t* d_idx, int64_t n_idx, const int64_t* d_dst_off,
                       uint64_t* d_dst) {
  PYG_ON_DEVICE(c);
  if (!c || n_idx < 0) return PYG_EINVAL;
  if (!n_idx) return PYG_OK;
  if (n_idx > 0x7fffffff) return PYG_EINVAL;
  k_gather_csr<<<static_cast<unsigned>(n_idx), 128, 0, c->stream>>>(d_src, d_src_off, d_idx, n_idx,
                                                                    d_dst_off, d_dst);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_nodes_compose_dev(pyg_ctx* c, int32_t n_rep, const int64_t* d_base_off,
                          const pyg_reservation* d_base, const int32_t* d_placed_off,
                          const int32_t* d_placed, const pyg_reservation* d_req,
                          const uint8_t* d_hold, int32_t hold_min, int64_t* d_out_off,
                          pyg_reservation* d_out) {
  PYG_ON_DEVICE(c);
  if (!c || n_rep < 0 || (d_placed_off && (!d_placed || !d_req))) return PYG_EINVAL;
  if (!n_rep) return PYG_OK;
  PYG_CUDA(cudaSetDevice(c->device));
  k_nodes_compose<<<1, 1024, 0, c->stream>>>(n_rep, d_base_off, d_base, d_placed_off, d_placed,
                                             d_req, d_hold, hold_min, d_out_off, d_out);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_release_hold_dev(pyg_ctx* c, const int64_t* d_tok_off, const int64_t* d_hash_off,
                         const uint64_t* d_hashes, int32_t R, const int32_t* d_placed_off,
                         const int32_t* d_placed, const int32_t* d_admitted,
                         const uint8_t* d_hold, int32_t hold, const int32_t* d_hold_index) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0) return PYG_EINVAL;
  if (R == 0 || c->n_rep == 0) return PYG_OK;
  PYG_CUDA(cudaSetDevice(c->device));
  k_release<<<c->n_rep, 256, 0, c->stream>>>(c->hd, d_tok_off, d_hash_off, d_hashes,
                                             d_placed_off, d_placed, d_admitted, d_hold, hold,
                                             d_hold_index);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_release_batch_dev(pyg_ctx* c, const int64_t* d_tok_off, const int64_t* d_hash_off,
                          const uint64_t* d_hashes, int32_t R, const int32_t* d_placed_off,
                          const int32_t* d_placed, const int32_t* d_admitted) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0) return PYG_EINVAL;
  if (R == 0 || c->n_rep == 0) return PYG_OK;
  k_release<<<c->n_rep, 256, 0, c->stream>>>(c->hd, d_tok_off, d_hash_off, d_hashes,
                                             d_placed_off, d_placed, d_admitted, nullptr, 0,
                                             nullptr);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

}  // extern "C"

// ======================================================= host-buffer entry
// Device buffers for the host entry live in pyg_ctx::d_list (shared with the completion
// sweep's lists; both are synchronous calls).
extern "C" int pyg_step_host(pyg_ctx* c, const pyg_batch_host* b, const pyg_nodes_host* nd,
                             int32_t mode, double eps, double now, int32_t spec, int32_t release,
                             pyg_decision* out_dec, int32_t* out_adm, int64_t* out_m3) {
  PYG_ON_DEVICE(c);
  if (!c || !b || !nd || b->n_req < 0 || nd->n_groups < 0) return PYG_EINVAL;
  const int32_t R = b->n_req;
  const int nrep = c->n_rep;
  const int64_t T = R ? b->tok_off[R] : 0;
  const int64_t A = nrep ? nd->asg_off[nrep] : 0;
  const int32_t G = nd->n_groups;
  const int32_t NC = G ? nd->cand_off[G] : 0;
  int32_t max_cand = 0;
  for (int g = 0; g < G; ++g) max_cand = std::max(max_cand, nd->cand_off[g + 1] - nd->cand_off[g]);
  int64_t H = 0;
  for (int32_t r = 0; r < R; ++r) H += (b->tok_off[r + 1] - b->tok_off[r] + c->B - 1) / c->B;
  // device layout (each region 256-byte aligned)
  auto al = [](size_t x) { return (x + 255) & ~size_t{255}; };
  size_t off = 0;
  const size_t o_tok = off; off += al(T * 8 + 16);
  const size_t o_toff = off; off += al((R + 1) * 8);
  const size_t o_hoff = off; off += al((R + 1) * 8);
  const size_t o_hash = off; off += al(H * 8 + 8);
  const size_t o_req = off; off += al(R * sizeof(pyg_reservation) + 8);
  const size_t o_grp = off; off += al(R * 4 + 4);
  const size_t o_wf = off; off += al(R * 4 + 4);
  const size_t o_role = off; off += al(R * 4 + 4);
  const size_t o_rid = off; off += al(nrep * 4 + 4);
  const size_t o_kv = off; off += al(nrep * 8 + 8);
  const size_t o_aoff = off; off += al((nrep + 1) * 8);
  const size_t o_asg = off; off += al(A * sizeof(pyg_reservation) + 8);
  const size_t o_coff = off; off += al((G + 1) * 4);
  const size_t o_cand = off; off += al(NC * 4 + 4);
  const size_t o_stg = off; off += al(static_cast<size_t>(R) * std::max(max_cand, 1) * 4);
  const size_t o_dec = off; off += al(R * sizeof(pyg_decision) + 8);
  const size_t o_poff = off; off += al((nrep + 1) * 4);
  const size_t o_pl = off; off += al(R * 4 + 4);
  const size_t o_adm = off; off += al(R * 4 + 4);
  const size_t o_m3 = off; off += al(R * 24 + 8);
  if (off > c->d_list_size) {
    if (c->d_list) {
      PYG_CUDA(cudaStreamSynchronize(c->stream));
      cudaFree(c->d_list);
      c->d_list = nullptr;
    }
    PYG_CUDA(cudaMalloc(&c->d_list, off));
    c->d_list_size = off;
  }
  char* d = static_cast<char*>(c->d_list);
  auto h2d = [&](size_t o, const void* src, size_t n) -> int {
    if (n) PYG_CUDA(cudaMemcpyAsync(d + o, src, n, cudaMemcpyHostToDevice, c->stream));
    return PYG_OK;
  };
  int rc;
  if ((rc = h2d(o_tok, b->tokens, T * 8))) return rc;
  if ((rc = h2d(o_toff, b->tok_off, (R + 1) * 8))) return rc;
  if ((rc = h2d(o_req, b->req, R * sizeof(pyg_reservation)))) return rc;
  if ((rc = h2d(o_grp, b->group, R * 4))) return rc;
  if ((rc = h2d(o_wf, b->workflow, R * 4))) return rc;
  if ((rc = h2d(o_role, b->role, R * 4))) return rc;
  if ((rc = h2d(o_rid, nd->replica_id, nrep * 4))) return rc;
  if ((rc = h2d(o_kv, nd->kv_capacity, nrep * 8))) return rc;
  if ((rc = h2d(o_aoff, nd->asg_off, (nrep + 1) * 8))) return rc;
  if ((rc = h2d(o_asg, nd->asg, A * sizeof(pyg_reservation)))) return rc;
  if ((rc = h2d(o_coff, nd->cand_off, (G + 1) * 4))) return rc;
  if ((rc = h2d(o_cand, nd->cand, NC * 4))) return rc;
  auto* tok = reinterpret_cast<uint64_t*>(d + o_tok);
  auto* toff = reinterpret_cast<int64_t*>(d + o_toff);
  auto* hoff = reinterpret_cast<int64_t*>(d + o_hoff);
  auto* hash = reinterpret_cast<uint64_t*>(d + o_hash);
  if ((rc = pyg_hash_offsets_dev(c, toff, R, hoff, nullptr))) return rc;
  if ((rc = pyg_hash_batch_dev(c, tok, toff, R, hoff, hash))) return rc;
  auto* grp = reinterpret_cast<int32_t*>(d + o_grp);
  auto* coff = reinterpret_cast<int32_t*>(d + o_coff);
  auto* cand = reinterpret_cast<int32_t*>(d + o_cand);
  auto* stg = reinterpret_cast<int32_t*>(d + o_stg);
  if ((rc = pyg_staged_matrix_dev(c, tok, toff, hoff, hash, R, grp, G, coff, cand, max_cand,
                                   stg)))
    return rc;
  pyg_nodes_dev ndv{reinterpret_cast<int32_t*>(d + o_rid), reinterpret_cast<int64_t*>(d + o_kv),
                    reinterpret_cast<int64_t*>(d + o_aoff),
                    reinterpret_cast<pyg_reservation*>(d + o_asg)};
  auto* dec = reinterpret_cast<pyg_decision*>(d + o_dec);
  auto* poff = reinterpret_cast<int32_t*>(d + o_poff);
  auto* pl = reinterpret_cast<int32_t*>(d + o_pl);
  if ((rc = pyg_route_batch_dev(c, mode, &ndv, reinterpret_cast<pyg_reservation*>(d + o_req), R,
                                grp, G, coff, cand, max_cand, stg, eps, dec, poff, pl)))
    return rc;
  auto* adm = reinterpret_cast<int32_t*>(d + o_adm);
  auto* m3 = reinterpret_cast<int64_t*>(d + o_m3);
  if ((rc = pyg_admit_batch_dev(c, tok, toff, hoff, hash, reinterpret_cast<int32_t*>(d + o_wf),
                                reinterpret_cast<int32_t*>(d + o_role), R, poff, pl, now, spec,
                                adm, m3)))
    return rc;
  if (release && (rc = pyg_release_batch_dev(c, toff, hoff, hash, R, poff, pl, adm))) return rc;
  if (R && out_dec)
    PYG_CUDA(cudaMemcpyAsync(out_dec, dec, R * sizeof(pyg_decision), cudaMemcpyDeviceToHost,
                             c->stream));
  if (R && out_adm)
    PYG_CUDA(cudaMemcpyAsync(out_adm, adm, R * 4, cudaMemcpyDeviceToHost, c->stream));
  if (R && out_m3) PYG_CUDA(cudaMemcpyAsync(out_m3, m3, R * 24, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return pyg_check_device_error(c);
}
