// device_ops.cuh -- warp/CTA-level building blocks of the hot path:
// ordered block puts (K5), compaction, eviction select (K4), prefix match (K2)
// and route evaluation (K3).  Each cites the reference function it restates.
#pragma once

#include "common.cuh"

namespace pyg {

constexpr unsigned kFull = 0xffffffffu;

// --------------------------------------------------------------- block scan
// Exclusive scan of one int64 per thread over the CTA; returns the prefix and
// writes the total to *total (all threads).  smem: >= 33 int64.
__device__ __forceinline__ int64_t block_exscan(int64_t v, int64_t* sm, int64_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t s = lane < nw ? sm[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sm[lane] = s;  // inclusive per-warp totals
    if (lane == 31) sm[32] = s;
  }
  __syncthreads();
  const int64_t wp = w ? sm[w - 1] : 0;
  *total = sm[32];
  __syncthreads();
  return wp + x - v;
}

// ------------------------------------------------------------ ordered puts
// One item of an ordered put list (TierStore::put semantics per item).
struct PutItem {
  uint64_t hash, parent;
  int64_t s, e;
  int32_t wf, role;
  int32_t orphan;
};

// Applies TierStore::put (hierarchy.cpp:44-66) for items 0..n-1 IN ORDER,
// 32 at a time on one warp.  Equal hashes inside a chunk are grouped with
// __match_any_sync so the first occurrence inserts (taking the next id) and
// the later ones touch it, exactly as the sequential loop does.  New ids are
// counter + rank among new items (ids follow item order).  Must be called by
// all 32 lanes of one warp; the caller owns the tier (no concurrent mutation).
// Returns (to lane 0) the id of the last item (for single puts).
template <class Get>
__device__ uint64_t warp_put_ordered(const CtxDev& c, TierDev* tp, int64_t n, Get get, double now,
                                     int32_t pin_delta) {
  const int lane = threadIdx.x & 31;
  const TierDev t = *tp;
  uint64_t* ctr = &c.counters[t.counter];
  int64_t log_len = t.log_len;
  uint64_t next_id = *ctr;
  int64_t occ_add = 0, nnew_total = 0;
  uint64_t last_id = 0;
  for (int64_t base = 0; base < n; base += 32) {
    const int64_t i = base + lane;
    const bool active = i < n;
    PutItem it{};
    if (active) it = get(i);
    const unsigned am = __ballot_sync(kFull, active);
    unsigned grp = __match_any_sync(kFull, it.hash) & am;
    const bool leader = active && (__ffs(grp) - 1) == lane;
    const int cnt = __popc(grp);
    int64_t li = -1;
    if (leader) li = idx_find(t, it.hash);
    const bool isnew = leader && li < 0;
    const unsigned nm = __ballot_sync(kFull, isnew);
    const int rank = __popc(nm & lanemask_lt());
    int64_t sz = 0;
    uint64_t my_id = 0;
    if (isnew) {
      const int64_t pos = log_len + rank;
      Block b;
      b.id = next_id + rank;
      b.hash = it.hash;
      b.parent = it.parent;
      b.s = it.s;
      b.e = it.e;
      b.la = now;
      b.wf = it.wf;
      b.role = it.role;
      b.pin = (pin_delta > 0 ? pin_delta : 0) + (cnt - 1) * pin_delta;
      b.flags = kAlive | (it.orphan ? kOrphan : 0);
      t.log[pos] = b;
      idx_insert(t, it.hash, pos);
      sz = b.e - b.s;
      my_id = b.id;
    } else if (leader) {
      Block& b = t.log[li];
      b.la = now;
      b.pin += cnt * pin_delta;
      my_id = b.id;
    }
    // the id seen by each item (followers take their leader's)
    const int src = active ? __ffs(grp) - 1 : lane;
    my_id = __shfl_sync(kFull, my_id, src);
    // ragged-index notes for new blocks, serialized (several may share a parent)
    unsigned rm = __ballot_sync(kFull, isnew && (it.s % c.B == 0) && (it.e % c.B != 0));
    while (rm) {
      const int l = __ffs(rm) - 1;
      if (lane == l) {
        Block b;
        b.s = it.s;
        b.e = it.e;
        b.parent = it.parent;
        b.flags = it.orphan ? kOrphan : 0;
        ridx_note(t, b, c.B);
        if (it.orphan && (it.e - it.s) >= 64) atomicAdd(reinterpret_cast<unsigned long long*>(&tp->n_long_orphans), 1ULL);
      }
      __syncwarp();
      rm &= rm - 1;
    }
    const int nnew = __popc(nm);
    occ_add += warp_sum(sz);
    log_len += nnew;
    next_id += nnew;
    nnew_total += nnew;
    const int lastl = __popc(am) - 1;
    last_id = __shfl_sync(kFull, my_id, lastl < 0 ? 0 : lastl);
    __syncwarp();
  }
  __syncwarp();
  if (lane == 0) {
    tp->log_len = log_len;
    tp->n_alive += nnew_total;
    tp->occupancy += occ_add;
    tp->idx_used += nnew_total;
    *ctr = next_id;
  }
  __syncwarp();
  return last_id;
}

// warp_put_ordered on a whole CTA (same semantics, item order = id order): items are taken
// blockDim at a time; each probes the index in parallel, new blocks get consecutive ids
// and log slots by a block scan, existing ones are touched.  Exact only when no two items
// of a chunk share a hash (the sequential loop would insert the first and touch it with the
// second): a 1024-slot shared filter on the low 32 hash bits detects possible repeats and
// such a chunk (never seen with chain hashes) runs through warp_put_ordered instead.
// sdup: 1024 uint32 of shared memory; sm: >= 41 int64.  touch(log index) is called for every
// existing block the puts touch (not for chunks that took the warp path); returns whether
// any chunk took the warp path.
struct NoTouch {
  __device__ __forceinline__ void operator()(int64_t) const {}
};
template <class Get, class Touch = NoTouch>
__device__ bool block_put_ordered(const CtxDev& c, TierDev* tp, int64_t n, Get get, double now,
                                  int32_t pin_delta, uint32_t* sdup, int64_t* sm,
                                  Touch touch = Touch()) {
  bool slow = false;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t cnt = min(static_cast<int64_t>(blockDim.x), n - base);
    for (int j = threadIdx.x; j < 1024; j += blockDim.x) sdup[j] = 0;
    if (threadIdx.x == 0) sm[40] = 0;
    __syncthreads();
    const bool act = threadIdx.x < cnt;
    PutItem it{};
    if (act) {
      it = get(base + threadIdx.x);
      uint32_t k = static_cast<uint32_t>(it.hash) | 1u;  // 0 marks an empty slot
      uint32_t sl = (static_cast<uint32_t>(it.hash >> 32) * 2654435761u) >> 22;
      for (;;) {
        const uint32_t prev = atomicCAS(sdup + sl, 0u, k);
        if (prev == 0u) break;
        if (prev == k) {
          sm[40] = 1;  // possible repeat (or a 32-bit filter collision)
          break;
        }
        sl = (sl + 1) & 1023u;
      }
    }
    __syncthreads();
    if (sm[40]) {  // exact sequential semantics for this chunk
      __syncthreads();
      if (threadIdx.x < 32) {
        struct Shift {
          Get g;
          int64_t b;
          __device__ PutItem operator()(int64_t i) const { return g(b + i); }
        } sh{get, base};
        warp_put_ordered(c, tp, cnt, sh, now, pin_delta);
      }
      __syncthreads();
      slow = true;
      continue;
    }
    const TierDev t = *tp;
    int64_t li = -1;
    if (act) li = idx_find(t, it.hash);
    const bool isnew = act && li < 0;
    int64_t nnew;
    const int64_t rank = block_exscan(isnew ? 1 : 0, sm, &nnew);
    int64_t sz = 0;
    bool rag = false;
    if (isnew) {
      const int64_t pos = t.log_len + rank;
      Block b;
      b.id = c.counters[t.counter] + static_cast<uint64_t>(rank);
      b.hash = it.hash;
      b.parent = it.parent;
      b.s = it.s;
      b.e = it.e;
      b.la = now;
      b.wf = it.wf;
      b.role = it.role;
      b.pin = pin_delta > 0 ? pin_delta : 0;
      b.flags = kAlive | (it.orphan ? kOrphan : 0);
      t.log[pos] = b;
      idx_insert(t, it.hash, pos);
      sz = b.e - b.s;
      rag = (it.s % c.B == 0) && (it.e % c.B != 0);
    } else if (act) {
      Block& b = t.log[li];
      b.la = now;
      b.pin += pin_delta;
      touch(li);
    }
    int64_t occ_add, nrag;
    block_exscan(sz, sm, &occ_add);
    block_exscan(rag ? 1 : 0, sm, &nrag);
    // ragged-index notes: one thread when several (they may share a parent key)
    if (nrag == 1 && rag) {
      Block b;
      b.s = it.s;
      b.e = it.e;
      b.parent = it.parent;
      b.flags = it.orphan ? kOrphan : 0;
      ridx_note(t, b, c.B);
      if (it.orphan && (it.e - it.s) >= 64)
        atomicAdd(reinterpret_cast<unsigned long long*>(&tp->n_long_orphans), 1ULL);
    }
    if (nrag > 1) {
      for (int64_t j = 0; j < cnt; ++j) {
        if (threadIdx.x == j && rag) {
          Block b;
          b.s = it.s;
          b.e = it.e;
          b.parent = it.parent;
          b.flags = it.orphan ? kOrphan : 0;
          ridx_note(t, b, c.B);
          if (it.orphan && (it.e - it.s) >= 64)
            atomicAdd(reinterpret_cast<unsigned long long*>(&tp->n_long_orphans), 1ULL);
        }
        __syncthreads();
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tp->log_len += nnew;
      tp->n_alive += nnew;
      tp->occupancy += occ_add;
      tp->idx_used += nnew;
      c.counters[t.counter] += static_cast<uint64_t>(nnew);
    }
    __syncthreads();
  }
  return slow;
}

// ------------------------------------------------------------- compaction
// In-place stable compaction of a tier's log (drops dead records, keeps id
// order) and rebuild of idx / ridx.  Whole CTA; smem >= 33 int64.
__device__ inline void block_compact(const CtxDev& c, TierDev* tp, int64_t* sm) {
  const TierDev t = *tp;
  const int64_t n = t.log_len;
  int64_t write = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool alive = i < n && (t.log[i].flags & kAlive);
    Block b;
    if (alive) b = t.log[i];
    __syncthreads();
    int64_t tot;
    const int64_t pos = write + block_exscan(alive ? 1 : 0, sm, &tot);
    if (alive) t.log[pos] = b;
    write += tot;
    __syncthreads();
  }
  const uint64_t nslots = t.idx_mask + 1;
  for (uint64_t i = threadIdx.x; i < nslots; i += blockDim.x) {
    t.idx[i] = Slot{0, 0};
    t.ridx[i] = RSlot{0, 0};
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < write; i += blockDim.x) idx_insert(t, t.log[i].hash, i);
  __syncthreads();
  // ragged index: warp 0, chunks of 32, equal keys grouped
  int64_t long_orphans = 0;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int64_t base = 0; base < write; base += 32) {
      const int64_t i = base + lane;
      bool el = false;
      uint64_t key = 0, bits = 0;
      if (i < write) {
        const Block& b = t.log[i];
        if (b.s % c.B == 0 && b.e % c.B != 0 && b.e > b.s) {
          const int64_t len = b.e - b.s;
          if (b.flags & kOrphan) {
            if (len < 64) {
              el = true;
              key = orphan_key(b.s);
              bits = 1ULL << len;
            } else {
              long_orphans++;
            }
          } else {
            el = true;
            key = b.parent;
            bits = 1ULL << len;
          }
        }
      }
      const unsigned em = __ballot_sync(kFull, el);
      unsigned grp = __match_any_sync(kFull, key) & em;
      // OR the bits of the group into the leader
      uint64_t acc = 0;
      for (int l = 0; l < 32; ++l) {
        const uint64_t v = __shfl_sync(kFull, bits, l);
        if ((grp >> l) & 1u) acc |= v;
      }
      if (el && (__ffs(grp) - 1) == lane) ridx_add(t, key, acc);
      __syncwarp();
    }
    long_orphans = warp_sum(long_orphans);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tp->log_len = write;
    tp->n_alive = write;
    tp->idx_used = write;
    tp->n_long_orphans = long_orphans;
  }
  __syncthreads();
}

// ------------------------------------------------------------ prefix match
// Aligned walk of TierStore::matched_prefix (hierarchy.cpp:84-91), one warp:
// probes 32 boundary hashes at a time and stops at the first miss.
// Returns the number of leading blocks present (all lanes).
__device__ __forceinline__ int64_t warp_walk(const TierDev& t, const uint64_t* hashes, int64_t nh) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = 0; base < nh; base += 32) {
    const int64_t i = base + lane;
    const bool miss = i < nh && idx_find(t, hashes[i]) < 0;
    const unsigned mm = __ballot_sync(kFull, miss);
    if (mm) return base + __ffs(mm) - 1;
  }
  return nh;
}

// Same walk by one thread (staged-matrix / admission path).
__device__ __forceinline__ int64_t thread_walk(const TierDev& t, const uint64_t* hashes,
                                               int64_t nh) {
  int64_t k = 0;
  while (k < nh && idx_find(t, hashes[k]) >= 0) ++k;
  return k;
}

// Ragged check of TierStore::matched_prefix (hierarchy.cpp:92-103), one
// thread.  The reference scans every block starting at `matched` and re-hashes
// tokens[0, span_end) for each; here the candidates are the span lengths noted
// under the query's own prefix hash (ridx), and each candidate is verified by
// one idx probe of the running hash plus a span check.  Identical result up to
// 64-bit hash collisions (the reference itself treats equal chain hashes as
// equal prefixes, hierarchy.hpp:26-28).
struct AllVisible {
  __device__ __forceinline__ bool operator()(int64_t) const { return true; }
};

// vis(log index): whether a present block counts (the ordered L3 resolution of
// batched admission hides blocks an earlier admission of the same call erases).
template <class Vis = AllVisible>
__device__ inline int64_t ragged_extend(const TierDev& t, const Block* log, const uint64_t* tokens,
                                 int64_t L, const uint64_t* hashes, int64_t matched, int B,
                                 Vis vis = Vis()) {
  if (matched >= L || matched % B != 0) return matched;
  const uint64_t parent = matched == 0 ? kFnvOffset : hashes[matched / B - 1];
  uint64_t mask = ridx_get(t, parent) | ridx_get(t, orphan_key(matched));
  mask &= ~1ULL;
  int64_t best = matched;
  if (mask) {
    uint64_t h = parent;
    const int64_t lim = L - matched < 63 ? L - matched : 63;
    for (int64_t o = 1; o <= lim; ++o) {
      h = fnv_token(h, tokens[matched + o - 1]);
      if ((mask >> o) & 1ULL) {
        const int64_t e = matched + o;
        if (e % B != 0) {
          const int64_t li = idx_find(t, h);
          if (li >= 0 && log[li].s == matched && log[li].e == e && vis(li)) best = e;
        }
      }
      if ((mask >> o) <= 1ULL) break;  // no higher candidate
    }
  }
  if (t.n_long_orphans > 0) {
    // orphan blocks (direct TierStore::put) longer than 63 tokens: literal scan
    for (int64_t k = 0; k < t.log_len; ++k) {
      const Block& b = log[k];
      if (!(b.flags & kAlive) || !(b.flags & kOrphan) || b.s != matched) continue;
      if (b.e > L || b.e % B == 0 || b.e - b.s < 64 || b.e <= best || !vis(k)) continue;
      uint64_t h = parent;
      for (int64_t x = matched; x < b.e; ++x) h = fnv_token(h, tokens[x]);
      if (h == b.hash) best = b.e;
    }
  }
  return best;
}

__device__ __forceinline__ int64_t matched_from_blocks(int64_t k, int64_t L, int B) {
  const int64_t m = k * B;
  return m < L ? m : L;
}

// ---------------------------------------------------------------- eviction
// Sort key of evict_for_space (manager.cpp:125-129): dead lineage first, then
// last_access ascending, then block_id ascending.  The log is in id order, so
// the log index stands in for the id.  hi = order(last_access); lo = class<<31
// | log index (class 0 = dead).
__device__ __forceinline__ bool key_less(uint64_t ah, uint32_t al, uint64_t bh, uint32_t bl) {
  const uint32_t ac = al >> 31, bc = bl >> 31;
  if (ac != bc) return ac < bc;
  if (ah != bh) return ah < bh;
  return (al & 0x7fffffffu) < (bl & 0x7fffffffu);
}

__device__ inline void block_bitonic(uint64_t* hi, uint32_t* lo, int64_t n) {
  for (int64_t k = 2; k <= n; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t ixj = i ^ j;
        if (ixj > i) {
          const bool asc = (i & k) == 0;
          const uint64_t h1 = hi[i], h2 = hi[ixj];
          const uint32_t l1 = lo[i], l2 = lo[ixj];
          const bool gt = key_less(h2, l2, h1, l1);
          if (gt == asc) {
            hi[i] = h2;
            hi[ixj] = h1;
            lo[i] = l2;
            lo[ixj] = l1;
          }
        }
      }
      __syncthreads();
    }
  }
}

constexpr int64_t kSmemSortCap = 8192;  // 96 KB of keys

struct EvictOut {
  int64_t n_freed;
  int64_t freed_tokens;
  int32_t satisfied;
};

// evict_for_space (manager.cpp:102-138) on one tier, whole CTA.
// excess = base + needed - capacity must be computed by the caller (base =
// l1_occupancy for L1).  Candidates = alive unpinned blocks (pin <= 0), in the
// reference order (dead first, last_access ascending, block id ascending); the
// shortest prefix with sum(size) >= excess is erased (all candidates if that is
// unsatisfiable).  freed ids are written in eviction order to out_ids[0..cap).
// smem_keys: kSmemSortCap*12 bytes or nullptr (then the tier scratch is used);
// sm: >= 41 int64.
//
// The candidates are gathered once (key = order(last_access) + class | size |
// log index, log index = id order).  Then, group by group -- a group = the
// candidates sharing (class, last_access) -- the smallest remaining group is
// found with one block reduction; it is taken whole while it does not reach the
// remaining excess, else the cut falls inside it and its members are taken in
// id (= gather) order.  Last-access values are event times, so the cut is
// usually a few groups in; after kEvictGroups groups the remainder is finished
// by a full bitonic sort (block_evict_sorted), which continues the same order.
constexpr int kEvictGroups = 24;

struct EvGroup {  // a (class, last_access) key + the total size of its members
  uint32_t cls;   // 0 dead, 1 live, 2 none
  uint64_t h;
  int64_t sz;
};

__device__ __forceinline__ bool grp_less(uint32_t ac, uint64_t ah, uint32_t bc, uint64_t bh) {
  return ac != bc ? ac < bc : ah < bh;
}

__device__ __forceinline__ EvGroup grp_min(EvGroup a, EvGroup b) {
  if (a.cls == b.cls && a.h == b.h) return EvGroup{a.cls, a.h, a.sz + b.sz};
  return grp_less(a.cls, a.h, b.cls, b.h) ? a : b;
}

__device__ inline EvGroup block_grp_min(EvGroup g) {
  __shared__ int64_t sm[3 * 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    EvGroup y{__shfl_xor_sync(kFull, g.cls, o), __shfl_xor_sync(kFull, g.h, o),
              __shfl_xor_sync(kFull, g.sz, o)};
    g = grp_min(g, y);
  }
  if (lane == 0) {
    sm[3 * w] = g.cls;
    sm[3 * w + 1] = static_cast<int64_t>(g.h);
    sm[3 * w + 2] = g.sz;
  }
  __syncthreads();
  EvGroup r{2u, ~0ull, 0};
  for (int k = 0; k < nw; ++k)
    r = grp_min(r, EvGroup{static_cast<uint32_t>(sm[3 * k]), static_cast<uint64_t>(sm[3 * k + 1]),
                           sm[3 * k + 2]});
  __syncthreads();
  return r;
}

// The sorted remainder (used after kEvictGroups groups, and for candidate sets larger than
// the shared key buffer): the shortest sorted prefix of the alive unpinned blocks with
// sum(size) >= excess, bitonic sort of (class, order(last_access), log index).
__device__ inline EvictOut block_evict_sorted(const CtxDev& c, TierDev* tp, int64_t excess,
                                              int speculative, uint64_t* out_ids, int64_t cap,
                                              unsigned char* smem_keys, int64_t* sm) {
  EvictOut r{0, 0, 1};
  if (excess <= 0) return r;
  const TierDev t = *tp;
  const int64_t n = t.log_len;
  int64_t mine = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const Block& b = t.log[i];
    mine += ((b.flags & kAlive) && b.pin <= 0) ? 1 : 0;
  }
  int64_t ncand;
  block_exscan(mine, sm, &ncand);
  int64_t np2 = 1;
  while (np2 < ncand) np2 <<= 1;
  uint64_t* khi;
  uint32_t* klo;
  if (smem_keys && np2 <= kSmemSortCap) {
    khi = reinterpret_cast<uint64_t*>(smem_keys);
    klo = reinterpret_cast<uint32_t*>(smem_keys + kSmemSortCap * 8);
  } else {
    khi = t.scratch;
    klo = reinterpret_cast<uint32_t*>(t.scratch + 2 * t.log_cap);
  }
  int64_t write = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool cand = false;
    uint64_t h = 0;
    uint32_t l = 0;
    if (i < n) {
      const Block& b = t.log[i];
      cand = (b.flags & kAlive) && b.pin <= 0;
      if (cand) {
        bool dead = false;
        if (speculative) {
          const bool live = b.wf >= 0 && b.wf < c.reg_cap && c.reg_present[b.wf] &&
                            b.role >= 0 && b.role < 64 && ((c.reg_mask[b.wf] >> b.role) & 1ULL);
          dead = !live;  // FutureRegistry::lineage_live (manager.cpp:19-23)
        }
        h = order_double(b.la);
        l = (dead ? 0u : 0x80000000u) | static_cast<uint32_t>(i);
      }
    }
    int64_t tot;
    const int64_t pos = write + block_exscan(cand ? 1 : 0, sm, &tot);
    if (cand) {
      khi[pos] = h;
      klo[pos] = l;
    }
    write += tot;
  }
  for (int64_t i = ncand + threadIdx.x; i < np2; i += blockDim.x) {
    khi[i] = ~0ULL;
    klo[i] = 0xffffffffu;
  }
  __syncthreads();
  block_bitonic(khi, klo, np2);
  int64_t cum = 0, cut = ncand;  // cut = number of victims
  for (int64_t base = 0; base < ncand; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    int64_t sz = 0;
    if (i < ncand) {
      const Block& b = t.log[klo[i] & 0x7fffffffu];
      sz = b.e - b.s;
    }
    int64_t tot;
    const int64_t before = cum + block_exscan(sz, sm, &tot);
    const bool stop_here = i < ncand && before < excess && before + sz >= excess;
    if (stop_here) sm[40] = i + 1;
    __syncthreads();
    const bool found = (cum + tot) >= excess;
    if (found) {
      cut = sm[40];
      __syncthreads();
      break;
    }
    cum += tot;
    __syncthreads();
  }
  int64_t freed = 0;
  for (int64_t i = threadIdx.x; i < cut; i += blockDim.x) {
    const int64_t li = klo[i] & 0x7fffffffu;
    if (out_ids && i < cap) out_ids[i] = t.log[li].id;
    freed += erase_at(t, li);
  }
  int64_t ftot;
  block_exscan(freed, sm, &ftot);
  if (threadIdx.x == 0) {
    tp->occupancy -= ftot;
    tp->n_alive -= cut;
  }
  __syncthreads();
  r.n_freed = cut;
  r.freed_tokens = ftot;
  r.satisfied = ftot >= excess;
  return r;
}

// Warp-segmented ordered passes: warp w of the CTA owns the contiguous range
// [w*seg, min(n, (w+1)*seg)); a range total per warp, one block-level prefix over the
// warps, then each warp walks its range in order with warp scans -- one CTA barrier per
// pass instead of one per 512 elements.
struct WarpSeg {
  int64_t lo, hi;
};
__device__ __forceinline__ WarpSeg warp_seg(int64_t n) {
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
  const int64_t seg = (n + nw - 1) / nw;
  const int64_t lo = min(n, w * seg);
  return WarpSeg{lo, min(n, lo + seg)};
}
// exclusive prefix of the per-warp totals (every lane of warp w gets the sum over warps < w);
// total over all warps to *tot.  swp: >= 32 int64 of shared memory.
__device__ __forceinline__ int64_t warp_seg_prefix(int64_t wtot, int64_t* swp, int64_t* tot) {
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) swp[w] = wtot;
  __syncthreads();
  int64_t pre = 0, all = 0;
  for (int k = 0; k < nw; ++k) {
    const int64_t v = swp[k];
    pre += k < w ? v : 0;
    all += v;
  }
  __syncthreads();
  *tot = all;
  return pre;
}
__device__ __forceinline__ int64_t warp_incl_scan(int64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

__device__ __forceinline__ bool evict_candidate(const Block& b) {
  return (b.flags & kAlive) && b.pin <= 0;
}
// (pin, flags) of a record in one 8-byte load
__device__ __forceinline__ bool evict_candidate_pf(const Block* b) {
  const int2 pf = *reinterpret_cast<const int2*>(&b->pin);
  return (pf.y & kAlive) && pf.x <= 0;
}

// Eviction candidates of one warp's log range, in log order.  The scans are bound by the
// latency of HBM / L2 reads of the 64-byte records, so each lane keeps kScanU records in
// flight: first the (pin, flags) word of all of them, then the key fields of the candidates.
constexpr int kScanU = 4;
constexpr int kGatherU = 2;
__device__ __forceinline__ int64_t warp_count_candidates(const TierDev& t, int64_t lo,
                                                         int64_t hi) {
  const int lane = threadIdx.x & 31;
  int64_t wc = 0;
  for (int64_t base = lo; base < hi; base += 32 * kScanU) {
    bool cand[kScanU];
#pragma unroll
    for (int u = 0; u < kScanU; ++u) {
      const int64_t i = base + 32 * u + lane;
      cand[u] = i < hi ? evict_candidate_pf(t.log + i) : false;
    }
#pragma unroll
    for (int u = 0; u < kScanU; ++u) wc += __popc(__ballot_sync(kFull, cand[u]));
  }
  return wc;
}
// Writes the sort keys of the candidates in [lo, hi) from position wpos on:
// khi = order(last_access), klo = live << 31 | size << 24 | log index.
__device__ __forceinline__ void warp_gather_candidates(const CtxDev& c, const TierDev& t,
                                                       int64_t lo, int64_t hi, int64_t wpos,
                                                       int speculative, uint64_t* khi,
                                                       uint32_t* klo) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = lo; base < hi; base += 32 * kGatherU) {
    bool cand[kGatherU];
#pragma unroll
    for (int u = 0; u < kGatherU; ++u) {
      const int64_t i = base + 32 * u + lane;
      cand[u] = i < hi ? evict_candidate_pf(t.log + i) : false;
    }
    double la[kGatherU];
    int32_t wf[kGatherU], role[kGatherU], sz[kGatherU];
#pragma unroll
    for (int u = 0; u < kGatherU; ++u) {
      la[u] = 0.0;
      wf[u] = role[u] = sz[u] = 0;
      if (cand[u]) {
        const Block& b = t.log[base + 32 * u + lane];
        la[u] = b.la;
        wf[u] = b.wf;
        role[u] = b.role;
        sz[u] = static_cast<int32_t>(b.e - b.s);
      }
    }
#pragma unroll
    for (int u = 0; u < kGatherU; ++u) {
      bool dead = false;
      if (cand[u] && speculative) {
        const bool live = wf[u] >= 0 && wf[u] < c.reg_cap && c.reg_present[wf[u]] &&
                          role[u] >= 0 && role[u] < 64 &&
                          ((c.reg_mask[wf[u]] >> role[u]) & 1ULL);
        dead = !live;  // FutureRegistry::lineage_live (manager.cpp:19-23)
      }
      const unsigned m = __ballot_sync(kFull, cand[u]);
      if (cand[u]) {
        const int64_t pos = wpos + __popc(m & lanemask_lt());
        khi[pos] = order_double(la[u]);
        klo[pos] = (dead ? 0u : 0x80000000u) | (static_cast<uint32_t>(sz[u]) << 24) |
                   static_cast<uint32_t>(base + 32 * u + lane);
      }
      wpos += __popc(m);
    }
  }
}

__device__ inline EvictOut block_evict(const CtxDev& c, TierDev* tp, int64_t excess, int speculative,
                                uint64_t* out_ids, int64_t cap, unsigned char* smem_keys,
                                int64_t* sm) {
  __shared__ int64_t swp[32];
  EvictOut res{0, 0, 1};
  if (excess <= 0) return res;
  const TierDev t = *tp;
  const int64_t n = t.log_len;
  const int lane = threadIdx.x & 31;
  // candidates per warp range of the log
  const WarpSeg ls = warp_seg(n);
  const int64_t wc = warp_count_candidates(t, ls.lo, ls.hi);
  int64_t ncand;
  const int64_t wbase = warp_seg_prefix(wc, swp, &ncand);
  int64_t opos = 0, rem = excess, ftok = 0;
  bool done = false;
  // the grouped path needs the keys in shared memory: log index < 2^24, size < 128
  if (smem_keys && ncand <= kSmemSortCap && n < (1 << 24) && c.B < 128) {
    uint64_t* khi = reinterpret_cast<uint64_t*>(smem_keys);
    uint32_t* klo = reinterpret_cast<uint32_t*>(smem_keys + kSmemSortCap * 8);
    // gather in log (= id) order: key = order(last_access) | class, size, log index
    warp_gather_candidates(c, t, ls.lo, ls.hi, wbase, speculative, khi, klo);
    __syncthreads();
    const WarpSeg cs = warp_seg(ncand);
    uint32_t pc = 0;   // groups <= (pc, ph) are taken (none while `first`)
    uint64_t ph = 0;
    bool first = true;
    for (int g = 0; g < kEvictGroups; ++g) {
      EvGroup loc{2u, ~0ull, 0};
      for (int64_t i = threadIdx.x; i < ncand; i += blockDim.x) {
        const uint32_t cl = klo[i] >> 31;
        const uint64_t h = khi[i];
        if (!first && !grp_less(pc, ph, cl, h)) continue;
        loc = grp_min(loc, EvGroup{cl, h, static_cast<int64_t>((klo[i] >> 24) & 0x7fu)});
      }
      const EvGroup m = block_grp_min(loc);
      if (m.cls == 2u) {  // nothing left: every candidate is freed, unsatisfied
        done = true;
        break;
      }
      const bool whole = m.sz < rem;
      if (whole && !out_ids) {
        // the whole group goes; order is irrelevant without an id list
        int64_t cnt = 0;
        for (int64_t i = threadIdx.x; i < ncand; i += blockDim.x) {
          const uint32_t lo = klo[i];
          if ((lo >> 31) == m.cls && khi[i] == m.h) {
            erase_at(t, lo & 0xffffffu);
            ++cnt;
          }
        }
        int64_t ct;
        warp_seg_prefix(warp_sum(cnt), swp, &ct);
        opos += ct;
      } else {
        // members in id order: sizes before each member within the group decide the cut
        int64_t ms = 0, mc = 0;
        for (int64_t base = cs.lo; base < cs.hi; base += 32) {
          const int64_t i = base + lane;
          const bool mem = i < cs.hi && (klo[i] >> 31) == m.cls && khi[i] == m.h;
          ms += warp_sum(mem ? static_cast<int64_t>((klo[i] >> 24) & 0x7fu) : int64_t{0});
        }
        int64_t all;
        int64_t run = warp_seg_prefix(ms, swp, &all);
        // count of taken members before this warp's range (for the id list positions)
        for (int64_t base = cs.lo; base < cs.hi; base += 32) {
          const int64_t i = base + lane;
          const bool mem = i < cs.hi && (klo[i] >> 31) == m.cls && khi[i] == m.h;
          const int64_t sz = mem ? static_cast<int64_t>((klo[i] >> 24) & 0x7fu) : 0;
          const int64_t incl = warp_incl_scan(sz);
          const bool take = mem && (whole || run + incl - sz < rem);
          mc += __popc(__ballot_sync(kFull, take));
          run += __shfl_sync(kFull, incl, 31);
        }
        int64_t ntk;
        int64_t tpos = opos + warp_seg_prefix(mc, swp, &ntk);
        run = warp_seg_prefix(ms, swp, &all);
        for (int64_t base = cs.lo; base < cs.hi; base += 32) {
          const int64_t i = base + lane;
          const bool mem = i < cs.hi && (klo[i] >> 31) == m.cls && khi[i] == m.h;
          const int64_t sz = mem ? static_cast<int64_t>((klo[i] >> 24) & 0x7fu) : 0;
          const int64_t incl = warp_incl_scan(sz);
          const bool take = mem && (whole || run + incl - sz < rem);
          const unsigned tm = __ballot_sync(kFull, take);
          if (take) {
            const int64_t li = klo[i] & 0xffffffu;
            const int64_t at = tpos + __popc(tm & lanemask_lt());
            if (out_ids && at < cap) out_ids[at] = t.log[li].id;
            erase_at(t, li);
          }
          tpos += __popc(tm);
          run += __shfl_sync(kFull, incl, 31);
        }
        opos += ntk;
        __syncthreads();
      }
      if (!whole) {
        done = true;
        break;
      }
      rem -= m.sz;
      pc = m.cls;
      ph = m.h;
      first = false;
    }
    {  // tokens freed by the grouped phase: the sizes of the erased candidates
      int64_t f = 0;
      for (int64_t i = threadIdx.x; i < ncand; i += blockDim.x) {
        const uint32_t lo = klo[i];
        if (!(t.log[lo & 0xffffffu].flags & kAlive)) f += (lo >> 24) & 0x7fu;
      }
      warp_seg_prefix(warp_sum(f), swp, &ftok);
      rem = excess - ftok;
    }
    if (threadIdx.x == 0) {
      tp->occupancy -= ftok;
      tp->n_alive -= opos;
    }
    __syncthreads();
    res.n_freed = opos;
    res.freed_tokens = ftok;
    res.satisfied = ftok >= excess;
    if (!done) {  // more than kEvictGroups groups: finish with the sorted path
      const EvictOut rest = block_evict_sorted(c, tp, rem, speculative,
                                               out_ids ? out_ids + opos : nullptr,
                                               out_ids ? max(int64_t{0}, cap - opos) : 0,
                                               smem_keys, sm);
      res.n_freed += rest.n_freed;
      res.freed_tokens += rest.freed_tokens;
      res.satisfied = res.freed_tokens >= excess;
    }
  } else {
    res = block_evict_sorted(c, tp, excess, speculative, out_ids, cap, smem_keys, sm);
  }
  if (threadIdx.x == 0 && c.stats) {
    atomicAdd(c.stats, static_cast<unsigned long long>(res.n_freed));
    atomicAdd(c.stats + 1, static_cast<unsigned long long>(res.freed_tokens));
    atomicAdd(c.stats + 2, 1ULL);
    if (!res.satisfied) atomicAdd(c.stats + 3, 1ULL);
  }
  __syncthreads();
  return res;
}

// evict_for_space for the batched admission kernel, which evicts on one replica's L1 many
// times in a row (k_admit: one CTA per replica, placements in order).  Between two of its
// evictions the candidate set only shrinks -- victims are erased, blocks touched by the
// admission's insert_chain become pinned, new blocks arrive pinned, nothing is unpinned
// and the registry is fixed -- so the gathered candidate list (same layout as block_evict)
// stays in shared memory for the CTA's next evictions: erased and pinned entries are marked
// removed (size field 0x7f) instead of re-reading the whole log.  ec->valid = 0 forces a
// fresh gather (first eviction, after a log compaction).  Same selection as block_evict.
struct EvCache {
  int64_t ncand;
  int32_t valid;
  uint64_t* khi;  // the cached keys: shared memory, or the tier scratch beyond kSmemSortCap
  uint32_t* klo;
};
constexpr uint32_t kRemoved = 0x7fu << 24;

__device__ __forceinline__ bool ev_removed(uint32_t lo) { return ((lo >> 24) & 0x7fu) == 0x7fu; }

// marks log index li removed from the cached candidates (binary search: gathered in log order)
__device__ __forceinline__ void ev_cache_drop(uint32_t* klo, int64_t ncand, int64_t li) {
  int64_t lo = 0, hi = ncand;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (static_cast<int64_t>(klo[mid] & 0xffffffu) < li) lo = mid + 1;
    else hi = mid;
  }
  if (lo < ncand && static_cast<int64_t>(klo[lo] & 0xffffffu) == li) klo[lo] |= kRemoved;
}

__device__ inline EvictOut block_evict_admit(const CtxDev& c, TierDev* tp, int64_t excess,
                                             int speculative, unsigned char* smem_keys,
                                             int64_t* sm, EvCache* ec) {
  __shared__ int64_t swp[32];
  EvictOut res{0, 0, 1};
  if (excess <= 0) return res;
  const TierDev t = *tp;
  const int lane = threadIdx.x & 31;
  if (!ec->valid) {
    const int64_t n = t.log_len;
    const WarpSeg ls = warp_seg(n);
    const int64_t wc = warp_count_candidates(t, ls.lo, ls.hi);
    int64_t ncand;
    const int64_t wbase = warp_seg_prefix(wc, swp, &ncand);
    if (n >= (1 << 24) || c.B >= 127) {
      res = block_evict_sorted(c, tp, excess, speculative, nullptr, 0, smem_keys, sm);
      goto stats;
    }
    // keys in shared memory, or (a large L1: config 3's 8.8k-block tiers) in the tier scratch
    uint64_t* khi = ncand <= kSmemSortCap ? reinterpret_cast<uint64_t*>(smem_keys) : t.scratch;
    uint32_t* klo = ncand <= kSmemSortCap
                        ? reinterpret_cast<uint32_t*>(smem_keys + kSmemSortCap * 8)
                        : reinterpret_cast<uint32_t*>(t.scratch + 2 * t.log_cap);
    warp_gather_candidates(c, t, ls.lo, ls.hi, wbase, speculative, khi, klo);
    if (threadIdx.x == 0) {
      ec->ncand = ncand;
      ec->valid = 1;
      ec->khi = khi;
      ec->klo = klo;
    }
    __syncthreads();
  }
  {
    const int64_t ncand = ec->ncand;
    uint64_t* khi = ec->khi;
    uint32_t* klo = ec->klo;
    const WarpSeg cs = warp_seg(ncand);
    int64_t rem = excess, nfreed = 0, ftok = 0;
    uint32_t pc = 0;
    uint64_t ph = 0;
    bool first = true, done = false;
    for (int g = 0; g < kEvictGroups; ++g) {
      EvGroup loc{2u, ~0ull, 0};
      for (int64_t i = threadIdx.x; i < ncand; i += blockDim.x) {
        const uint32_t lo = klo[i];
        if (ev_removed(lo)) continue;
        const uint32_t cl = lo >> 31;
        const uint64_t h = khi[i];
        if (!first && !grp_less(pc, ph, cl, h)) continue;
        loc = grp_min(loc, EvGroup{cl, h, static_cast<int64_t>((lo >> 24) & 0x7fu)});
      }
      const EvGroup m = block_grp_min(loc);
      if (m.cls == 2u) {  // nothing left: every candidate freed, unsatisfied
        done = true;
        break;
      }
      const bool whole = m.sz < rem;
      int64_t tk = 0, tsz = 0;
      if (whole) {
        for (int64_t i = threadIdx.x; i < ncand; i += blockDim.x) {
          const uint32_t lo = klo[i];
          if (!ev_removed(lo) && (lo >> 31) == m.cls && khi[i] == m.h) {
            erase_at(t, lo & 0xffffffu);
            klo[i] = lo | kRemoved;
            ++tk;
            tsz += (lo >> 24) & 0x7fu;
          }
        }
      } else {
        int64_t ms = 0;
        for (int64_t base = cs.lo; base < cs.hi; base += 32) {
          const int64_t i = base + lane;
          bool mem = false;
          uint32_t lo = 0;
          if (i < cs.hi) {
            lo = klo[i];
            mem = !ev_removed(lo) && (lo >> 31) == m.cls && khi[i] == m.h;
          }
          ms += warp_sum(mem ? static_cast<int64_t>((lo >> 24) & 0x7fu) : int64_t{0});
        }
        int64_t all;
        int64_t run = warp_seg_prefix(ms, swp, &all);
        for (int64_t base = cs.lo; base < cs.hi; base += 32) {
          const int64_t i = base + lane;
          bool mem = false;
          uint32_t lo = 0;
          if (i < cs.hi) {
            lo = klo[i];
            mem = !ev_removed(lo) && (lo >> 31) == m.cls && khi[i] == m.h;
          }
          const int64_t sz = mem ? static_cast<int64_t>((lo >> 24) & 0x7fu) : 0;
          const int64_t incl = warp_incl_scan(sz);
          if (mem && run + incl - sz < rem) {
            erase_at(t, lo & 0xffffffu);
            klo[i] = lo | kRemoved;
            ++tk;
            tsz += sz;
          }
          run += __shfl_sync(kFull, incl, 31);
        }
      }
      int64_t s1, s2;
      warp_seg_prefix(warp_sum(tk), swp, &s1);
      warp_seg_prefix(warp_sum(tsz), swp, &s2);
      nfreed += s1;
      ftok += s2;
      if (!whole) {
        done = true;
        break;
      }
      rem -= m.sz;
      pc = m.cls;
      ph = m.h;
      first = false;
    }
    if (threadIdx.x == 0) {
      tp->occupancy -= ftok;
      tp->n_alive -= nfreed;
    }
    __syncthreads();
    res.n_freed = nfreed;
    res.freed_tokens = ftok;
    res.satisfied = ftok >= excess;
    if (!done) {  // more than kEvictGroups groups: the sorted path finishes (regathers)
      if (threadIdx.x == 0) ec->valid = 0;
      const EvictOut rest = block_evict_sorted(c, tp, excess - ftok, speculative, nullptr, 0,
                                               smem_keys, sm);
      res.n_freed += rest.n_freed;
      res.freed_tokens += rest.freed_tokens;
      res.satisfied = res.freed_tokens >= excess;
    }
  }
stats:
  if (threadIdx.x == 0 && c.stats) {
    atomicAdd(c.stats, static_cast<unsigned long long>(res.n_freed));
    atomicAdd(c.stats + 1, static_cast<unsigned long long>(res.freed_tokens));
    atomicAdd(c.stats + 2, 1ULL);
    if (!res.satisfied) atomicAdd(c.stats + 3, 1ULL);
  }
  __syncthreads();
  return res;
}

// ----------------------------------------------------------------- routing
// Per-node evaluation of sched::route (router.cpp:19-50): capacity_holds
// (router.cpp:7-11) + oom_bound ordered sum (router.cpp:13-17).
struct NodeEval {
  bool feasible;
  int64_t headroom;
  double bound;
};

__device__ __forceinline__ int64_t res_tokens(const int64_t p, const int64_t u, const int64_t g) {
  return p + (u > g ? u : g);  // Reservation::tokens (router.hpp:21)
}

// Lexicographic route reduction state.  W = argmax (headroom, staged, -id, -pos)
// (the reference's running update is a strict lexicographic max on
// (headroom, staged, -replica_id) taken in input order);
// tiebreak = first position with headroom H < first position with
// (headroom, staged) == (H, S): that is exactly when the last non-id-tie update
// of the reference loop was a staged tie-win (router.cpp:35-39).
struct RouteAcc {
  int64_t h;
  int64_t s;
  int32_t id;
  int32_t pos;  // -1 = none
};

__device__ __forceinline__ bool acc_better(const RouteAcc& a, const RouteAcc& b) {
  if (a.pos < 0) return false;
  if (b.pos < 0) return true;
  if (a.h != b.h) return a.h > b.h;
  if (a.s != b.s) return a.s > b.s;
  if (a.id != b.id) return a.id < b.id;
  return a.pos < b.pos;
}

__device__ __forceinline__ RouteAcc warp_best(RouteAcc a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    RouteAcc b;
    b.h = __shfl_xor_sync(kFull, a.h, o);
    b.s = __shfl_xor_sync(kFull, a.s, o);
    b.id = __shfl_xor_sync(kFull, a.id, o);
    b.pos = __shfl_xor_sync(kFull, a.pos, o);
    if (acc_better(b, a)) a = b;
  }
  return a;
}

// single-instruction warp reductions (REDUX); 64-bit values as (signed hi, unsigned lo)
__device__ __forceinline__ int64_t redux_max_i64(int64_t v) {
  const int hi = static_cast<int>(v >> 32);
  const unsigned lo = static_cast<unsigned>(v);
  const int mh = __reduce_max_sync(kFull, hi);
  const unsigned ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
  return (static_cast<int64_t>(mh) << 32) | ml;
}

__device__ __forceinline__ int32_t warp_min_i32(int32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

}  // namespace pyg
