// common.cuh -- device data layout and primitives shared by all kernels.
//
// HBM layout (one TierDev per tier; 2 per replica + 1 shared L3 per GPU):
//   log  : Block[log_cap], 64 B records, ascending block_id (the reference's
//          std::map<block_id, CacheBlock> order, hierarchy.hpp:116).  New
//          blocks are appended (ids come from a monotone counter), erase marks
//          the record dead; compaction drops dead records in order.
//   idx  : Slot[2*log_cap] open-addressed chain_hash -> log index
//          (by_chain_hash_, hierarchy.hpp:117).  16 B slots, linear probing,
//          load factor <= 0.5, tombstones cleared by compaction.
//   ridx : RSlot[2*log_cap] "ragged index": parent chain hash -> bitmask of
//          span lengths of ragged blocks (span_end % B != 0) hanging off that
//          prefix.  Replaces the by_span_start_ multimap scan of
//          TierStore::matched_prefix (hierarchy.cpp:92-103) with one probe;
//          the mask is a superset (erase does not clear bits), candidates are
//          verified through idx + span check.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pyg {

constexpr uint64_t kFnvOffset = 1469598103934665603ULL;  // tokens.hpp:19 (non-standard)
constexpr uint64_t kFnvPrime = 1099511628211ULL;         // tokens.hpp:20
constexpr uint64_t kTomb = ~0ULL;
constexpr uint64_t kOrphanTag = 0x9E3779B97F4A7C15ULL;

enum : int32_t { kAlive = 1, kOrphan = 2 };

struct __align__(16) Block {
  uint64_t id;
  uint64_t hash;
  uint64_t parent;  // chain hash of [0, s) for blocks inserted by chain; unused for orphans
  int64_t s, e;     // span [s, e)
  double la;        // last_access
  int32_t wf, role;
  int32_t pin;
  int32_t flags;    // kAlive | kOrphan
};
static_assert(sizeof(Block) == 64, "Block must be 64 bytes");

struct __align__(16) Slot {
  uint64_t key;
  uint64_t val;  // 0 empty, kTomb tombstone, else log index + 1
};

struct __align__(16) RSlot {
  uint64_t key;
  uint64_t mask;  // bit 0 = occupied, bit o = a ragged block of length o hangs off key
};

struct TierDev {
  Block* log;
  Slot* idx;
  RSlot* ridx;
  uint64_t* scratch;  // 2*log_cap words of per-tier scratch (eviction sort keys)
  int64_t log_cap;
  uint64_t idx_mask;  // idx and ridx sizes - 1
  int64_t capacity;   // tokens (TierStore::capacity_)
  int32_t counter;    // index into the ctx id-counter array
  int32_t replica;    // owning replica, -1 for L3
  // mutable, kernel-maintained
  int64_t log_len;
  int64_t n_alive;
  int64_t occupancy;  // TierStore::occupancy_
  int64_t idx_used;
  int64_t n_long_orphans;
};

struct CtxDev {
  TierDev* tiers;       // [2*n_rep + 1]; replica r: L1 = 2r, L2 = 2r+1; L3 = 2*n_rep
  uint64_t* counters;   // [n_rep + 1] next block id per replica (+ L3), hierarchy.hpp:116,122
  int64_t* decode;      // [n_rep] decode_tokens_ (hierarchy.hpp:121)
  int32_t* off;         // [n_rep] replica status Off
  uint8_t* reg_present; // FutureRegistry (manager.hpp:24-32)
  uint64_t* reg_mask;
  int32_t reg_cap;
  int32_t n_rep;
  int32_t B;
  int32_t pad;
  int32_t* error;       // device error flag
  unsigned long long* stats;  // [8] evicted blocks, evicted tokens, evictions run, unsatisfied,
                              //     admissions tried, admitted, L3 tokens promoted, -
  // L2 directory (dir.cuh); main == nullptr until built
  uint64_t* dir_main;
  uint64_t* dir_rver;
  uint64_t dir_main_mask, dir_rver_mask;
  int32_t dir_stride;
  int32_t rep_base;     // global index of replica 0 of this ctx
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  return x;
}

// fnv1a(uint64 v, h) (tokens.hpp:30-36): 8 little-endian bytes.  The 64-bit
// product by P = 2^40 + 0x1B3 is split into 32-bit halves: lo' = lo*0x1B3,
// hi' = hi*0x1B3 + carry + (lo << 8); the lo chain is the only serial path.
__device__ __forceinline__ uint64_t fnv_token(uint64_t h, uint64_t v) {
  uint32_t lo = static_cast<uint32_t>(h), hi = static_cast<uint32_t>(h >> 32);
  const uint32_t vl = static_cast<uint32_t>(v), vh = static_cast<uint32_t>(v >> 32);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w = i < 4 ? vl : vh;
    const uint32_t x = lo ^ ((w >> (8 * (i & 3))) & 0xffu);  // LOP3 (+SHF)
    uint64_t p;                                                // IMAD.WIDE.U32
    asm("mul.wide.u32 %0, %1, 435;" : "=l"(p) : "r"(x));
    uint32_t t;                                                // LEA: (x << 8) + carry
    asm("{\n\t.reg .u32 s;\n\tshl.b32 s, %1, 8;\n\tadd.u32 %0, s, %2;\n\t}"
        : "=r"(t) : "r"(x), "r"(static_cast<uint32_t>(p >> 32)));
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(hi) : "r"(hi), "r"(t));  // IMAD
    lo = static_cast<uint32_t>(p);
  }
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ int64_t blocks_of(int64_t n, int B) { return (n + B - 1) / B; }

// ---------------------------------------------------------------- index ops
__device__ __forceinline__ int64_t idx_find(const TierDev& t, uint64_t key) {
  uint64_t i = mix64(key) & t.idx_mask;
  for (;;) {
    const Slot s = t.idx[i];
    if (s.val == 0) return -1;
    if (s.val != kTomb && s.key == key) return static_cast<int64_t>(s.val - 1);
    i = (i + 1) & t.idx_mask;
  }
}

// returns slot index holding key, or -1
__device__ __forceinline__ int64_t idx_find_slot(const TierDev& t, uint64_t key) {
  uint64_t i = mix64(key) & t.idx_mask;
  for (;;) {
    const Slot s = t.idx[i];
    if (s.val == 0) return -1;
    if (s.val != kTomb && s.key == key) return static_cast<int64_t>(i);
    i = (i + 1) & t.idx_mask;
  }
}

// Insert a key known to be absent.  Concurrent inserters must hold distinct keys.
__device__ __forceinline__ void idx_insert(const TierDev& t, uint64_t key, int64_t log_i) {
  uint64_t i = mix64(key) & t.idx_mask;
  for (;;) {
    unsigned long long* pv = reinterpret_cast<unsigned long long*>(&t.idx[i].val);
    if (*reinterpret_cast<volatile unsigned long long*>(pv) == 0) {
      if (atomicCAS(pv, 0ULL, static_cast<unsigned long long>(log_i + 1)) == 0ULL) {
        t.idx[i].key = key;
        return;
      }
    }
    i = (i + 1) & t.idx_mask;
  }
}

__device__ __forceinline__ uint64_t orphan_key(int64_t s) {
  return kOrphanTag ^ mix64(static_cast<uint64_t>(s) + 0x632BE59BD9B4E019ULL);
}

__device__ __forceinline__ uint64_t ridx_get(const TierDev& t, uint64_t key) {
  uint64_t i = mix64(key ^ 0xA0761D6478BD642FULL) & t.idx_mask;
  for (;;) {
    const RSlot s = t.ridx[i];
    if (s.mask == 0) return 0;
    if (s.key == key) return s.mask;
    i = (i + 1) & t.idx_mask;
  }
}

// Single-writer per key (callers serialize same-key adds).
__device__ __forceinline__ void ridx_add(const TierDev& t, uint64_t key, uint64_t bits) {
  uint64_t i = mix64(key ^ 0xA0761D6478BD642FULL) & t.idx_mask;
  for (;;) {
    unsigned long long* pm = reinterpret_cast<unsigned long long*>(&t.ridx[i].mask);
    unsigned long long m = *reinterpret_cast<volatile unsigned long long*>(pm);
    if (m == 0) {
      if (atomicCAS(pm, 0ULL, 1ULL) == 0ULL) {
        t.ridx[i].key = key;
        __threadfence();
        atomicOr(pm, static_cast<unsigned long long>(bits | 1ULL));
        return;
      }
      continue;  // lost the race; re-read this slot
    }
    if (*reinterpret_cast<volatile uint64_t*>(&t.ridx[i].key) == key) {
      atomicOr(pm, static_cast<unsigned long long>(bits | 1ULL));
      return;
    }
    i = (i + 1) & t.idx_mask;
  }
}

// Records a newly inserted block in the ragged index if it can ever be a
// ragged match (span_start % B == 0 and span_end % B != 0).
__device__ __forceinline__ void ridx_note(const TierDev& t, const Block& b, int B) {
  if (b.s % B != 0 || b.e % B == 0 || b.e <= b.s) return;
  const int64_t len = b.e - b.s;
  if (b.flags & kOrphan) {
    if (len < 64) ridx_add(t, orphan_key(b.s), 1ULL << len);
  } else {
    ridx_add(t, b.parent, 1ULL << len);  // non-orphans come from chains: len < B <= 64
  }
}

// ------------------------------------------------------------- warp helpers
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v, unsigned mask = 0xffffffffu) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// order-preserving map of a double to uint64 (ascending); -0.0 == +0.0
__device__ __forceinline__ uint64_t order_double(double d) {
  d = d + 0.0;
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

// ------------------------------------------------------------ tier mutation
// Erase by log index (TierStore::erase, hierarchy.cpp:68-82).  Caller owns the
// tier (no concurrent mutation of the same record).  Returns the block size.
__device__ __forceinline__ int64_t erase_at(const TierDev& t, int64_t li) {
  Block& b = t.log[li];
  b.flags &= ~kAlive;
  const int64_t sl = idx_find_slot(t, b.hash);
  if (sl >= 0) t.idx[sl].val = kTomb;
  return b.e - b.s;
}

}  // namespace pyg
