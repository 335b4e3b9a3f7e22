// dir.cuh -- the L2 directory: one device hash table over the L2 tiers of EVERY
// replica of the cluster (all shards), used to compute a request's whole
// staged row (NodeView::staged_l2_prefix for each candidate, engine.cpp:640-648)
// with ONE chain walk instead of one walk per candidate replica.
//
//   main : chain_hash            -> replica bitmask   (TierStore::find_chain presence,
//                                                      hierarchy.cpp:32-42, aligned walk :88-91)
//   rver : (chain_hash, s, e)    -> replica bitmask   (ragged candidates: a block with
//                                                      span [s, e), s%B == 0, e%B != 0)
//   rlen : parent | orphan_key(s)-> bitmask of ragged lengths e-s (a superset)
//
// Identity: for replica n, walking the request's boundary hashes while bit n
// stays set in main[] gives TierStore::matched_prefix's aligned walk on n's
// L2; the ragged check (hierarchy.cpp:92-103) is "some block of n with span
// [m, m+o), m+o <= L, (m+o)%B != 0 and hash FNV(tokens[0, m+o))" which is bit
// n of rver[(h(m+o), m, m+o)].  Candidates o come from rlen under the query's
// own prefix hash (chain blocks) or under orphan_key(m) (direct puts).
// Orphans longer than 63 tokens are rare (direct TierStore::put only): their
// replicas are flagged in `long_mask` and handled by the literal scan.
//
// The directory is derived state.  A shard builds it from the L2 records of all
// shards (pyg_dir_build_dev); batched admission clears bits as it erases L2
// blocks; every other L2 mutation marks it stale (rebuilt before next use).
// Keys: 0 marks an empty slot, so a chain hash of 0 is stored as kZeroAlias
// (a 2^-64 aliasing, the same class of event as the 64-bit chain-hash
// collisions the reference already treats as prefix equality, hierarchy.hpp:26-28).
#pragma once

#include "common.cuh"

namespace pyg {

constexpr uint64_t kZeroAlias = 0x8BADF00DDEADBEEFULL;
constexpr int kDirMaxWords = 16;  // <= 1024 replicas

struct DirRecord {  // one alive L2 block (export / build unit), 40 B
  uint64_t hash;
  uint64_t parent;
  int64_t s, e;
  int32_t replica;  // global replica index
  int32_t flags;    // kOrphan; kDirLongOrphan marks "replica has long orphans"
};
constexpr int32_t kDirLongOrphan = 0x100;

struct DirDev {
  uint64_t* main;     // [main_cap][stride] : key, mask[W], pad
  uint64_t* rver;     // [rver_cap][stride]
  uint64_t* rlen;     // [rlen_cap][2] : key, length mask
  uint64_t* long_mask;  // [W]
  uint64_t main_mask, rver_mask, rlen_mask;  // capacities - 1
  int32_t W;          // mask words
  int32_t stride;     // words per main/rver slot (1 + W rounded up to even)
  int32_t n_global;   // replicas in the cluster
  int32_t rep_base;   // global index of this ctx's replica 0
};

__device__ __forceinline__ uint64_t dir_key(uint64_t h) { return h ? h : kZeroAlias; }

__device__ __forceinline__ uint64_t rver_key(uint64_t h, int64_t s, int64_t e) {
  return dir_key(h ^ mix64(static_cast<uint64_t>(e) * 0x9E3779B97F4A7C15ULL +
                           static_cast<uint64_t>(s) + 0x2545F4914F6CDD1DULL));
}

// returns the slot index of key (inserting it if absent); table sized so it never fills
__device__ __forceinline__ uint64_t dir_slot_insert(uint64_t* tab, uint64_t cap_mask, int stride,
                                                    uint64_t key) {
  uint64_t i = mix64(key) & cap_mask;
  for (;;) {
    unsigned long long* pk = reinterpret_cast<unsigned long long*>(tab + i * stride);
    unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(pk);
    if (k == 0) k = atomicCAS(pk, 0ULL, static_cast<unsigned long long>(key));
    if (k == 0 || k == key) return i;
    i = (i + 1) & cap_mask;
  }
}

__device__ __forceinline__ int64_t dir_slot_find(const uint64_t* tab, uint64_t cap_mask,
                                                 int stride, uint64_t key) {
  uint64_t i = mix64(key) & cap_mask;
  for (;;) {
    const uint64_t k = tab[i * stride];
    if (k == key) return static_cast<int64_t>(i);
    if (k == 0) return -1;
    i = (i + 1) & cap_mask;
  }
}

__device__ __forceinline__ void dir_set_bit(uint64_t* tab, uint64_t cap_mask, int stride,
                                            uint64_t key, int bit) {
  const uint64_t i = dir_slot_insert(tab, cap_mask, stride, key);
  atomicOr(reinterpret_cast<unsigned long long*>(tab + i * stride + 1 + (bit >> 6)),
           1ULL << (bit & 63));
}

__device__ __forceinline__ void dir_clear_bit(uint64_t* tab, uint64_t cap_mask, int stride,
                                              uint64_t key, int bit) {
  const int64_t i = dir_slot_find(tab, cap_mask, stride, key);
  if (i < 0) return;
  atomicAnd(reinterpret_cast<unsigned long long*>(tab + i * stride + 1 + (bit >> 6)),
            ~(1ULL << (bit & 63)));
}

// An L2 block of global replica `rep` was erased (batched admission): clear its
// presence bits.  rlen stays a superset.
__device__ __forceinline__ void dir_note_erase(const CtxDev& c, const Block& b, int local_rep) {
  if (!c.dir_main) return;
  const int rep = c.rep_base + local_rep;
  dir_clear_bit(c.dir_main, c.dir_main_mask, c.dir_stride, dir_key(b.hash), rep);
  if (b.s % c.B == 0 && b.e % c.B != 0 && b.e > b.s)
    dir_clear_bit(c.dir_rver, c.dir_rver_mask, c.dir_stride, rver_key(b.hash, b.s, b.e), rep);
}

}  // namespace pyg
