/*
 * pyg_oracle.h -- CPU restatement of the Pythia scheduling hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 kernels
 * in paper_2604_25899_b200/csrc.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * path never links or calls it (there is no CPU fallback).
 *
 * Every function restates one reference function literally (same loop order,
 * same tie-breaks, same quirks) and cites the reference file:line it follows.
 * Paths are relative to /root/reference/proj/.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against
 *   (1) the known-answer tests of tests/test_cache.cpp and tests/test_sched.cpp,
 *   (2) golden vectors in tests/golden/ produced by the reference itself
 *       (oracle/_ref, compiled unmodified from the reference sources by
 *       oracle/Makefile; generator script tests/golden/make_golden.py), and
 *   (3) randomized differential runs against oracle/_ref when it is present.
 *
 * Representation notes (equivalences, not changes of behaviour):
 *   - Lineage strings (workflow_id, role_id) are interned to dense ints by the
 *     caller; the reference compares strings (hierarchy.hpp:20-24), interning is
 *     a bijection.
 *   - FutureRegistry role sets are 64-bit masks over interned role ids
 *     (manager.hpp:24-32).
 *   - The reference is built RelWithDebInfo (CMakeLists.txt:8-10), i.e. with
 *     NDEBUG: the asserts in TierStore::put/erase (hierarchy.cpp:50,71) are
 *     compiled out.  The restatement mirrors that (pins may go negative,
 *     erase of a pinned block proceeds).
 */
#ifndef PYG_ORACLE_H
#define PYG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* inc/workflow/tokens.hpp:19-20 (the offset is the reference's, NOT standard FNV). */
#define O_FNV_OFFSET 1469598103934665603ULL
#define O_FNV_PRIME 1099511628211ULL

typedef struct {
  uint64_t id, hash;
  int64_t s, e;    /* span [s, e) */
  int32_t wf, role;
  double la;       /* last_access */
  int32_t pin;
  int32_t alive;
} o_block;

typedef struct {
  int64_t capacity, occupancy;
  o_block* b;      /* ascending block_id (== std::map order), dead entries kept until compaction */
  int64_t n, cap, n_alive;
  uint64_t* hk;    /* chain_hash -> index into b (alive blocks only) */
  int64_t* hv;
  uint8_t* hs;     /* 0 empty, 1 full, 2 tombstone */
  int64_t hcap, hused;
} o_tier;

typedef struct {
  o_tier l1, l2;
  int64_t decode_tokens;
  uint64_t next_id;
  int32_t off;     /* replica status Off (engine.cpp:1069) */
} o_cache;

typedef struct {
  o_tier store;
  uint64_t next_id;
} o_l3;

typedef struct {
  int32_t n, cap;
  uint8_t* present;
  uint64_t* mask;
} o_registry;

/* ---- hashing: tokens.hpp:22-36, hierarchy.cpp:21-30 ---- */
uint64_t o_fnv1a_bytes(const char* s, int64_t n, uint64_t h);
uint64_t o_fnv1a_u64(uint64_t v, uint64_t h);
int64_t o_chain_hashes(const uint64_t* tokens, int64_t n, int64_t B, uint64_t* out);

/* ---- TierStore: hierarchy.cpp:32-104 ---- */
void o_tier_init(o_tier* t, int64_t capacity);
void o_tier_free(o_tier* t);
void o_tier_copy(o_tier* dst, const o_tier* src);
const o_block* o_tier_find(const o_tier* t, uint64_t hash);
o_block* o_tier_find_mut(o_tier* t, uint64_t hash);
o_block* o_tier_by_id(o_tier* t, uint64_t id);
uint64_t o_tier_put(o_tier* t, uint64_t hash, int64_t s, int64_t e, int32_t wf, int32_t role,
                    double now, int32_t pin_delta, uint64_t* counter);
void o_tier_erase(o_tier* t, uint64_t id);
int64_t o_matched_prefix(const o_tier* t, const uint64_t* tokens, int64_t n,
                         const uint64_t* hashes, int64_t nh, int64_t B);
/* writes alive blocks in id order; returns count */
int64_t o_tier_dump(const o_tier* t, o_block* out, int64_t cap);

/* ---- CacheHierarchy: hierarchy.cpp:106-142, hierarchy.hpp:91-123 ---- */
void o_cache_init(o_cache* c, int64_t l1_cap, int64_t l2_cap);
void o_cache_free(o_cache* c);
o_tier* o_cache_tier(o_cache* c, int32_t tier); /* tier(L3) aliases L2 (hierarchy.cpp:106-107) */
void o_lookup(const o_cache* c, const o_l3* l3, const uint64_t* tokens, int64_t n, int64_t B,
              int64_t out[3]);
void o_insert_chain(o_cache* c, int32_t tier, const uint64_t* tokens, int64_t n, int64_t upto,
                    int32_t wf, int32_t role, double now, int32_t pin_delta, int64_t B);
void o_unpin_chain(o_cache* c, const uint64_t* tokens, int64_t n, int64_t upto, int64_t B);
int64_t o_l1_occupancy(const o_cache* c);

void o_l3_init(o_l3* l3);
void o_l3_free(o_l3* l3);
void o_l3_copy(o_l3* dst, const o_l3* src);

/* ---- FutureRegistry: manager.cpp:13-23 ---- */
void o_registry_init(o_registry* r);
void o_registry_free(o_registry* r);
void o_registry_update(o_registry* r, int32_t wf, uint64_t role_mask);
void o_registry_drop(o_registry* r, int32_t wf);
int o_lineage_live(const o_registry* r, int32_t wf, int32_t role);

/* ---- evict_for_space: manager.cpp:102-138 ---- */
/* returns satisfied; freed ids (in eviction order) written to out_ids (if non-null, up to cap);
   *n_freed = total count, *freed_tokens = tokens freed */
int o_evict_for_space(o_cache* c, int32_t tier, int64_t needed, const o_registry* reg,
                      int speculative, uint64_t* out_ids, int64_t cap, int64_t* n_freed,
                      int64_t* freed_tokens);

/* ---- completion: manager.cpp:25-58 ---- */
typedef struct {
  int32_t kind; /* 0 Free, 1 RetainAndWriteL3 */
  int32_t tier;
  uint64_t id;
} o_action;
int64_t o_on_request_complete(const o_cache* c, int32_t wf, uint64_t future_mask, int profiled,
                              o_action* out, int64_t cap);
void o_apply_completion(const o_action* acts, int64_t n, o_cache* c, o_l3* l3, double now);

/* ---- router: router.cpp:7-50 ---- */
typedef struct {
  int64_t prompt_len, upper;
  double alpha;
  int64_t tokens_generated;
} o_res;
typedef struct {
  int32_t target; /* -1 == nullopt (wait) */
  int32_t tiebreak;
  int64_t headroom;
  double oom_bound;
} o_decision;
int64_t o_res_tokens(const o_res* r);
/* nodes given as arrays; assigned reservations in CSR asg_off[n_nodes+1] */
int o_capacity_holds(int64_t kv_capacity, const o_res* asg, int64_t na, const o_res* req);
double o_oom_bound(const o_res* asg, int64_t na, const o_res* req);
o_decision o_route(int32_t n_nodes, const int32_t* replica_id, const int64_t* kv_capacity,
                   const int64_t* asg_off, const o_res* asg, const int64_t* staged,
                   const o_res* req, double epsilon);
int32_t o_route_least_outstanding(int32_t n_nodes, const int32_t* replica_id,
                                  const int64_t* asg_off);

/* ---- engine composition helpers (sim/engine.cpp) ---- */
/* erase_chain_span: engine.cpp:849-861 */
void o_erase_chain_span(o_tier* t, const uint64_t* tokens, int64_t n, int64_t from, int64_t to,
                        int64_t B);
/* cache part of start_prefill: engine.cpp:799-829.  Returns 1 if admitted (eviction satisfied),
   0 if blocked.  match[3] receives the lookup.  If l3_lookup is non-null it is used for the lookup
   (a snapshot) while erasures go to l3_live. */
int o_admit(o_cache* c, const o_l3* l3_lookup, o_l3* l3_live, const o_registry* reg,
            int speculative, const uint64_t* seq, int64_t len, int32_t wf, int32_t role, double now,
            int64_t B, int64_t match[3]);
/* apply_completion_policy: engine.cpp:1063-1080 (audit omitted; registry update included) */
void o_completion_policy(o_cache* caches, int32_t n_rep, o_l3* l3, o_registry* reg, int32_t wf,
                         uint64_t future_mask, double now);

/* heap constructors for FFI callers */
o_cache* o_cache_new(int64_t l1_cap, int64_t l2_cap);
void o_cache_delete(o_cache* c);
o_cache* o_cache_clone(const o_cache* c);
void o_cache_set_off(o_cache* c, int32_t off);
void o_add_decode_tokens(o_cache* c, int64_t n);
o_l3* o_l3_new(void);
void o_l3_delete(o_l3* l);
o_l3* o_l3_clone(const o_l3* l);
o_registry* o_registry_new(void);
void o_registry_delete(o_registry* r);
o_tier* o_store_of(o_cache* c, o_l3* l3, int32_t tier);
uint64_t* o_counter_of(o_cache* c, o_l3* l3, int32_t tier);

#ifdef __cplusplus
}
#endif
#endif
