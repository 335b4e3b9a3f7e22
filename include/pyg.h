/*
 * pyg.h -- C-ABI of the B200-native Pythia scheduling hot path.
 *
 * The reference (arXiv 2604.25899, /root/reference/proj) has no FFI: its
 * engine calls the cache/scheduler classes directly.  Each
 * entry point below replaces one reference call and names it.  A C++ engine
 * keeps its interfaces by routing the class methods through these functions
 * (INTEGRATION.md shows the adapter); nothing in the signatures is C++ or torch.
 *
 * Conventions
 *   - Every call returns PYG_OK (0) or a negative PYG_E* code; the message is
 *     in pyg_last_error() (thread-local).  No C++ exception crosses the ABI.
 *   - Caller owns every host buffer; the library owns the device tables.
 *   - One pyg_ctx per caller thread and GPU (the reference engine is single-
 *     threaded).  Calls are stream-ordered on the ctx stream and,
 *     unless the name ends in _dev, synchronous.
 *   - Lineage strings (workflow_id, role_id) are interned by the caller to
 *     dense ints; FutureRegistry role sets are 64-bit masks over role ids.
 *   - Tier ids: 0 = L1, 1 = L2, 2 = L3.  CacheHierarchy-level calls keep the
 *     reference quirk that tier(L3) aliases L2 (hierarchy.cpp:106-107);
 *     TierStore-level calls (pyg_tier_*, pyg_matched_prefix) address the
 *     shared L3 store with tier 2.
 *   - _dev calls take device pointers and do not synchronize.
 *   - There is no CPU fallback: every call runs CUDA kernels, and a missing or
 *     failing device is an error (PYG_ECUDA).
 */
#ifndef PYG_H
#define PYG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PYG_OK 0
#define PYG_EINVAL (-1)
#define PYG_ENOMEM (-2)
#define PYG_ECUDA (-3)
#define PYG_ECAPACITY (-4)
#define PYG_ENOTSUP (-5)

#define PYG_L1 0
#define PYG_L2 1
#define PYG_L3 2

typedef struct pyg_ctx pyg_ctx;

typedef struct {
  int32_t block_tokens;        /* B, 1..64; reference: kBlockTokens (hierarchy.hpp:15) */
  int32_t n_replicas;          /* CacheHierarchy instances on this GPU (engine.cpp:141-155) */
  int32_t device;              /* CUDA device ordinal */
  int32_t reserved;
  const int64_t* l1_capacity;  /* [n_replicas] tokens, CacheHierarchy(l1, l2) (hierarchy.hpp:100) */
  const int64_t* l2_capacity;  /* [n_replicas] */
  int64_t min_blocks;          /* initial per-tier block capacity hint (tables grow) */
} pyg_config;

/* Mirrors CacheBlock (hierarchy.hpp:29-40) with interned lineage. 56 bytes. */
typedef struct {
  uint64_t block_id;
  uint64_t chain_hash;
  int64_t span_start, span_end;
  int32_t workflow, role;
  double last_access;
  int32_t pin_count;
  int32_t alive;
} pyg_block;

/* Mirrors sched::Reservation (router.hpp:15-22). */
typedef struct {
  int64_t prompt_len, upper;
  double alpha;
  int64_t tokens_generated;
} pyg_reservation;

/* Mirrors sched::RoutingDecision (router.hpp:31-36); target -1 == nullopt (wait). */
typedef struct {
  int32_t target;
  int32_t tiebreak;
  int64_t headroom;
  double oom_bound;
} pyg_decision;

/* ---------------------------------------------------------------- context */
int pyg_create(const pyg_config* cfg, pyg_ctx** out);
void pyg_destroy(pyg_ctx* ctx);
const char* pyg_last_error(void);
/* Launch on an external stream (cudaStream_t); NULL is the default stream.  Until this is
   called the ctx uses its own non-blocking stream. */
int pyg_set_stream(pyg_ctx* ctx, void* cuda_stream);
int pyg_synchronize(pyg_ctx* ctx);
/* number of kernels this ctx has launched (for the bench's gpu_launches claim) */
int64_t pyg_kernel_launches(pyg_ctx* ctx);
/* Counters since creation / the last reset (synchronizes the ctx stream), out[8]: [0] blocks
   evicted by evict_for_space, [1] their tokens, [2] evictions that had work (excess > 0),
   [3] of those unsatisfied, [4] batched admissions tried, [5] admitted, [6] L3 tokens
   promoted by batched admission, [7] whether the last admission call matched anything in L3
   (the sharded L3 chain's skip condition). */
int pyg_stats(pyg_ctx* ctx, int64_t* out, int32_t reset);
/* (Re)sets a replica's tier capacities -- CacheHierarchy(l1_capacity, l2_capacity)
   (hierarchy.hpp:100) for a replica slot the engine provisions later (engine.cpp:197, 1482). */
int pyg_set_capacity(pyg_ctx* ctx, int32_t replica, int64_t l1_capacity, int64_t l2_capacity);

/* ------------------------------------------------------------- hashing */
/* chain_boundary_hashes (hierarchy.cpp:21-30).  out holds ceil(n/B) hashes. */
int pyg_chain_hashes(pyg_ctx* ctx, const uint64_t* tokens, int64_t n, uint64_t* out,
                     int64_t* n_out);

/* ------------------------------------------------- TierStore (per tier) */
/* TierStore::put (hierarchy.cpp:44-66); id counter = replica's for L1/L2, L3's for L3. */
int pyg_tier_put(pyg_ctx* ctx, int32_t replica, int32_t tier, uint64_t chain_hash,
                 int64_t span_start, int64_t span_end, int32_t workflow, int32_t role, double now,
                 int32_t pin_delta, uint64_t* out_id);
/* TierStore::erase (hierarchy.cpp:68-82) */
int pyg_tier_erase(pyg_ctx* ctx, int32_t replica, int32_t tier, uint64_t block_id);
/* One block of a pyg_tier_put_many list (TierStore::put arguments, hierarchy.cpp:44-66). */
typedef struct {
  uint64_t chain_hash;
  int64_t span_start, span_end;
  int32_t workflow, role;
} pyg_put_item;
/* TierStore::erase / put of a whole list, in list order, stream-ordered (no host sync; the
   host arrays may be reused when the call returns).  put_many returns no ids: for callers
   that do not use them (apply_completion's L3 writes, manager.cpp:44-58). */
int pyg_tier_erase_many(pyg_ctx* ctx, int32_t replica, int32_t tier, const uint64_t* ids,
                        int64_t n);
int pyg_tier_put_many(pyg_ctx* ctx, int32_t replica, int32_t tier, const pyg_put_item* items,
                      int64_t n, double now, int32_t pin_delta);
/* TierStore::find_chain (hierarchy.cpp:32-42) */
int pyg_tier_find(pyg_ctx* ctx, int32_t replica, int32_t tier, uint64_t chain_hash,
                  pyg_block* out, int32_t* found);
/* TierStore::occupancy/capacity/blocks().size() (hierarchy.hpp:50-52) */
int pyg_tier_stats(pyg_ctx* ctx, int32_t replica, int32_t tier, int64_t* occupancy,
                   int64_t* capacity, int64_t* n_blocks);
/* TierStore::blocks() in id order (hierarchy.hpp:52); returns the count in *n (may exceed cap) */
int pyg_tier_dump(pyg_ctx* ctx, int32_t replica, int32_t tier, pyg_block* out, int64_t cap,
                  int64_t* n);
/* TierStore::matched_prefix (hierarchy.cpp:84-104) */
int pyg_matched_prefix(pyg_ctx* ctx, int32_t replica, int32_t tier, const uint64_t* tokens,
                       int64_t n, int64_t* out);

/* -------------------------------------------------------- CacheHierarchy */
/* CacheHierarchy::lookup (hierarchy.cpp:109-117); with_l3 = 0 passes nullptr */
int pyg_lookup(pyg_ctx* ctx, int32_t replica, const uint64_t* tokens, int64_t n,
               int32_t with_l3, int64_t out[3]);
/* CacheHierarchy::insert_chain (hierarchy.cpp:119-130) */
/* CacheHierarchy::lookup of ONE prompt on replicas 0..n_rep-1 at once (the engine's node_view
   loop, engine.cpp:640-648): out[3r..3r+2] = replica r's (l1, l2, l3). */
int pyg_lookup_all(pyg_ctx* ctx, const uint64_t* tokens, int64_t n, int32_t with_l3,
                   int32_t n_rep, int64_t* out);
int pyg_insert_chain(pyg_ctx* ctx, int32_t replica, int32_t tier, const uint64_t* tokens,
                     int64_t n, int64_t upto, int32_t workflow, int32_t role, double now,
                     int32_t pin_delta);
/* CacheHierarchy::unpin_chain (hierarchy.cpp:132-142) */
int pyg_unpin_chain(pyg_ctx* ctx, int32_t replica, const uint64_t* tokens, int64_t n,
                    int64_t upto);
/* CacheHierarchy::add_decode_tokens / l1_occupancy (hierarchy.hpp:111-114) */
int pyg_add_decode_tokens(pyg_ctx* ctx, int32_t replica, int64_t n);
int pyg_l1_occupancy(pyg_ctx* ctx, int32_t replica, int64_t* out);
/* Engine::erase_chain_span (engine.cpp:849-861); tier is TierStore-level (2 = shared L3) */
int pyg_erase_chain_span(pyg_ctx* ctx, int32_t replica, int32_t tier, const uint64_t* tokens,
                         int64_t n, int64_t from, int64_t to);
/* replica status Off (engine.cpp:145; the completion sweep skips it, engine.cpp:1069) */
int pyg_set_replica_off(pyg_ctx* ctx, int32_t replica, int32_t off);

/* ------------------------------------------------------- cache manager */
/* FutureRegistry::update / drop (manager.cpp:13-17) */
int pyg_registry_update(pyg_ctx* ctx, int32_t workflow, uint64_t role_mask);
int pyg_registry_drop(pyg_ctx* ctx, int32_t workflow);
/* evict_for_space (manager.cpp:102-138).  freed ids in eviction order (up to cap); *n_freed is
   the full count. */
int pyg_evict_for_space(pyg_ctx* ctx, int32_t replica, int32_t tier, int64_t needed,
                        int32_t speculative, uint64_t* freed, int64_t cap, int64_t* n_freed,
                        int64_t* freed_tokens, int32_t* satisfied);
/* on_request_complete + apply_completion on one replica (manager.cpp:25-58).  future_mask =
   future_roles(position) (path_analysis.cpp:547-551, evaluated on the host); profiled = 0 for
   an unprofiled request (no actions). */
int pyg_complete(pyg_ctx* ctx, int32_t replica, int32_t workflow, uint64_t future_mask,
                 int32_t profiled, double now, int64_t* n_actions);
/* L3 dead-lineage erase of apply_completion_policy (engine.cpp:1074-1080) */
int pyg_l3_dead_sweep(pyg_ctx* ctx, int32_t workflow, uint64_t future_mask);
/* the whole apply_completion_policy (engine.cpp:1063-1080): registry update, sweep of every
   non-Off replica, then the L3 dead sweep */
int pyg_completion_policy(pyg_ctx* ctx, int32_t workflow, uint64_t future_mask, double now);

/* ----------------------------------------------------------------- router */
/* sched::route (router.cpp:19-50) for one request; nodes as arrays, assigned reservations as a
   CSR (asg_off[n_nodes+1]); staged[n] = NodeView::staged_l2_prefix. */
int pyg_route(pyg_ctx* ctx, int32_t n_nodes, const int32_t* replica_id,
              const int64_t* kv_capacity, const int64_t* asg_off, const pyg_reservation* asg,
              const int64_t* staged, const pyg_reservation* req, double epsilon,
              pyg_decision* out);
/* sched::route_least_outstanding (router.cpp:52-62) */
int pyg_route_least_outstanding(pyg_ctx* ctx, int32_t n_nodes, const int32_t* replica_id,
                                const int64_t* asg_off, int32_t* out);

/* ============================================================ batched path */
/* A batch of R requests, device resident.  tokens CSR: tok_off[R+1]; boundary hashes CSR:
   hash_off[R+1] with hash_off[r+1]-hash_off[r] = ceil(len_r / B) (pyg_hash_offsets_dev). */

/* hash_off from tok_off (exclusive scan of ceil(len/B)); also returns the total on the host
   if total != NULL (one sync). */
int pyg_hash_offsets_dev(pyg_ctx* ctx, const int64_t* d_tok_off, int32_t n_req,
                         int64_t* d_hash_off, int64_t* total);
/* K1: chain_boundary_hashes for every request of the batch. */
int pyg_hash_batch_dev(pyg_ctx* ctx, const uint64_t* d_tokens, const int64_t* d_tok_off,
                       int32_t n_req, const int64_t* d_hash_off, uint64_t* d_hashes);
/* Caps K1's persistent grid at n_ctas CTAs (0 = one per SM, the default).  A hashing ctx
   whose K1 overlaps another ctx's step on a second stream leaves SMs free for the step's
   latency-bound kernels (route, admission) this way. */
int pyg_set_hash_ctas(pyg_ctx* ctx, int32_t n_ctas);
/* K1 grid: 1 (default) persistent, one CTA per SM pulling tasks; 0 one task per warp (CTAs
   retire as their 8 tasks finish, so kernels of a higher-priority stream interleave); 2 as 0
   with at most one K1 CTA per SM (shared memory padded), the rest of each SM left to the
   step's kernels. */
int pyg_set_hash_grid(pyg_ctx* ctx, int32_t mode);
/* Admission gate: K1 launches of hash_ctx pause (warps sleep between 16-token chunks) while
   step_ctx runs an admission (pyg_admit_batch_dev / pyg_admit_shard_dev), so the
   latency-bound admission gets its SMs' issue slots; step_ctx = NULL removes the gate.
   Same device; honoured with K1 grid modes 1 and 2 (room for admission CTAs beside the
   paused K1 CTAs).  step_ctx must outlive hash_ctx's K1 launches. */
int pyg_set_hash_gate(pyg_ctx* hash_ctx, pyg_ctx* step_ctx);
/* K1 prefix memo (default off; CSR path, B % 16 == 0, persistent grid, bursts of >= 1,024
   requests): requests sharing their first 16 tokens take the chain states of one leader's
   first 2,048 tokens for every leading 16-token chunk whose tokens equal the leader's
   (k_memo_match compares them before K1).  Measured: 22 % faster K1 on 40k requests sharing
   2,048-token prefixes, 28 % slower on config 4 (profiles/r02_k1_prefix_memo_ab.txt). */
int pyg_set_hash_memo(pyg_ctx* ctx, int32_t on);
/* K1 hashes prompts of >= min_tokens tokens as split tasks: one warp per prompt, 512 tokens
   at a time, through the low-byte decomposition of FNV-1a (k_hash.cu) -- the same hashes,
   without the long-prompt tail of one lane per request.  0 = never; -1 (default) = a
   threshold from the batch's token count (1,024 .. 16,384 tokens).  Requires B % 16 == 0
   (otherwise ignored). */
int pyg_set_hash_split(pyg_ctx* ctx, int64_t min_tokens);

/* K2: staged matrix.  For request r and its j-th candidate replica cand[cand_off[g_r]+j]
   (g_r = d_group[r] < n_groups), d_staged[r*max_cand + j] = tier(L2).matched_prefix(prompt_r)
   == lookup(prompt, nullptr).l2 as node_view computes it (engine.cpp:640-648).  Computed with
   one walk per request through the L2 directory (every candidate at once); candidates are
   global replica indices (== this ctx's replica indices unless pyg_set_shard was called) and
   must be distinct within a group.  A single-GPU ctx rebuilds a stale directory here. */
int pyg_staged_matrix_dev(pyg_ctx* ctx, const uint64_t* d_tokens, const int64_t* d_tok_off,
                          const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t n_req,
                          const int32_t* d_group, int32_t n_groups, const int32_t* d_cand_off,
                          const int32_t* d_cand, int32_t max_cand, int32_t* d_staged);

/* ------------------------------------------------------- L2 directory / shards */
/* This ctx holds global replicas [rep_base, rep_base + n_replicas) of an n_global-replica
   cluster whose replicas are spread over several ctxs (one per GPU). */
int pyg_set_shard(pyg_ctx* ctx, int32_t rep_base, int32_t n_global);
/* Records (40 B each: hash, parent, span_start, span_end, global replica, flags) of every
   alive L2 block of this ctx; cap from pyg_dir_export_cap.  *n_out = count. */
int64_t pyg_dir_export_cap(pyg_ctx* ctx);
int pyg_dir_export_dev(pyg_ctx* ctx, void* d_records, int64_t cap, int64_t* n_out);
/* (Re)build the directory from the records of every shard (their concatenation). */
int pyg_dir_build_dev(pyg_ctx* ctx, const void* d_records, int64_t n);

/* K2: lookup (l1,l2,l3 matches) of request r against replica d_replica[r] (-1 = skip). */
int pyg_lookup_batch_dev(pyg_ctx* ctx, const uint64_t* d_tokens, const int64_t* d_tok_off,
                         const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t n_req,
                         const int32_t* d_replica, int32_t with_l3, int64_t* d_match3);

/* Node table for batched routing: one node per replica of this ctx, in replica order.
   assigned reservations as a CSR over replicas (device). */
typedef struct {
  const int32_t* replica_id;      /* [n_rep] NodeView::replica_id */
  const int64_t* kv_capacity;     /* [n_rep] */
  const int64_t* asg_off;         /* [n_rep+1] */
  const pyg_reservation* asg;     /* assigned reservations, pool then active (engine.cpp:644-645) */
} pyg_nodes_dev;

#define PYG_ROUTE_SNAPSHOT 0
#define PYG_ROUTE_SEQ_COMMIT 1

/* K3: route every request of the batch.  Candidate groups: group g's candidates are
   cand[cand_off[g] .. cand_off[g+1]) (replica indices of this ctx, ascending id order =
   ready_replicas, engine.cpp:630-638).  SNAPSHOT: each request sees the same node state
   (bit-exact to sched::route per request).  SEQ_COMMIT: requests are routed in order and each
   placement is appended to its node before the next request (engine.cpp:683-688).
   d_placed_off/d_placed (optional, SEQ_COMMIT): per-replica lists of placed request indices
   in placement order, CSR [n_rep+1] and [n_req]. */
int pyg_route_batch_dev(pyg_ctx* ctx, int32_t mode, const pyg_nodes_dev* nodes,
                        const pyg_reservation* d_req, int32_t n_req, const int32_t* d_group,
                        int32_t n_groups, const int32_t* d_cand_off, const int32_t* d_cand,
                        int32_t max_cand, const int32_t* d_staged, double epsilon,
                        pyg_decision* d_out, int32_t* d_placed_off, int32_t* d_placed);

/* K4+K5: admission of placed requests (cache side of start_prefill, engine.cpp:799-829), one
   CTA per replica in placement order: lookup(seq,&l3) -> evict_for_space(L1, len-l1) ->
   erase promoted L2 span -> insert_chain(L1, pin+1).  L3 lookups see the L3 state at the start
   of the call; promoted L3 spans are erased after all admissions (replica order).
   d_admitted[r] = 1 admitted, 0 blocked; d_match3[3r..] = lookup. */
int pyg_admit_batch_dev(pyg_ctx* ctx, const uint64_t* d_tokens, const int64_t* d_tok_off,
                        const int64_t* d_hash_off, const uint64_t* d_hashes,
                        const int32_t* d_wf, const int32_t* d_role, int32_t n_req,
                        const int32_t* d_placed_off, const int32_t* d_placed, double now,
                        int32_t speculative, int32_t* d_admitted, int64_t* d_match3);

/* K5: release admitted requests: unpin_chain(seq, len) on the target replica for every r with
   d_admitted[r] != 0 (hierarchy.cpp:132-142). */
int pyg_release_batch_dev(pyg_ctx* ctx, const int64_t* d_tok_off, const int64_t* d_hash_off,
                          const uint64_t* d_hashes, int32_t n_req, const int32_t* d_placed_off,
                          const int32_t* d_placed, const int32_t* d_admitted);

/* Node-table bookkeeping between bursts (the steady-state step): d_out holds, per replica,
   the base reservations then the reservations d_req[d_placed[j]] of the requests a burst
   placed there (d_placed_off/d_placed from pyg_route_batch_dev) that are still held
   (d_hold[r] >= hold_min; d_hold NULL = all), in placement order -- the pool order of
   reservation_of (engine.cpp:616-628, 686).  d_placed_off may be NULL (base only).
   d_out needs base + placed entries; d_out_off [n_rep+1]. */
int pyg_nodes_compose_dev(pyg_ctx* ctx, int32_t n_rep, const int64_t* d_base_off,
                          const pyg_reservation* d_base, const int32_t* d_placed_off,
                          const int32_t* d_placed, const pyg_reservation* d_req,
                          const uint8_t* d_hold, int32_t hold_min, int64_t* d_out_off,
                          pyg_reservation* d_out);
/* pyg_release_batch_dev restricted to requests with d_hold[i] == hold (their completion
   step), i = d_hold_index[r] (NULL: i = r; the sharded step maps receive slots to global
   request indices): unpin_chain(seq, len) of each (hierarchy.cpp:132-142). */
int pyg_release_hold_dev(pyg_ctx* ctx, const int64_t* d_tok_off, const int64_t* d_hash_off,
                         const uint64_t* d_hashes, int32_t n_req, const int32_t* d_placed_off,
                         const int32_t* d_placed, const int32_t* d_admitted,
                         const uint8_t* d_hold, int32_t hold, const int32_t* d_hold_index);
/* FutureRegistry::update (manager.cpp:13-23) for n DISTINCT workflows at once (a burst's
   issue-time updates, engine.cpp:605-609, last write per workflow); max_wf >= every id. */
int pyg_registry_update_batch_dev(pyg_ctx* ctx, int32_t n, const int32_t* d_wf,
                                  const uint64_t* d_mask, int32_t max_wf);
/* Grow the device registry to hold workflow ids 0..max_wf now (synchronizes), so later
   updates never reallocate inside a stream-ordered step. */
int pyg_registry_reserve(pyg_ctx* ctx, int32_t max_wf);

/* ------------------------------------------------------ sharded step (multi-GPU) */
/* With pyg_set_shard, pyg_route_batch_dev routes over the WHOLE cluster: the node table,
   candidate lists and placed CSR ([n_global+1]) use global replica indices, and every shard
   runs the same route over the all-gathered batch (bit-identical decisions everywhere).
   Admission then runs on the owner shard only, over a local batch of the requests placed on
   its replicas (local replica indices), in two calls:
   pyg_admit_shard_dev = start_prefill except the L3 promotion: L1/L2 lookups, eviction, the
   promoted L2 span erase (exported as DirRecords so other shards clear their directory bits
   with pyg_dir_clear_dev / pyg_shard_apply_lists_dev), insert_chain.  d_counts[0] = L2
   records written.
   pyg_shard_l3_resolve_dev = the L3 part, in engine order (engine.cpp:742-746, 806,
   826-828): admission p of this shard sees the live L3 as left by every admission before p.
   The shared L3 (hierarchy.hpp:76-85) is replicated on every shard; call it once the L3
   erase lists of every LOWER shard (lower global replicas = earlier admissions) have been
   applied to this shard's replica (pyg_shard_apply_lists_range_dev).  It lists the chain
   hashes this shard's admissions erase (d_counts[1]) instead of erasing them, writes the
   L3 matches and clamps both counts to their caps (overflow sets device error 4). */
int pyg_admit_shard_dev(pyg_ctx* ctx, const uint64_t* d_tokens, const int64_t* d_tok_off,
                        const int64_t* d_hash_off, const uint64_t* d_hashes,
                        const int32_t* d_wf, const int32_t* d_role, int32_t n_req,
                        const int32_t* d_placed_off, const int32_t* d_placed, double now,
                        int32_t speculative, int32_t* d_admitted, int64_t* d_match3,
                        void* d_l2_erased, int64_t l2_cap, int64_t* d_counts);
int pyg_shard_l3_resolve_dev(pyg_ctx* ctx, const uint64_t* d_tokens, const int64_t* d_tok_off,
                             const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t n_req,
                             const int32_t* d_placed_off, const int32_t* d_placed,
                             const int32_t* d_admitted, int64_t* d_match3,
                             uint64_t* d_l3_hashes, int64_t l3_cap, int64_t l2_cap,
                             int64_t* d_counts);
/* n is an upper bound; d_count (device, optional) holds the actual count (no host sync) */
int pyg_dir_clear_dev(pyg_ctx* ctx, const void* d_records, int64_t n, const int64_t* d_count);
int pyg_l3_erase_hashes_dev(pyg_ctx* ctx, const uint64_t* d_hashes, int64_t n,
                            const int64_t* d_count);
/* dst segment k = src segment idx[k] of a uint64 CSR (packing tokens/hashes of placed
   requests for their owner shard); dst_off is the exclusive scan of the segment lengths. */
int pyg_gather_csr_dev(pyg_ctx* ctx, const uint64_t* d_src, const int64_t* d_src_off,
                       const int64_t* d_idx, int64_t n_idx, const int64_t* d_dst_off,
                       uint64_t* d_dst);

/* ------------------------------------------- peer-memory exchange (NVLink P2P) */
/* One shard's exchange window as seen by the importing process (pointers obtained with
   pyg_ipc_import from the owner's pyg_ipc_export handles).  Inputs of its requests (tokens,
   boundary hashes and their CSR offsets), its receive list (global request indices placed on
   its replicas, ascending, with device count), its admission results in receive order, and its
   exported erase lists (L2 DirRecords, L3 chain hashes; list_counts[0..1]). */
typedef struct {
  const uint64_t* tokens;
  const int64_t* tok_off;
  const uint64_t* hashes;
  const int64_t* hash_off;
  const int32_t* recv_gidx;
  const int64_t* recv_count;
  const int32_t* admitted;
  const int64_t* match3;
  const void* l2_list;
  const uint64_t* l3_list;
  const int64_t* list_counts;
  const int32_t* workflow;      /* lineage of its requests */
  const int32_t* role;
} pyg_peer;

/* CUDA IPC: handle (64 bytes) + offset of the allocation holding d_ptr; import maps it into this
   process once (cached) and returns the device pointer. */
int pyg_ipc_export(const void* d_ptr, void* handle_out, int64_t* offset_out);
int pyg_ipc_import(pyg_ctx* ctx, const void* handle, int64_t offset, void** d_ptr_out);

/* Requests of the burst routed to this shard's replicas (ascending global index) with their
   token / hash offsets in the receive buffers; count stays on the device.  cap bounds the
   count (the prompt tokens placed on a replica never exceed its kv_capacity).  Lineage
   (workflow, role) of the received requests is gathered from the burst-wide arrays. */
int pyg_shard_recv_plan_dev(pyg_ctx* ctx, int32_t R_total, const pyg_decision* d_dec,
                            const pyg_peer* d_peers, int32_t world, const int64_t* d_req_off,
                            int64_t cap, int32_t* d_recv_gidx, int64_t* d_recv_count,
                            int64_t* d_recv_toff, int64_t* d_recv_hoff, int32_t* d_recv_wf,
                            int32_t* d_recv_role);
/* Route inputs of this shard's requests as compact rows for the all-gather: tokens()
   (router.hpp:19-21) and alpha (4 words), candidate group (1 word), staged row as 16-bit
   (staged16 != 0; every prompt < 65536 tokens) or 32-bit values.  unpack rebuilds the
   reservation as {tokens(), 0, alpha, 0}, which routes identically (capacity_holds and
   oom_bound read only tokens() and alpha, router.cpp:7-17). */
int pyg_shard_pack_dev(pyg_ctx* ctx, const pyg_reservation* d_req, const int32_t* d_group,
                       const int32_t* d_staged, int32_t n_req, int32_t max_cand, int32_t staged16,
                       int32_t* d_rows);
int pyg_shard_unpack_dev(pyg_ctx* ctx, const int32_t* d_rows, int32_t n_req, int32_t max_cand,
                         int32_t staged16, pyg_reservation* d_req, int32_t* d_group,
                         int32_t* d_staged);
/* The all-gather's NVLink replacement: rebuilds the whole burst's reservations, groups and
   staged rows straight from every shard's packed rows (d_rows_of[k] = shard k's d_rows as
   mapped in this process; shard k holds requests [d_req_off[k], d_req_off[k+1])). */
int pyg_shard_unpack_peer_dev(pyg_ctx* ctx, const int64_t* d_rows_of, int32_t world,
                              const int64_t* d_req_off, int32_t n_req_total, int32_t max_cand,
                              int32_t staged16, pyg_reservation* d_req, int32_t* d_group,
                              int32_t* d_staged);
/* The same, with the staged rows copied only for requests of the groups in own_mask (bit g =
   group g < 64; 0 = every group): a shard that routes only its own models needs no others. */
int pyg_shard_unpack_peer_own_dev(pyg_ctx* ctx, const int64_t* d_rows_of, int32_t world,
                                  const int64_t* d_req_off, int32_t n_req, int32_t max_cand,
                                  int32_t s16, uint64_t own_mask, pyg_reservation* d_req,
                                  int32_t* d_group, int32_t* d_staged);
/* Cross-GPU stream barrier over peer memory (replaces a one-element NCCL all-reduce).
   signal: after a system-scope fence, writes seq into slot `me` of every shard's flag array
   (d_flag_of[k] = shard k's int64 flags[world], mapped here).  wait: blocks this stream until
   every slot of this shard's own flags (d_flags) is >= seq; a peer that never signals flags a
   device error after ~10 s instead of hanging. */
int pyg_shard_signal_dev(pyg_ctx* ctx, const int64_t* d_flag_of, int32_t world, int32_t me,
                         int64_t seq);
int pyg_shard_wait_dev(pyg_ctx* ctx, const int64_t* d_flags, int32_t world, int64_t seq);
/* Pull the received requests' tokens and hashes from their origin shards (peer loads). */
int pyg_shard_pull_dev(pyg_ctx* ctx, const pyg_peer* d_peers, int32_t world,
                       const int64_t* d_req_off, const int32_t* d_recv_gidx,
                       const int64_t* d_recv_count, const int64_t* d_recv_toff,
                       const int64_t* d_recv_hoff, uint64_t* d_tok_out, int64_t tok_cap,
                       uint64_t* d_hash_out, int64_t hash_cap);
/* Global per-replica placed CSR -> this shard's per-local-replica lists of receive positions. */
int pyg_shard_local_placed_dev(pyg_ctx* ctx, const int32_t* d_placed_off, const int32_t* d_placed,
                               const int32_t* d_recv_gidx, const int64_t* d_recv_count,
                               int32_t* d_p_off, int32_t* d_p_loc);
/* After a cross-GPU barrier: erase every shard's listed L3 hashes from this shard's L3 replica
   and clear the other shards' erased L2 blocks from the directory. */
int pyg_shard_apply_lists_dev(pyg_ctx* ctx, const pyg_peer* d_peers, int32_t world, int32_t me);
/* The same for a subset: L3 erase lists of peers [l3_lo, l3_hi), and (with_l2) the L2
   directory clears of every peer except me. */
/* The first half of the L3 chain for rank me: wait for the L3 lists of ranks < me and apply
   them -- skipped on the device when none of this rank's admissions (the last
   pyg_admit_shard_dev) matched anything in L3, since erasures can only shrink a match. */
int pyg_shard_l3_prepare_dev(pyg_ctx* ctx, const pyg_peer* d_peers, const int64_t* d_flags,
                             int32_t world, int32_t me, int64_t seq);
int pyg_shard_apply_lists_range_dev(pyg_ctx* ctx, const pyg_peer* d_peers, int32_t world,
                                    int32_t me, int32_t l3_lo, int32_t l3_hi, int32_t with_l2);
/* Admission results of this shard's own requests, read from their owner shards. */
int pyg_shard_results_dev(pyg_ctx* ctx, const pyg_peer* d_peers, int32_t world,
                          const int64_t* d_rep_off, const pyg_decision* d_dec, int64_t req_base,
                          int32_t R_local, int32_t* d_admitted, int64_t* d_match3);

/* ------------------------------------------------ K6: next-use from the workflow DAG */
/* One node of a flattened path expression (PathNode, path_expr.hpp:21-38), preorder: every
   node's descendants follow it.  kind: 0 Atom, 1 Seq, 2 Repeat, 3 ParallelFanout,
   4 Optional, 5 Terminal (PathKind order).  Seq children are ch_list[ch_begin..ch_end). */
typedef struct {
  int32_t kind, role, min, max;
  double p_continue, p;
  int32_t child, ch_begin, ch_end, pad;
} pyg_path_node;

/* expected_distance_to(cursor, role) (path_analysis.cpp:553-557) for every cursor and role
   < n_roles, and future_roles(cursor) (path_analysis.cpp:547-551) as role masks.  Cursors are
   PathCursor::frames() as a CSR: frames [d_frame_off[c], d_frame_off[c+1]) of (node id,
   progress), root frame first, atom frame last.  d_dist[c*n_roles + role] = NaN for nullopt.
   Bit-exact FP64 (no contraction). */
int pyg_next_use_dev(pyg_ctx* ctx, const pyg_path_node* d_nodes, int32_t n_nodes,
                     const int32_t* d_ch_list, int32_t n_cursors, const int32_t* d_frame_off,
                     const int32_t* d_frame_node, const int32_t* d_frame_prog, int32_t n_roles,
                     double* d_dist, uint64_t* d_future);
/* Predicted next use of every block of a tier in id order (the pyg_tier_dump order):
   d_dist[d_wf_cursor[block.workflow]*n_roles + block.role], NaN when the workflow has no
   cursor (-1) or the role has no future occurrence.  *d_count = number of blocks. */
int pyg_block_next_use_dev(pyg_ctx* ctx, int32_t replica, int32_t tier, const int32_t* d_wf_cursor,
                           int32_t n_wf, const double* d_dist, int32_t n_roles, double* d_out,
                           int64_t cap, int64_t* d_count);
/* FutureRegistry::update from cursors (engine.cpp:605-609 at issue: future_roles plus the
   current role; engine.cpp:1064-1065 at completion: d_current_role = NULL).  d_cursor[i] = -1
   registers an empty set.  max_wf bounds the workflow ids (registry capacity). */
int pyg_registry_from_cursors_dev(pyg_ctx* ctx, int32_t n, int32_t max_wf, const int32_t* d_wf,
                                  const int32_t* d_cursor, const uint64_t* d_future,
                                  const int32_t* d_current_role);

/* ------------------------------------------------- device prompt assembly (§8f-4) */
/* One segment of assemble_prompt (prompt.cpp:128-164) resolved by the host to a range of a
   device token pool: a Ref into a resident exchange (request / response tokens in HBM), a
   literal's tokenization, or freshly uploaded tokens. */
typedef struct {
  int64_t src;  /* pool offset */
  int64_t len;  /* tokens */
} pyg_segment;

/* Concatenates each request's segments: d_tok_off[n_req+1] (exclusive scan of the request
   lengths) and the token CSR d_tokens, ready for pyg_hash_batch_dev.  Segments of request r
   are d_segs[d_seg_off[r] .. d_seg_off[r+1]). */
int pyg_assemble_dev(pyg_ctx* ctx, int32_t n_req, const int64_t* d_seg_off,
                     const pyg_segment* d_segs, const uint64_t* d_pool, int64_t* d_tok_off,
                     uint64_t* d_tokens);
/* Prompt assembly fused with K1: the same d_tok_off / d_tokens as pyg_assemble_dev, plus
   d_hash_off[n_req+1] (exclusive scan of ceil(len/B)) and the boundary hashes d_hashes of
   pyg_hash_batch_dev (chain_boundary_hashes, hierarchy.cpp:21-30), in one pass over the
   pool: the hashing kernel stages each request's tokens from the pool segments and writes
   them to d_tokens as it hashes.  n_segs = d_seg_off[n_req] and n_tokens >= the total prompt
   length size its work buffers (the host knows both: it built the descriptors); a device
   error is flagged if the batch exceeds them. */
int pyg_assemble_hash_dev(pyg_ctx* ctx, int32_t n_req, const int64_t* d_seg_off,
                          const pyg_segment* d_segs, int64_t n_segs, const uint64_t* d_pool,
                          int64_t n_tokens, int64_t* d_tok_off, uint64_t* d_tokens,
                          int64_t* d_hash_off, uint64_t* d_hashes);

/* ----------------------------------------- worker batch formation / preemption (§8f-3) */
/* sched::QueueItem (worker.hpp:11-16) with the request id replaced by its rank in the
   ids' string order (ties in form_batch / select_preemption_victim break on request_id). */
typedef struct {
  double base_priority;
  double enqueue_time;
  int64_t reservation;
  int64_t id_rank;
} pyg_queue_item;

/* form_batch (worker.cpp:16-37) for n_sets queues at once (one per replica): items of set s
   are d_items[d_off[s] .. d_off[s+1]) (at most 4096); d_order[d_off[s] + k] = index (within
   the set) of the k-th admitted item, d_n_admitted[s] = admitted count. */
int pyg_form_batch_dev(pyg_ctx* ctx, int32_t n_sets, const int64_t* d_off,
                       const pyg_queue_item* d_items, const int64_t* d_active_reservation,
                       const int64_t* d_capacity, double now, double aging_rate, int32_t* d_order,
                       int32_t* d_n_admitted);
/* select_preemption_victim (worker.cpp:39-58) per set; -1 for an empty set. */
int pyg_preemption_victim_dev(pyg_ctx* ctx, int32_t n_sets, const int64_t* d_off,
                              const pyg_queue_item* d_items, double now, double aging_rate,
                              int32_t* d_victim);

/* ------------------------------------------------------ forward staging (§8f-2) */
#define PYG_STAGE_PROMOTE_TO_HOST 0   /* StageAction::Kind (manager.hpp) */
#define PYG_STAGE_BACKGROUND_PREFILL 1
#define PYG_STAGE_SKIP 2
#define PYG_SKIP_NONE 0
#define PYG_SKIP_UNRESOLVED 1         /* Skip reasons (manager.cpp:70-96) */
#define PYG_SKIP_ALREADY_STAGED 2
#define PYG_SKIP_GPU_BUSY 3
#define PYG_SKIP_NO_REPLICA 4         /* no ready replica of the model (engine.cpp:1150) */

typedef struct {
  int32_t target;  /* replica index of this ctx (-1: none) */
  int32_t kind;
  int32_t reason;
  int32_t pad;
  int64_t from, to;
} pyg_stage_action;

/* Batched forward staging for successor prefixes (tokens CSR + boundary hashes): target =
   ready candidate with the largest L2 prefix, ties to the lowest replica id (engine.cpp
   fire_prefetch :1137-1166); action from lookup(prefix, &l3) on it (on_prefetch_requested,
   manager.cpp:60-100).  d_gpu_idle[replica] = active and pool both empty. */
int pyg_stage_plan_dev(pyg_ctx* ctx, const uint64_t* d_tokens, const int64_t* d_tok_off,
                       const int64_t* d_hash_off, const uint64_t* d_hashes, int32_t n_prefix,
                       const int32_t* d_group, int32_t n_groups, const int32_t* d_cand_off,
                       const int32_t* d_cand, int32_t max_cand, const int32_t* d_replica_id,
                       const int8_t* d_gpu_idle, pyg_stage_action* d_out);

/* ------------------------------------------------- host-buffer batch entry */
/* The drop-in batch call for a C++ engine: host arrays in, host arrays out.  Copies the batch
   to the device (pinned host memory is fastest), runs K1..K5 exactly as the _dev sequence
   hash -> staged -> route -> admit [-> release] does, copies the results back, synchronizes. */
typedef struct {
  int32_t n_req;
  int32_t reserved;
  const uint64_t* tokens;       /* CSR by tok_off */
  const int64_t* tok_off;       /* [n_req+1] */
  const pyg_reservation* req;   /* [n_req] */
  const int32_t* group;         /* [n_req] candidate group (model) */
  const int32_t* workflow;      /* [n_req] interned lineage */
  const int32_t* role;          /* [n_req] */
} pyg_batch_host;

typedef struct {
  const int32_t* replica_id;    /* [n_rep] */
  const int64_t* kv_capacity;   /* [n_rep] */
  const int64_t* asg_off;       /* [n_rep+1] */
  const pyg_reservation* asg;
  int32_t n_groups;
  int32_t reserved;
  const int32_t* cand_off;      /* [n_groups+1] */
  const int32_t* cand;
} pyg_nodes_host;

int pyg_step_host(pyg_ctx* ctx, const pyg_batch_host* batch, const pyg_nodes_host* nodes,
                  int32_t mode, double epsilon, double now, int32_t speculative, int32_t release,
                  pyg_decision* out_decisions, int32_t* out_admitted, int64_t* out_match3);

/* device error flag set by batched kernels (capacity overflow etc.); reads and clears it */
int pyg_check_device_error(pyg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
