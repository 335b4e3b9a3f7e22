// ref_shim.cpp -- extern "C" driver over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources where they lie under /root/reference/proj/src (nothing is
// copied into this repo) into oracle/_ref/libpythia_ref{16,64}.so.  The B=16
// flavour sees a generated copy of hierarchy.hpp with kBlockTokens = 16
// (written to oracle/_ref/overlay16/, git-ignored).
//
// Used by tests/ to pin the C restatement (oracle/pyg_oracle.c) against the
// reference itself, by tests/golden/make_golden.py to emit golden vectors, and
// by bench.py --impl reference as the reference CPU arm.
//
// Lineage ints are turned into the strings "w<k>" / "r<k>"; FutureRegistry
// masks into sets of those role names.

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "pythia/cache/hierarchy.hpp"
#include "pythia/cache/manager.hpp"
#include "pythia/sched/router.hpp"
#include "pythia/sched/worker.hpp"
#include "pythia/workflow/path_analysis.hpp"
#include "pythia/workflow/path_expr.hpp"
#include "pythia/workflow/prompt.hpp"

using namespace pythia;
using cache::CacheHierarchy;
using cache::SharedL3;
using cache::Tier;

namespace {
std::string wf_name(int32_t w) { return "w" + std::to_string(w); }
std::string role_name(int32_t r) { return "r" + std::to_string(r); }
int32_t parse_int(const std::string& s) { return s.size() > 1 ? std::stoi(s.substr(1)) : -1; }
Tier to_tier(int32_t t) { return t == 0 ? Tier::L1 : (t == 1 ? Tier::L2 : Tier::L3); }
std::set<std::string> mask_roles(uint64_t m) {
  std::set<std::string> s;
  for (int i = 0; i < 64; ++i)
    if ((m >> i) & 1u) s.insert(role_name(i));
  return s;
}
workflow::TokenSeq seq_of(const uint64_t* t, int64_t n) { return workflow::TokenSeq(t, t + n); }
}  // namespace

struct pref_block {
  uint64_t id, hash;
  int64_t s, e;
  int32_t wf, role;
  double la;
  int32_t pin;
  int32_t alive;
};

struct pref_res {
  int64_t prompt_len, upper;
  double alpha;
  int64_t tokens_generated;
};

struct pref_decision {
  int32_t target;
  int32_t tiebreak;
  int64_t headroom;
  double oom_bound;
};

extern "C" {

int64_t pref_block_tokens() { return cache::kBlockTokens; }

uint64_t pref_fnv1a_str(const char* s, int64_t n) {
  return workflow::fnv1a(std::string_view(s, static_cast<size_t>(n)));
}
uint64_t pref_fnv1a_u64(uint64_t v, uint64_t h) { return workflow::fnv1a(v, h); }
uint64_t pref_response_token(const char* rid, int64_t index) {
  return workflow::response_token(rid, static_cast<size_t>(index));
}

int64_t pref_chain_hashes(const uint64_t* tokens, int64_t n, uint64_t* out) {
  auto h = cache::chain_boundary_hashes(seq_of(tokens, n));
  if (out) std::memcpy(out, h.data(), h.size() * sizeof(uint64_t));
  return static_cast<int64_t>(h.size());
}

// ---- CacheHierarchy / SharedL3 ----
void* pref_cache_new(int64_t l1, int64_t l2) { return new CacheHierarchy(l1, l2); }
void pref_cache_free(void* c) { delete static_cast<CacheHierarchy*>(c); }
void* pref_cache_clone(void* c) { return new CacheHierarchy(*static_cast<CacheHierarchy*>(c)); }
void* pref_l3_new() { return new SharedL3(); }
void pref_l3_free(void* l) { delete static_cast<SharedL3*>(l); }
void* pref_l3_clone(void* l) { return new SharedL3(*static_cast<SharedL3*>(l)); }

static cache::TierStore& store_of(void* c, void* l3, int32_t tier) {
  if (tier == 2 && l3) return static_cast<SharedL3*>(l3)->store();
  return static_cast<CacheHierarchy*>(c)->tier(to_tier(tier));
}

void pref_lookup(void* c, void* l3, const uint64_t* tokens, int64_t n, int64_t out[3]) {
  auto m = static_cast<CacheHierarchy*>(c)->lookup(seq_of(tokens, n),
                                                    static_cast<SharedL3*>(l3));
  out[0] = m.l1;
  out[1] = m.l2;
  out[2] = m.l3;
}

int64_t pref_matched_prefix(void* c, void* l3, int32_t tier, const uint64_t* tokens, int64_t n) {
  auto seq = seq_of(tokens, n);
  auto h = cache::chain_boundary_hashes(seq);
  return store_of(c, l3, tier).matched_prefix(seq, h);
}

void pref_insert_chain(void* c, int32_t tier, const uint64_t* tokens, int64_t n, int64_t upto,
                       int32_t wf, int32_t role, double now, int32_t pin) {
  static_cast<CacheHierarchy*>(c)->insert_chain(to_tier(tier), seq_of(tokens, n), upto,
                                                {wf_name(wf), role_name(role)}, now, pin);
}

void pref_unpin_chain(void* c, const uint64_t* tokens, int64_t n, int64_t upto) {
  static_cast<CacheHierarchy*>(c)->unpin_chain(seq_of(tokens, n), upto);
}

uint64_t pref_tier_put(void* c, void* l3, int32_t tier, uint64_t hash, int64_t s, int64_t e,
                       int32_t wf, int32_t role, double now, int32_t pin) {
  uint64_t* ctr = (tier == 2 && l3) ? static_cast<SharedL3*>(l3)->id_counter()
                                    : static_cast<CacheHierarchy*>(c)->id_counter();
  return store_of(c, l3, tier).put(hash, s, e, {wf_name(wf), role_name(role)}, now, pin, ctr);
}

void pref_tier_erase(void* c, void* l3, int32_t tier, uint64_t id) {
  store_of(c, l3, tier).erase(id);
}

int64_t pref_tier_occupancy(void* c, void* l3, int32_t tier) {
  return store_of(c, l3, tier).occupancy();
}

int64_t pref_tier_dump(void* c, void* l3, int32_t tier, pref_block* out, int64_t cap) {
  const auto& blocks = store_of(c, l3, tier).blocks();
  int64_t k = 0;
  for (const auto& [id, b] : blocks) {
    if (out && k < cap) {
      out[k] = {b.block_id, b.chain_hash, b.span_start, b.span_end,
                parse_int(b.lineage.workflow_id), parse_int(b.lineage.role_id),
                b.last_access, b.pin_count, 1};
    }
    ++k;
  }
  return k;
}

void pref_add_decode_tokens(void* c, int64_t n) {
  static_cast<CacheHierarchy*>(c)->add_decode_tokens(n);
}
int64_t pref_l1_occupancy(void* c) { return static_cast<CacheHierarchy*>(c)->l1_occupancy(); }

// ---- FutureRegistry ----
void* pref_registry_new() { return new cache::FutureRegistry(); }
void pref_registry_free(void* r) { delete static_cast<cache::FutureRegistry*>(r); }
void pref_registry_update(void* r, int32_t wf, uint64_t mask) {
  static_cast<cache::FutureRegistry*>(r)->update(wf_name(wf), mask_roles(mask));
}
void pref_registry_drop(void* r, int32_t wf) {
  static_cast<cache::FutureRegistry*>(r)->drop(wf_name(wf));
}

// ---- evict_for_space ----
int32_t pref_evict(void* c, int32_t tier, int64_t needed, void* reg, int32_t speculative,
                   uint64_t* out_ids, int64_t cap, int64_t* n_freed, int64_t* freed_tokens) {
  auto res = cache::evict_for_space(*static_cast<CacheHierarchy*>(c), to_tier(tier), needed,
                                    *static_cast<cache::FutureRegistry*>(reg), speculative != 0);
  int64_t k = 0;
  for (uint64_t id : res.freed) {
    if (out_ids && k < cap) out_ids[k] = id;
    ++k;
  }
  *n_freed = k;
  *freed_tokens = res.freed_tokens;
  return res.satisfied ? 1 : 0;
}

// ---- router ----
pref_decision pref_route(int32_t n_nodes, const int32_t* replica_id, const int64_t* kv_capacity,
                         const int64_t* asg_off, const pref_res* asg, const int64_t* staged,
                         const pref_res* req, double epsilon) {
  std::vector<sched::NodeView> nodes(static_cast<size_t>(n_nodes));
  for (int32_t n = 0; n < n_nodes; ++n) {
    nodes[n].replica_id = replica_id[n];
    nodes[n].kv_capacity = kv_capacity[n];
    nodes[n].staged_l2_prefix = staged[n];
    for (int64_t i = asg_off[n]; i < asg_off[n + 1]; ++i) {
      nodes[n].assigned.push_back({asg[i].prompt_len, asg[i].upper, asg[i].alpha,
                                   asg[i].tokens_generated});
    }
  }
  sched::Reservation r{req->prompt_len, req->upper, req->alpha, req->tokens_generated};
  auto d = sched::route(nodes, r, epsilon);
  pref_decision out{};
  out.target = d.target ? *d.target : -1;
  out.tiebreak = d.cache_tiebreak_used ? 1 : 0;
  out.headroom = d.headroom;
  out.oom_bound = d.oom_bound;
  return out;
}

int32_t pref_route_least_outstanding(int32_t n_nodes, const int32_t* replica_id,
                                     const int64_t* asg_off) {
  std::vector<sched::NodeView> nodes(static_cast<size_t>(n_nodes));
  for (int32_t n = 0; n < n_nodes; ++n) {
    nodes[n].replica_id = replica_id[n];
    nodes[n].assigned.resize(static_cast<size_t>(asg_off[n + 1] - asg_off[n]));
  }
  auto t = sched::route_least_outstanding(nodes);
  return t ? *t : -1;
}

// ---- path analysis (host-side workflow ingestion; used to derive future masks) ----
// history is a list of role names separated by ','; returns -1 if the history
// cannot be located.  Role names must be "r<k>" with k < 64.
int64_t pref_future_mask(const char* expr, const char* history, uint64_t* mask_out) {
  auto e = std::make_shared<const workflow::PathExpr>(workflow::parse_path_expr(expr));
  std::vector<std::string> h;
  std::string cur;
  for (const char* p = history;; ++p) {
    if (*p == ',' || *p == '\0') {
      if (!cur.empty()) h.push_back(cur);
      cur.clear();
      if (*p == '\0') break;
    } else {
      cur.push_back(*p);
    }
  }
  auto pos = workflow::locate_position(*e, h);
  if (!pos) return -1;
  uint64_t m = 0;
  for (const auto& r : workflow::future_roles(*pos)) {
    int32_t k = parse_int(r);
    if (k >= 0 && k < 64) m |= uint64_t{1} << k;
  }
  *mask_out = m;
  return 0;
}

// expected_distance_to (path_analysis.cpp:553-557); returns 0 and writes the
// distance, 1 if nullopt, -1 if the history cannot be located.
int64_t pref_expected_distance(const char* expr, const char* history, const char* role,
                               double* out) {
  auto e = std::make_shared<const workflow::PathExpr>(workflow::parse_path_expr(expr));
  std::vector<std::string> h;
  std::string cur;
  for (const char* p = history;; ++p) {
    if (*p == ',' || *p == '\0') {
      if (!cur.empty()) h.push_back(cur);
      cur.clear();
      if (*p == '\0') break;
    } else {
      cur.push_back(*p);
    }
  }
  auto pos = workflow::locate_position(*e, h);
  if (!pos) return -1;
  auto d = workflow::expected_distance_to(*pos, role);
  if (!d) return 1;
  *out = *d;
  return 0;
}

// ---- completion (manager.cpp:25-58) with an explicit future mask ----
// Builds the action list the way on_request_complete does, but from a mask
// instead of a PathCursor, then runs the reference apply_completion.  The
// cursor-driven variant is pref_complete_expr below.
int64_t pref_complete_mask(void* c, void* l3, int32_t wf, uint64_t future_mask, double now) {
  auto* cache = static_cast<CacheHierarchy*>(c);
  std::set<std::string> future = mask_roles(future_mask);
  std::vector<cache::CompletionAction> actions;
  for (Tier t : {Tier::L1, Tier::L2}) {
    for (const auto& [id, block] : cache->tier(t).blocks()) {
      if (block.pinned()) continue;
      if (block.lineage.workflow_id != wf_name(wf)) continue;
      actions.push_back({future.count(block.lineage.role_id)
                             ? cache::CompletionAction::Kind::RetainAndWriteL3
                             : cache::CompletionAction::Kind::Free,
                         t, id});
    }
  }
  cache::apply_completion(actions, *cache, *static_cast<SharedL3*>(l3), now);
  return static_cast<int64_t>(actions.size());
}

// Cursor-driven: the reference on_request_complete on a real envelope.
int64_t pref_complete_expr(void* c, void* l3, int32_t wf, const char* expr, const char* history,
                           double now) {
  auto e = std::make_shared<const workflow::PathExpr>(workflow::parse_path_expr(expr));
  std::vector<std::string> h;
  std::string cur;
  for (const char* p = history;; ++p) {
    if (*p == ',' || *p == '\0') {
      if (!cur.empty()) h.push_back(cur);
      cur.clear();
      if (*p == '\0') break;
    } else {
      cur.push_back(*p);
    }
  }
  auto pos = workflow::locate_position(*e, h);
  if (!pos) return -1;
  workflow::RequestEnvelope env;
  env.request_id = "req";
  env.app_metadata = {"t", wf_name(wf), h.back()};
  env.sys_annotations = workflow::SysAnnotations{};
  env.sys_annotations->path_regex = e;
  env.position = *pos;
  auto* cache = static_cast<CacheHierarchy*>(c);
  auto actions = cache::on_request_complete(env, *cache);
  cache::apply_completion(actions, *cache, *static_cast<SharedL3*>(l3), now);
  return static_cast<int64_t>(actions.size());
}

// L3 dead-lineage sweep of apply_completion_policy (engine.cpp:1074-1080).
void pref_l3_dead_sweep(void* l3, int32_t wf, uint64_t future_mask) {
  auto& store = static_cast<SharedL3*>(l3)->store();
  std::set<std::string> future = mask_roles(future_mask);
  std::vector<uint64_t> dead;
  for (const auto& [id, block] : store.blocks()) {
    if (block.lineage.workflow_id == wf_name(wf) && !future.count(block.lineage.role_id)) {
      dead.push_back(id);
    }
  }
  for (uint64_t id : dead) store.erase(id);
}

// erase_chain_span (engine.cpp:849-861 is a private static of the engine; this is the same
// loop over the public TierStore API).
void pref_erase_chain_span(void* c, void* l3, int32_t tier, const uint64_t* tokens, int64_t n,
                           int64_t from, int64_t to) {
  auto& store = store_of(c, l3, tier);
  auto hashes = cache::chain_boundary_hashes(seq_of(tokens, n));
  for (size_t i = 0; i < hashes.size(); ++i) {
    int64_t span_end = std::min<int64_t>(static_cast<int64_t>(i + 1) * cache::kBlockTokens, n);
    if (span_end <= from || span_end > to) continue;
    if (const cache::CacheBlock* b = store.find_chain(hashes[i])) {
      if (!b->pinned()) store.erase(b->block_id);
    }
  }
}

// One burst of R requests through the reference engine's hot-path call
// pattern (the CPU baseline of bench.py; same contract as pyg_step_host):
//   node_view per candidate: staged = cache.lookup(prompt, nullptr).l2   engine.cpp:640-648
//   sched::route in issue order; SEQ_COMMIT pushes to the pool first     engine.cpp:650-692
//   per replica, per placed request: start_prefill cache side            engine.cpp:799-829
//     (one at a time against the live L3, as the engine's admit_on loop)
//   release: unpin_chain(seq, len)                                        hierarchy.cpp:132-142
// Returns the number of placed requests.
int64_t pref_step(void** caches, int32_t n_rep, void* l3v, void* regv, int32_t spec,
                  const uint64_t* tokens, const int64_t* tok_off, int32_t R, const pref_res* res,
                  const int32_t* group, const int32_t* wf, const int32_t* role,
                  const int32_t* replica_id, const int64_t* kv_cap, const int64_t* asg_off,
                  const pref_res* asg, const int32_t* cand_off, const int32_t* cand, int32_t mode,
                  double eps, double now, int32_t release, pref_decision* out_dec,
                  int32_t* out_adm) {
  auto* l3 = static_cast<SharedL3*>(l3v);
  auto* reg = static_cast<cache::FutureRegistry*>(regv);
  std::vector<std::vector<sched::Reservation>> pools(static_cast<size_t>(n_rep));
  for (int n = 0; n < n_rep; ++n)
    for (int64_t k = asg_off[n]; k < asg_off[n + 1]; ++k)
      pools[n].push_back({asg[k].prompt_len, asg[k].upper, asg[k].alpha, asg[k].tokens_generated});
  std::vector<std::vector<int32_t>> placed(static_cast<size_t>(n_rep));
  int64_t n_placed = 0;
  for (int32_t r = 0; r < R; ++r) {
    workflow::TokenSeq prompt(tokens + tok_off[r], tokens + tok_off[r + 1]);
    const int g = group[r];
    std::vector<sched::NodeView> views;
    for (int32_t j = cand_off[g]; j < cand_off[g + 1]; ++j) {
      const int n = cand[j];
      sched::NodeView v;
      v.replica_id = replica_id[n];
      v.kv_capacity = kv_cap[n];
      v.assigned = pools[n];
      v.staged_l2_prefix = static_cast<CacheHierarchy*>(caches[n])->lookup(prompt, nullptr).l2;
      views.push_back(std::move(v));
    }
    sched::Reservation q{res[r].prompt_len, res[r].upper, res[r].alpha, res[r].tokens_generated};
    auto d = sched::route(views, q, eps);
    pref_decision od{};
    od.target = d.target ? *d.target : -1;
    od.tiebreak = d.cache_tiebreak_used;
    od.headroom = d.headroom;
    od.oom_bound = d.oom_bound;
    if (out_dec) out_dec[r] = od;
    if (out_adm) out_adm[r] = 0;
    if (d.target) {
      for (int32_t j = cand_off[g]; j < cand_off[g + 1]; ++j) {
        if (replica_id[cand[j]] == *d.target) {
          if (mode == 1) pools[cand[j]].push_back(q);
          placed[cand[j]].push_back(r);
          ++n_placed;
          break;
        }
      }
    }
  }
  std::vector<std::pair<int, int32_t>> admitted;
  for (int n = 0; n < n_rep; ++n) {
    auto* c = static_cast<CacheHierarchy*>(caches[n]);
    for (int32_t r : placed[n]) {
      workflow::TokenSeq seq(tokens + tok_off[r], tokens + tok_off[r + 1]);
      const int64_t len = static_cast<int64_t>(seq.size());
      auto m = c->lookup(seq, l3);  // live L3, as start_prefill (engine.cpp:806)
      auto ev = cache::evict_for_space(*c, Tier::L1, len - m.l1, *reg, spec != 0);
      if (!ev.satisfied) continue;
      const int64_t reusable = std::max({m.l1, m.l2, m.l3});
      const int64_t l2_part = std::max<int64_t>(std::min(reusable, m.l2) - m.l1, 0);
      const int64_t l3_part = std::max<int64_t>(reusable - std::max(m.l1, m.l2), 0);
      if (l2_part > 0) pref_erase_chain_span(c, nullptr, 1, seq.data(), len, m.l1, m.l1 + l2_part);
      if (l3_part > 0)
        pref_erase_chain_span(c, l3, 2, seq.data(), len, std::max(m.l1, m.l2), reusable);
      c->insert_chain(Tier::L1, seq, len, {wf_name(wf[r]), role_name(role[r])}, now, +1);
      if (out_adm) out_adm[r] = 1;
      admitted.emplace_back(n, r);
    }
  }
  if (release) {  // after every admission, as pyg_release_batch_dev
    for (auto [n, r] : admitted) {
      workflow::TokenSeq seq(tokens + tok_off[r], tokens + tok_off[r + 1]);
      static_cast<CacheHierarchy*>(caches[n])->unpin_chain(seq, static_cast<int64_t>(seq.size()));
    }
  }
  return n_placed;
}

// One burst of the steady-state bench (paper_2604_25899_b200/steady.py, bench.py): the
// reference engine's hot-path calls for a burst of R requests, with
//   - the node table given as a CSR (background load + earlier bursts' placements, pool
//     order), routed in issue order with sequential commit (engine.cpp:650-692);
//   - staged values: hash_once == 0 -> cache.lookup(prompt, nullptr).l2 per candidate, the
//     engine's node_view (engine.cpp:640-648, one rehash per candidate); hash_once != 0 ->
//     chain_boundary_hashes once + tier(L2).matched_prefix per candidate (hierarchy.hpp:44,
//     64-65: the same reference functions without the repeated hashing).  Computed over
//     n_threads host threads: nothing mutates L2 while a burst routes, so every order gives
//     the same values;
//   - admission per replica in placement order against the live L3 (engine.cpp:742-746,
//     799-829);
//   - no release: pref_release unpins an earlier burst.
// out_m3 [3R] (optional) = the admission lookups; out_staged [R * max_cand] (optional).
int64_t pref_burst(void** caches, int32_t n_rep, void* l3v, void* regv, int32_t spec,
                   const uint64_t* tokens, const int64_t* tok_off, int32_t R, const pref_res* res,
                   const int32_t* group, const int32_t* wf, const int32_t* role,
                   const int32_t* replica_id, const int64_t* kv_cap, const int64_t* asg_off,
                   const pref_res* asg, const int32_t* cand_off, const int32_t* cand,
                   int32_t n_groups, double eps, double now, int32_t hash_once,
                   int32_t n_threads, pref_decision* out_dec, int32_t* out_adm, int64_t* out_m3,
                   int32_t* out_staged) {
  auto* l3 = static_cast<SharedL3*>(l3v);
  auto* reg = static_cast<cache::FutureRegistry*>(regv);
  int32_t max_cand = 1;
  for (int g = 0; g < n_groups; ++g) max_cand = std::max(max_cand, cand_off[g + 1] - cand_off[g]);
  std::vector<int32_t> staged(static_cast<size_t>(R) * max_cand, 0);
  auto stage = [&](int32_t lo, int32_t hi) {
    for (int32_t r = lo; r < hi; ++r) {
      workflow::TokenSeq prompt(tokens + tok_off[r], tokens + tok_off[r + 1]);
      const int g = group[r];
      if (g < 0 || g >= n_groups) continue;
      std::vector<uint64_t> hs;
      if (hash_once) hs = cache::chain_boundary_hashes(prompt);
      for (int32_t j = cand_off[g]; j < cand_off[g + 1]; ++j) {
        const auto* c = static_cast<const CacheHierarchy*>(caches[cand[j]]);
        const int64_t v = hash_once ? c->tier(Tier::L2).matched_prefix(prompt, hs)
                                    : c->lookup(prompt, nullptr).l2;
        staged[static_cast<size_t>(r) * max_cand + (j - cand_off[g])] = static_cast<int32_t>(v);
      }
    }
  };
  const int nt = std::max(1, std::min<int32_t>(n_threads, std::max(1, R / 64)));
  if (nt == 1) {
    stage(0, R);
  } else {
    std::vector<std::thread> th;
    std::atomic<int32_t> next{0};
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&] {
        for (;;) {
          const int32_t a = next.fetch_add(64);
          if (a >= R) break;
          stage(a, std::min(R, a + 64));
        }
      });
    for (auto& x : th) x.join();
  }
  if (out_staged) std::memcpy(out_staged, staged.data(), staged.size() * sizeof(int32_t));
  std::vector<std::vector<sched::Reservation>> pools(static_cast<size_t>(n_rep));
  for (int n = 0; n < n_rep; ++n)
    for (int64_t k = asg_off[n]; k < asg_off[n + 1]; ++k)
      pools[n].push_back({asg[k].prompt_len, asg[k].upper, asg[k].alpha, asg[k].tokens_generated});
  std::vector<std::vector<int32_t>> placed(static_cast<size_t>(n_rep));
  int64_t n_placed = 0;
  for (int32_t r = 0; r < R; ++r) {
    const int g = group[r];
    std::vector<sched::NodeView> views;
    if (g >= 0 && g < n_groups) {
      for (int32_t j = cand_off[g]; j < cand_off[g + 1]; ++j) {
        const int n = cand[j];
        sched::NodeView v;
        v.replica_id = replica_id[n];
        v.kv_capacity = kv_cap[n];
        v.assigned = pools[n];
        v.staged_l2_prefix = staged[static_cast<size_t>(r) * max_cand + (j - cand_off[g])];
        views.push_back(std::move(v));
      }
    }
    sched::Reservation q{res[r].prompt_len, res[r].upper, res[r].alpha, res[r].tokens_generated};
    auto d = sched::route(views, q, eps);
    pref_decision od{};
    od.target = d.target ? *d.target : -1;
    od.tiebreak = d.cache_tiebreak_used;
    od.headroom = d.headroom;
    od.oom_bound = d.oom_bound;
    if (out_dec) out_dec[r] = od;
    if (out_adm) out_adm[r] = 0;
    if (out_m3) out_m3[3 * r] = out_m3[3 * r + 1] = out_m3[3 * r + 2] = 0;
    if (d.target) {
      for (int32_t j = cand_off[g]; j < cand_off[g + 1]; ++j) {
        if (replica_id[cand[j]] == *d.target) {
          pools[cand[j]].push_back(q);
          placed[cand[j]].push_back(r);
          ++n_placed;
          break;
        }
      }
    }
  }
  for (int n = 0; n < n_rep; ++n) {
    auto* c = static_cast<CacheHierarchy*>(caches[n]);
    for (int32_t r : placed[n]) {
      workflow::TokenSeq seq(tokens + tok_off[r], tokens + tok_off[r + 1]);
      const int64_t len = static_cast<int64_t>(seq.size());
      auto m = c->lookup(seq, l3);
      if (out_m3) {
        out_m3[3 * r] = m.l1;
        out_m3[3 * r + 1] = m.l2;
        out_m3[3 * r + 2] = m.l3;
      }
      auto ev = cache::evict_for_space(*c, Tier::L1, len - m.l1, *reg, spec != 0);
      if (!ev.satisfied) continue;
      const int64_t reusable = std::max({m.l1, m.l2, m.l3});
      const int64_t l2_part = std::max<int64_t>(std::min(reusable, m.l2) - m.l1, 0);
      const int64_t l3_part = std::max<int64_t>(reusable - std::max(m.l1, m.l2), 0);
      if (l2_part > 0) pref_erase_chain_span(c, nullptr, 1, seq.data(), len, m.l1, m.l1 + l2_part);
      if (l3_part > 0)
        pref_erase_chain_span(c, l3, 2, seq.data(), len, std::max(m.l1, m.l2), reusable);
      c->insert_chain(Tier::L1, seq, len, {wf_name(wf[r]), role_name(role[r])}, now, +1);
      if (out_adm) out_adm[r] = 1;
    }
  }
  return n_placed;
}

// unpin_chain(seq, len) of every admitted request of an earlier burst on its replica
// (hierarchy.cpp:132-142); rep[r] = replica index or -1.
void pref_release(void** caches, const uint64_t* tokens, const int64_t* tok_off, int32_t R,
                  const int32_t* rep, const int32_t* admitted) {
  for (int32_t r = 0; r < R; ++r) {
    if (rep[r] < 0 || !admitted[r]) continue;
    workflow::TokenSeq seq(tokens + tok_off[r], tokens + tok_off[r + 1]);
    static_cast<CacheHierarchy*>(caches[rep[r]])->unpin_chain(seq, static_cast<int64_t>(seq.size()));
  }
}

// assemble_prompt / assemble_resolvable_prefix (prompt.cpp:128-164) of a template in the
// reference's placeholder text form (parse_prompt_template, prompt.cpp:75-101) over a
// MapPromptHistory of n_ex exchanges (ids '\n'-separated; request / response token CSRs).
// prefix != 0: the resolvable prefix.  Returns 0 and the tokens (*n_out, up to cap written),
// 1 when assemble_prompt returns nullopt, -1 on a template parse error.
int pref_assemble(const char* text, int32_t n_ex, const char* ids, const int64_t* req_off,
                  const uint64_t* req_tok, const int64_t* resp_off, const uint64_t* resp_tok,
                  int32_t prefix, uint64_t* out, int64_t cap, int64_t* n_out,
                  int32_t* complete) {
  workflow::PromptTemplate t;
  try {
    t = workflow::parse_prompt_template(text);
  } catch (const std::exception&) {
    return -1;
  }
  workflow::MapPromptHistory h;
  std::string all(ids);
  size_t pos = 0;
  for (int32_t k = 0; k < n_ex; ++k) {
    const size_t nl = all.find('\n', pos);
    const std::string id = all.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
    pos = nl == std::string::npos ? all.size() : nl + 1;
    workflow::Exchange ex;
    ex.request.assign(req_tok + req_off[k], req_tok + req_off[k + 1]);
    ex.response.assign(resp_tok + resp_off[k], resp_tok + resp_off[k + 1]);
    h.entries[id] = std::move(ex);
  }
  workflow::TokenSeq seq;
  if (prefix) {
    auto r = workflow::assemble_resolvable_prefix(t, h);
    seq = std::move(r.tokens);
    if (complete) *complete = r.complete ? 1 : 0;
  } else {
    auto r = workflow::assemble_prompt(t, h);
    if (!r) return 1;
    seq = std::move(*r);
    if (complete) *complete = 1;
  }
  *n_out = static_cast<int64_t>(seq.size());
  if (out) std::memcpy(out, seq.data(), std::min<int64_t>(cap, *n_out) * sizeof(uint64_t));
  return 0;
}

// ---- path analysis over a flattened tree (preorder node arrays, the layout of
// pyg_path_node in include/pyg.h): builds the reference PathExpr, locates a history
// with locate_position (path_analysis.cpp), and evaluates expected_distance_to /
// future_roles there.  Frames come back as preorder node ids.
struct pref_path_node {
  int32_t kind, role, min, max;
  double p_continue, p;
  int32_t child, ch_begin, ch_end, pad;
};

namespace {
workflow::PathNodePtr build_node(const pref_path_node* n, const int32_t* ch, int32_t i) {
  const pref_path_node& x = n[i];
  switch (x.kind) {
    case 0: return workflow::PathNode::atom(role_name(x.role));
    case 1: {
      std::vector<workflow::PathNodePtr> kids;
      for (int32_t k = x.ch_begin; k < x.ch_end; ++k) kids.push_back(build_node(n, ch, ch[k]));
      return workflow::PathNode::seq(std::move(kids));
    }
    case 2: return workflow::PathNode::repeat(build_node(n, ch, x.child), x.min, x.max, x.p_continue);
    case 3: return workflow::PathNode::fanout(build_node(n, ch, x.child), x.min, x.max);
    case 4: return workflow::PathNode::optional(build_node(n, ch, x.child), x.p);
    default: return workflow::PathNode::terminal();
  }
}

void preorder_ids(const workflow::PathNode* node, std::map<const workflow::PathNode*, int32_t>& ids) {
  const int32_t id = static_cast<int32_t>(ids.size());
  ids[node] = id;
  if (node->kind == workflow::PathKind::Seq) {
    for (const auto& c : node->children) preorder_ids(c.get(), ids);
  } else if (node->child) {
    preorder_ids(node->child.get(), ids);
  }
}

std::vector<std::string> history_of(const int32_t* h, int32_t n) {
  std::vector<std::string> out;
  for (int32_t i = 0; i < n; ++i) out.push_back(role_name(h[i]));
  return out;
}
}  // namespace

extern "C" {

void* pref_path_build(const pref_path_node* nodes, const int32_t* ch_list, int32_t root) {
  try {
    return new workflow::PathExpr(build_node(nodes, ch_list, root));
  } catch (...) {
    return nullptr;
  }
}

void pref_path_free(void* e) { delete static_cast<workflow::PathExpr*>(e); }

// Frames of locate_position(history) as (preorder id, progress); returns the frame count,
// -1 if the history cannot be located.
int32_t pref_path_locate(void* e, const int32_t* hist, int32_t n_hist, int32_t* frame_node,
                         int32_t* frame_prog, int32_t cap) {
  auto* ex = static_cast<workflow::PathExpr*>(e);
  auto pos = workflow::locate_position(*ex, history_of(hist, n_hist));
  if (!pos) return -1;
  std::map<const workflow::PathNode*, int32_t> ids;
  preorder_ids(ex->root().get(), ids);
  const auto& fr = pos->frames();
  const int32_t nf = static_cast<int32_t>(fr.size());
  for (int32_t i = 0; i < nf && i < cap; ++i) {
    frame_node[i] = ids.at(fr[i].node);
    frame_prog[i] = fr[i].progress;
  }
  return nf;
}

// expected_distance_to at the located position: 0 = value written, 1 = nullopt, -1 = history
// not locatable.  *future_mask = future_roles as a role bitmask.
int32_t pref_path_distance(void* e, const int32_t* hist, int32_t n_hist, int32_t role,
                           double* out, uint64_t* future_mask) {
  auto* ex = static_cast<workflow::PathExpr*>(e);
  auto pos = workflow::locate_position(*ex, history_of(hist, n_hist));
  if (!pos) return -1;
  if (future_mask) {
    uint64_t m = 0;
    for (const auto& r : workflow::future_roles(*pos)) {
      int32_t k = parse_int(r);
      if (k >= 0 && k < 64) m |= uint64_t{1} << k;
    }
    *future_mask = m;
  }
  auto d = workflow::expected_distance_to(*pos, role_name(role));
  if (!d) return 1;
  *out = *d;
  return 0;
}

}  // extern "C"
// ---- worker batch formation / preemption (sched/worker.cpp) over plain arrays; request ids
// are "q%08lld" of the given rank, so string order == rank order.
int64_t pref_form_batch(int32_t n, const double* base, const double* enq, const int64_t* res,
                        const int64_t* id_rank, int64_t active_reservation, int64_t capacity,
                        double now, double aging, int32_t* out) {
  std::vector<sched::QueueItem> pool(n);
  char buf[32];
  for (int32_t i = 0; i < n; ++i) {
    std::snprintf(buf, sizeof(buf), "q%08lld", static_cast<long long>(id_rank[i]));
    pool[i] = {buf, base[i], enq[i], res[i]};
  }
  auto adm = sched::form_batch(pool, active_reservation, capacity, now, aging);
  for (size_t k = 0; k < adm.size(); ++k) out[k] = static_cast<int32_t>(adm[k]);
  return static_cast<int64_t>(adm.size());
}

int32_t pref_preemption_victim(int32_t n, const double* base, const double* enq,
                               const int64_t* res, const int64_t* id_rank, double now,
                               double aging) {
  std::vector<sched::QueueItem> act(n);
  char buf[32];
  for (int32_t i = 0; i < n; ++i) {
    std::snprintf(buf, sizeof(buf), "q%08lld", static_cast<long long>(id_rank[i]));
    act[i] = {buf, base[i], enq[i], res[i]};
  }
  return static_cast<int32_t>(sched::select_preemption_victim(act, now, aging));
}

}  // extern "C"
