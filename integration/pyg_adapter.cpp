// integration/pyg_adapter.cpp -- the reference-side binding a maintainer adds.
//
// Implements the reference's cache (hierarchy.hpp, manager.hpp) and router
// (router.hpp) interfaces over the C-ABI of libpyg_b200.so, so the reference's
// own simulator engine (src/sim/engine.cpp, unmodified) runs its hot path on a
// B200: lookups, inserts, pins, eviction, completion sweeps, staging lookups and
// every routing decision are device calls.  Compiled with the overlay headers in
// integration/overlay first on the include path (integration/Makefile).
//
// One pyg_ctx holds every replica of the simulation (slots handed out in the
// order the engine constructs CacheHierarchy objects) plus the shared L3.
// Workflow / role strings are interned to ints; role ids must stay < 64.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <map>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "pyg.h"
#include "pythia/cache/hierarchy.hpp"
#include "pythia/cache/manager.hpp"
#include "pythia/sched/router.hpp"
#include "pythia/sched/worker.hpp"

namespace {

void check(int rc) {
  if (rc != PYG_OK) throw std::runtime_error(std::string("libpyg_b200: ") + pyg_last_error());
}

// PYG_ADAPTER_PROFILE=1: calls and wall time per C-ABI entry, printed to stderr at exit
struct Prof {
  struct Row {
    int64_t calls = 0;
    double ms = 0;
  };
  std::map<std::string, Row> rows;
  bool on = std::getenv("PYG_ADAPTER_PROFILE") != nullptr;
  ~Prof() {
    if (!on) return;
    std::vector<std::pair<double, std::string>> v;
    for (auto& [k, r] : rows) v.emplace_back(r.ms, k);
    std::sort(v.rbegin(), v.rend());
    for (auto& [ms, k] : v)
      std::fprintf(stderr, "%10.1f ms %9lld calls  %s\n", ms, static_cast<long long>(rows[k].calls),
                   k.c_str());
  }
  static Prof& get() {
    static Prof p;
    return p;
  }
};
template <class F>
struct Timed {
  const char* name;
  F f;
  template <class... A>
  int operator()(A&&... a) const {
    Prof& p = Prof::get();
    if (!p.on) return f(std::forward<A>(a)...);
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = f(std::forward<A>(a)...);
    auto& r = p.rows[name];
    r.calls += 1;
    r.ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return rc;
  }
};
#define PYG_T(fn) Timed<decltype(&fn)>{#fn, &fn}

struct Backend {
  pyg_ctx* ctx = nullptr;
  int32_t next_slot = 0;
  int32_t max_slots = 0;
  // node_view memo: the engine asks lookup(prompt, nullptr) of every ready replica in turn
  // (engine.cpp:640-648); the first call computes all replicas' lookups in one device call
  // (pyg_lookup_all) and the next ones are served from here until any tier changes
  uint64_t epoch = 0;  // bumped by every mutating call
  struct {
    bool valid = false;
    uint64_t epoch = 0;
    int32_t n_slots = 0;
    std::vector<uint64_t> tokens;
    std::vector<int64_t> m;  // 3 per slot
  } view;
  // per-tier change epochs (key: 2*slot + tier for replica tiers, the last key for L3) so
  // a tier's snapshot (TierStore::blocks) is re-read only after that tier changed
  std::vector<uint64_t> tier_epoch;
  size_t tkey(int32_t slot, int32_t tier) const {
    return tier == 2 || slot < 0 ? 2 * static_cast<size_t>(max_slots) : 2 * static_cast<size_t>(slot) + tier;
  }
  // host mirrors, exact by construction: a tier's occupancy as read after its last change
  // (re-read once the tier's epoch moves), capacities (fixed), decode tokens per slot (every
  // change goes through add_decode_tokens; pushed to the device lazily, before the device
  // next reads it -- an eviction on that slot)
  std::vector<int64_t> occ, cap, decode, decode_pending;
  std::vector<uint64_t> occ_ep;
  std::vector<char> cap_ok;
  void bump() { ++epoch; }
  void bump(int32_t slot, int32_t tier) {
    ++epoch;
    ++tier_epoch[tkey(slot, tier)];
  }
  std::unordered_map<std::string, int32_t> wf_ids, role_ids;
  std::vector<std::string> wf_names, role_names;
  std::vector<pyg_block> dump_buf;

  static Backend& get() {
    static Backend b;
    if (!b.ctx) b.create();
    return b;
  }

  void create() {
    const char* e = std::getenv("PYG_ENGINE_MAX_REPLICAS");
    max_slots = e ? std::atoi(e) : 64;
    const char* d = std::getenv("PYG_ENGINE_DEVICE");
    std::vector<int64_t> zero(max_slots, 0);
    pyg_config cfg{static_cast<int32_t>(pythia::cache::kBlockTokens), max_slots, d ? std::atoi(d) : 0,
                   0, zero.data(), zero.data(), 256};  // tiers grow on demand
    check(PYG_T(pyg_create)(&cfg, &ctx));
    tier_epoch.assign(2 * static_cast<size_t>(max_slots) + 1, 0);
    occ.assign(tier_epoch.size(), 0);
    cap.assign(tier_epoch.size(), 0);
    occ_ep.assign(tier_epoch.size(), ~0ULL);
    cap_ok.assign(tier_epoch.size(), 0);
    decode.assign(max_slots, 0);
    decode_pending.assign(max_slots, 0);
  }
  void stats(int32_t slot, int32_t tier) {
    const size_t k = tkey(slot, tier);
    if (occ_ep[k] == tier_epoch[k] && cap_ok[k]) return;
    int64_t o, c, n;
    check(PYG_T(pyg_tier_stats)(ctx, slot < 0 ? 0 : slot, tier, &o, &c, &n));
    occ[k] = o;
    cap[k] = c;
    occ_ep[k] = tier_epoch[k];
    cap_ok[k] = 1;
  }
  int64_t occupancy(int32_t slot, int32_t tier) {
    stats(slot, tier);
    return occ[tkey(slot, tier)];
  }
  int64_t capacity(int32_t slot, int32_t tier) {
    stats(slot, tier);
    return cap[tkey(slot, tier)];
  }
  void flush_decode(int32_t slot) {
    if (decode_pending[slot] == 0) return;
    check(PYG_T(pyg_add_decode_tokens)(ctx, slot, decode_pending[slot]));
    decode_pending[slot] = 0;
  }

  int32_t wf(const std::string& s) {
    auto it = wf_ids.find(s);
    if (it != wf_ids.end()) return it->second;
    const int32_t id = static_cast<int32_t>(wf_names.size());
    wf_ids.emplace(s, id);
    wf_names.push_back(s);
    return id;
  }
  int32_t role(const std::string& s) {
    auto it = role_ids.find(s);
    if (it != role_ids.end()) return it->second;
    const int32_t id = static_cast<int32_t>(role_names.size());
    if (id >= 64) throw std::runtime_error("libpyg_b200 adapter: more than 64 distinct roles");
    role_ids.emplace(s, id);
    role_names.push_back(s);
    return id;
  }
  uint64_t mask(const std::set<std::string>& roles) {
    uint64_t m = 0;
    for (const auto& r : roles) m |= 1ULL << role(r);
    return m;
  }
  pythia::cache::CacheBlock block(const pyg_block& b) const {
    pythia::cache::CacheBlock x;
    x.block_id = b.block_id;
    x.chain_hash = b.chain_hash;
    x.span_start = b.span_start;
    x.span_end = b.span_end;
    x.lineage = {wf_names.at(b.workflow), role_names.at(b.role)};
    x.last_access = b.last_access;
    x.pin_count = b.pin_count;
    return x;
  }
};

int32_t api_slot(int32_t slot) { return slot < 0 ? 0 : slot; }

}  // namespace

namespace pythia::cache {

const char* tier_name(Tier t) {
  return t == Tier::L1 ? "L1" : t == Tier::L2 ? "L2" : "L3";
}

std::vector<uint64_t> chain_boundary_hashes(const workflow::TokenSeq& tokens) {
  Backend& b = Backend::get();
  std::vector<uint64_t> out((tokens.size() + kBlockTokens - 1) / kBlockTokens);
  int64_t n = 0;
  check(PYG_T(pyg_chain_hashes)(b.ctx, tokens.data(), static_cast<int64_t>(tokens.size()), out.data(), &n));
  out.resize(n);
  return out;
}

// ------------------------------------------------------------------ TierStore
TierStore::TierStore(int64_t) : slot_(-1), tier_(2) {}

int64_t TierStore::capacity() const { return Backend::get().capacity(slot_, tier_); }

int64_t TierStore::occupancy() const { return Backend::get().occupancy(slot_, tier_); }

const std::map<uint64_t, CacheBlock>& TierStore::blocks() const {
  Backend& b = Backend::get();
  const uint64_t ep = b.tier_epoch[b.tkey(slot_, tier_)];
  if (view_epoch_ == ep) return view_;
  view_epoch_ = ep;
  int64_t n = 0;
  if (b.dump_buf.empty()) b.dump_buf.resize(1 << 14);
  for (;;) {
    check(PYG_T(pyg_tier_dump)(b.ctx, api_slot(slot_), tier_, b.dump_buf.data(),
                        static_cast<int64_t>(b.dump_buf.size()), &n));
    if (n <= static_cast<int64_t>(b.dump_buf.size())) break;
    b.dump_buf.resize(2 * n);
  }
  view_.clear();
  for (int64_t i = 0; i < n; ++i)
    if (b.dump_buf[i].alive) view_.emplace_hint(view_.end(), b.dump_buf[i].block_id, b.block(b.dump_buf[i]));
  return view_;
}

const CacheBlock* TierStore::find_chain(uint64_t chain_hash) const {
  Backend& b = Backend::get();
  pyg_block x{};
  int32_t found = 0;
  check(PYG_T(pyg_tier_find)(b.ctx, api_slot(slot_), tier_, chain_hash, &x, &found));
  if (!found) return nullptr;
  found_ = b.block(x);
  return &found_;
}

CacheBlock* TierStore::find_chain_mut(uint64_t chain_hash) {
  return const_cast<CacheBlock*>(static_cast<const TierStore*>(this)->find_chain(chain_hash));
}

uint64_t TierStore::put(uint64_t chain_hash, int64_t span_start, int64_t span_end,
                        const Lineage& lineage, double now, int pin_delta, uint64_t*) {
  Backend& b = Backend::get();
  b.bump(slot_, tier_);
  uint64_t id = 0;
  check(PYG_T(pyg_tier_put)(b.ctx, api_slot(slot_), tier_, chain_hash, span_start, span_end,
                     b.wf(lineage.workflow_id), b.role(lineage.role_id), now, pin_delta, &id));
  return id;
}

void TierStore::erase(uint64_t block_id) {
  Backend::get().bump(slot_, tier_);
  check(PYG_T(pyg_tier_erase)(Backend::get().ctx, api_slot(slot_), tier_, block_id));
}

int64_t TierStore::matched_prefix(const workflow::TokenSeq& tokens,
                                  const std::vector<uint64_t>&) const {
  int64_t m = 0;
  check(PYG_T(pyg_matched_prefix)(Backend::get().ctx, api_slot(slot_), tier_, tokens.data(),
                           static_cast<int64_t>(tokens.size()), &m));
  return m;
}

// ------------------------------------------------------------- CacheHierarchy
CacheHierarchy::CacheHierarchy(int64_t l1_capacity, int64_t l2_capacity)
    : slot_(Backend::get().next_slot++), l1_(slot_, 0), l2_(slot_, 1) {
  Backend& b = Backend::get();
  if (slot_ >= b.max_slots)
    throw std::runtime_error("libpyg_b200 adapter: raise PYG_ENGINE_MAX_REPLICAS");
  check(PYG_T(pyg_set_capacity)(b.ctx, slot_, l1_capacity, l2_capacity));
  b.bump(slot_, 0);
  b.bump(slot_, 1);
}

CacheHierarchy::Match CacheHierarchy::lookup(const workflow::TokenSeq& prompt,
                                             const SharedL3* l3) const {
  Backend& b = Backend::get();
  if (l3 == nullptr) {  // node_view: every replica at once, memoized until a tier changes
    auto& v = b.view;
    if (!(v.valid && v.epoch == b.epoch && slot_ < v.n_slots && v.tokens == prompt)) {
      v.n_slots = b.next_slot;
      v.m.resize(3 * static_cast<size_t>(v.n_slots));
      check(PYG_T(pyg_lookup_all)(b.ctx, prompt.data(), static_cast<int64_t>(prompt.size()), 0,
                           v.n_slots, v.m.data()));
      v.tokens = prompt;
      v.epoch = b.epoch;
      v.valid = true;
    }
    return {v.m[3 * slot_], v.m[3 * slot_ + 1], 0};
  }
  int64_t m[3];
  check(PYG_T(pyg_lookup)(b.ctx, slot_, prompt.data(), static_cast<int64_t>(prompt.size()), 1, m));
  return {m[0], m[1], m[2]};
}

void CacheHierarchy::insert_chain(Tier t, const workflow::TokenSeq& tokens, int64_t upto,
                                  const Lineage& lineage, double now, int pin_delta) {
  Backend& b = Backend::get();
  b.bump(slot_, t == Tier::L1 ? 0 : 1);  // tier(L3) aliases L2
  check(PYG_T(pyg_insert_chain)(b.ctx, slot_, static_cast<int32_t>(t), tokens.data(),
                         static_cast<int64_t>(tokens.size()), upto, b.wf(lineage.workflow_id),
                         b.role(lineage.role_id), now, pin_delta));
}

void CacheHierarchy::unpin_chain(const workflow::TokenSeq& tokens, int64_t upto) {
  Backend::get().bump(slot_, 0);
  check(PYG_T(pyg_unpin_chain)(Backend::get().ctx, slot_, tokens.data(),
                        static_cast<int64_t>(tokens.size()), upto));
}

void CacheHierarchy::add_decode_tokens(int64_t n) {
  Backend& b = Backend::get();
  b.decode[slot_] += n;  // hierarchy.hpp:111; reaches the device before its next eviction
  b.decode_pending[slot_] += n;
}

// hierarchy.hpp:114: blocks + in-flight decode tokens
int64_t CacheHierarchy::l1_occupancy() const {
  Backend& b = Backend::get();
  return b.occupancy(slot_, 0) + b.decode[slot_];
}

int64_t CacheHierarchy::decode_tokens() const { return Backend::get().decode[slot_]; }

// ------------------------------------------------------------------- manager
std::set<std::string> future_nodes(const workflow::PathCursor& position) {
  return workflow::future_roles(position);
}

void FutureRegistry::update(const std::string& workflow_id, std::set<std::string> roles) {
  Backend& b = Backend::get();
  check(PYG_T(pyg_registry_update)(b.ctx, b.wf(workflow_id), b.mask(roles)));
  futures_[workflow_id] = std::move(roles);
}

void FutureRegistry::drop(const std::string& workflow_id) {
  Backend& b = Backend::get();
  check(PYG_T(pyg_registry_drop)(b.ctx, b.wf(workflow_id)));
  futures_.erase(workflow_id);
}

bool FutureRegistry::lineage_live(const Lineage& lineage) const {
  auto it = futures_.find(lineage.workflow_id);
  return it != futures_.end() && it->second.count(lineage.role_id) > 0;
}

// manager.cpp:25-42 over a device dump of the replica's L1 and L2
std::vector<CompletionAction> on_request_complete(const workflow::RequestEnvelope& req,
                                                  const CacheHierarchy& cache) {
  std::vector<CompletionAction> out;
  if (req.unprofiled() || !req.position) return out;
  const std::set<std::string> future = future_nodes(*req.position);
  for (Tier t : {Tier::L1, Tier::L2}) {
    for (const auto& [id, blk] : cache.tier(t).blocks()) {
      if (blk.pinned() || blk.lineage.workflow_id != req.app_metadata.workflow_id) continue;
      out.push_back({future.count(blk.lineage.role_id) ? CompletionAction::Kind::RetainAndWriteL3
                                                       : CompletionAction::Kind::Free,
                     t, id});
    }
  }
  return out;
}

// manager.cpp:44-58: one dump per tier, then device erases / L3 puts in action order
// manager.cpp:44-58: the erases (per tier) and the L3 writes go to the device as two ordered
// lists -- they touch different tiers, so only the order within each list matters
void apply_completion(const std::vector<CompletionAction>& actions, CacheHierarchy& cache,
                      SharedL3& l3, double now) {
  Backend& b = Backend::get();
  std::map<uint64_t, CacheBlock> view[2];
  bool have[2] = {false, false};
  std::vector<uint64_t> frees[2];
  std::vector<pyg_put_item> puts;
  for (const auto& a : actions) {
    const int k = a.tier == Tier::L1 ? 0 : 1;
    if (!have[k]) {
      view[k] = cache.tier(a.tier).blocks();
      have[k] = true;
    }
    auto it = view[k].find(a.block_id);
    if (it == view[k].end()) continue;
    if (a.kind == CompletionAction::Kind::Free) {
      frees[k].push_back(a.block_id);
      view[k].erase(it);
    } else {
      const CacheBlock& blk = it->second;
      puts.push_back({blk.chain_hash, blk.span_start, blk.span_end, b.wf(blk.lineage.workflow_id),
                      b.role(blk.lineage.role_id)});
    }
  }
  const int32_t slot = cache.tier(Tier::L1).slot();
  for (int k = 0; k < 2; ++k) {
    if (frees[k].empty()) continue;
    b.bump(slot, k);
    check(PYG_T(pyg_tier_erase_many)(b.ctx, slot, k, frees[k].data(),
                                     static_cast<int64_t>(frees[k].size())));
  }
  if (!puts.empty()) {
    b.bump(-1, 2);
    check(PYG_T(pyg_tier_put_many)(b.ctx, 0, 2, puts.data(), static_cast<int64_t>(puts.size()),
                                   now, 0));
  }
  (void)l3;
}

// manager.cpp:60-100 with device lookups
std::vector<StageAction> on_prefetch_requested(const workflow::RequestEnvelope& req,
                                               const CacheHierarchy& target_cache,
                                               const SharedL3& l3,
                                               const workflow::PromptHistory& history,
                                               bool gpu_idle) {
  std::vector<StageAction> out;
  if (req.unprofiled()) return out;
  for (const auto& [role, tmpl] : req.sys_annotations->prompt_composition) {
    StageAction a;
    a.successor_role = role;
    a.lineage = {req.app_metadata.workflow_id, role};
    auto prefix = workflow::assemble_resolvable_prefix(tmpl, history);
    if (prefix.tokens.empty()) {
      a.reason = "unresolved";
      out.push_back(std::move(a));
      continue;
    }
    a.tokens = std::move(prefix.tokens);
    const int64_t len = static_cast<int64_t>(a.tokens.size());
    const auto m = target_cache.lookup(a.tokens, &l3);
    const int64_t staged = std::max(m.l1, m.l2);
    if (staged >= len) {
      a.reason = "already-staged";
    } else if (m.l3 > staged) {
      a.kind = StageAction::Kind::PromoteToHost;
      a.from = staged;
      a.to = m.l3;
    } else if (gpu_idle) {
      a.kind = StageAction::Kind::BackgroundPrefill;
      a.from = staged;
      a.to = len;
    } else {
      a.reason = "gpu-busy";
    }
    out.push_back(std::move(a));
  }
  return out;
}

EvictionResult evict_for_space(CacheHierarchy& cache, Tier tier, int64_t needed,
                               const FutureRegistry&, bool speculative) {
  Backend& b = Backend::get();
  const int32_t slot = cache.tier(Tier::L1).slot();
  const int32_t tt = tier == Tier::L1 ? 0 : 1;  // tier(L3) aliases L2
  // manager.cpp:106-111 on the host mirrors: no excess, nothing to do
  const int64_t base = tt == 0 ? cache.l1_occupancy() : b.occupancy(slot, 1);
  if (base + needed - b.capacity(slot, tt) <= 0) {
    EvictionResult r;
    r.satisfied = true;
    return r;
  }
  b.flush_decode(slot);
  b.bump(slot, tt);
  static std::vector<uint64_t> ids(1 << 20);
  int64_t n = 0, ft = 0;
  int32_t ok = 0;
  check(PYG_T(pyg_evict_for_space)(b.ctx, cache.tier(Tier::L1).slot(), static_cast<int32_t>(tier), needed,
                            speculative, ids.data(), static_cast<int64_t>(ids.size()), &n, &ft,
                            &ok));
  if (n > static_cast<int64_t>(ids.size()))
    throw std::runtime_error("libpyg_b200 adapter: eviction list longer than 2^20 blocks");
  // the mirror follows without a device read: the tier lost exactly the freed tokens
  const size_t k = b.tkey(slot, tt);
  if (b.occ_ep[k] == b.tier_epoch[k] - 1) {
    b.occ[k] -= ft;
    b.occ_ep[k] = b.tier_epoch[k];
  }
  EvictionResult r;
  r.freed.assign(ids.begin(), ids.begin() + n);
  r.freed_tokens = ft;
  r.satisfied = ok != 0;
  return r;
}

}  // namespace pythia::cache

// -------------------------------------------------------------------- router
namespace pythia::sched {

bool capacity_holds(const NodeView& node, const Reservation& req) {
  int64_t sum = req.tokens();
  for (const auto& a : node.assigned) sum += a.tokens();
  return sum <= node.kv_capacity;
}

double oom_bound(const NodeView& node, const Reservation& req) {
  double b = req.alpha;
  for (const auto& a : node.assigned) b += a.alpha;
  return b;
}

RoutingDecision route(const std::vector<NodeView>& nodes, const Reservation& req, double eps) {
  Backend& b = Backend::get();
  const int32_t n = static_cast<int32_t>(nodes.size());
  std::vector<int32_t> rid(n);
  std::vector<int64_t> kv(n), off(n + 1, 0), staged(n);
  std::vector<pyg_reservation> asg;
  for (int32_t i = 0; i < n; ++i) {
    rid[i] = nodes[i].replica_id;
    kv[i] = nodes[i].kv_capacity;
    staged[i] = nodes[i].staged_l2_prefix;
    for (const auto& a : nodes[i].assigned)
      asg.push_back({a.prompt_len, a.upper, a.alpha, a.tokens_generated});
    off[i + 1] = static_cast<int64_t>(asg.size());
  }
  const pyg_reservation q{req.prompt_len, req.upper, req.alpha, req.tokens_generated};
  if (asg.empty()) asg.push_back({0, 0, 0.0, 0});  // never read: off[n] == 0
  pyg_decision d{};
  check(PYG_T(pyg_route)(b.ctx, n, rid.data(), kv.data(), off.data(), asg.data(), staged.data(), &q, eps,
                  &d));
  RoutingDecision out;
  if (d.target >= 0) out.target = d.target;
  out.headroom = d.headroom;
  out.oom_bound = d.oom_bound;
  out.cache_tiebreak_used = d.tiebreak != 0;
  return out;
}

double effective_priority(double base_priority, double enqueue_time, double now,
                          double aging_rate) {
  return base_priority + aging_rate * (now - enqueue_time);
}

namespace {
// QueueItems as device records; request ids become their rank in string order
std::vector<pyg_queue_item> queue_items(const std::vector<QueueItem>& q) {
  std::vector<size_t> by_id(q.size());
  for (size_t i = 0; i < q.size(); ++i) by_id[i] = i;
  std::sort(by_id.begin(), by_id.end(),
            [&](size_t a, size_t b) { return q[a].request_id < q[b].request_id; });
  std::vector<pyg_queue_item> out(q.size());
  for (size_t r = 0; r < by_id.size(); ++r) {
    const QueueItem& x = q[by_id[r]];
    out[by_id[r]] = {x.base_priority, x.enqueue_time, x.reservation, static_cast<int64_t>(r)};
  }
  return out;
}

struct DeviceQueue {  // one queue's arrays on the device for the K7 calls
  void* mem = nullptr;
  ~DeviceQueue() { cudaFree(mem); }
};
}  // namespace

std::vector<size_t> form_batch(const std::vector<QueueItem>& pool, int64_t active_reservation,
                               int64_t capacity, double now, double aging_rate) {
  if (pool.empty()) return {};
  Backend& b = Backend::get();
  const auto items = queue_items(pool);
  const int64_t n = static_cast<int64_t>(items.size());
  const int64_t hdr[4] = {0, n, active_reservation, capacity};
  DeviceQueue dq;
  const size_t bytes = 32 + n * sizeof(pyg_queue_item) + n * 4 + 8;
  if (cudaMalloc(&dq.mem, bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc");
  char* p = static_cast<char*>(dq.mem);
  cudaMemcpy(p, hdr, 32, cudaMemcpyHostToDevice);
  cudaMemcpy(p + 32, items.data(), n * sizeof(pyg_queue_item), cudaMemcpyHostToDevice);
  auto* d_order = reinterpret_cast<int32_t*>(p + 32 + n * sizeof(pyg_queue_item));
  auto* d_n = d_order + n;
  const auto* d_hdr = reinterpret_cast<const int64_t*>(p);
  check(PYG_T(pyg_set_stream)(b.ctx, nullptr));
  check(PYG_T(pyg_form_batch_dev)(b.ctx, 1, d_hdr, reinterpret_cast<const pyg_queue_item*>(p + 32),
                           d_hdr + 2, d_hdr + 3, now, aging_rate, d_order, d_n));
  int32_t na = 0;
  std::vector<int32_t> ord(n);
  cudaMemcpy(&na, d_n, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(ord.data(), d_order, n * 4, cudaMemcpyDeviceToHost);
  check(PYG_T(pyg_check_device_error)(b.ctx));
  return std::vector<size_t>(ord.begin(), ord.begin() + na);
}

size_t select_preemption_victim(const std::vector<QueueItem>& active, double now,
                                double aging_rate) {
  Backend& b = Backend::get();
  const auto items = queue_items(active);
  const int64_t n = static_cast<int64_t>(items.size());
  const int64_t hdr[2] = {0, n};
  DeviceQueue dq;
  if (cudaMalloc(&dq.mem, 16 + n * sizeof(pyg_queue_item) + 8) != cudaSuccess)
    throw std::runtime_error("cudaMalloc");
  char* p = static_cast<char*>(dq.mem);
  cudaMemcpy(p, hdr, 16, cudaMemcpyHostToDevice);
  cudaMemcpy(p + 16, items.data(), n * sizeof(pyg_queue_item), cudaMemcpyHostToDevice);
  auto* d_v = reinterpret_cast<int32_t*>(p + 16 + n * sizeof(pyg_queue_item));
  check(PYG_T(pyg_set_stream)(b.ctx, nullptr));
  check(PYG_T(pyg_preemption_victim_dev)(b.ctx, 1, reinterpret_cast<const int64_t*>(p),
                                  reinterpret_cast<const pyg_queue_item*>(p + 16), now, aging_rate,
                                  d_v));
  int32_t v = 0;
  cudaMemcpy(&v, d_v, 4, cudaMemcpyDeviceToHost);
  return static_cast<size_t>(v);
}

std::optional<int> route_least_outstanding(const std::vector<NodeView>& nodes) {
  Backend& b = Backend::get();
  const int32_t n = static_cast<int32_t>(nodes.size());
  if (n == 0) return std::nullopt;
  std::vector<int32_t> rid(n);
  std::vector<int64_t> off(n + 1, 0);
  for (int32_t i = 0; i < n; ++i) {
    rid[i] = nodes[i].replica_id;
    off[i + 1] = off[i] + static_cast<int64_t>(nodes[i].assigned.size());
  }
  int32_t t = -1;
  check(PYG_T(pyg_route_least_outstanding)(b.ctx, n, rid.data(), off.data(), &t));
  if (t < 0) return std::nullopt;
  return t;
}

}  // namespace pythia::sched
