/*
 * pyg_oracle.c -- CPU restatement of the Pythia scheduling hot path.
 * TEST INFRASTRUCTURE ONLY (see pyg_oracle.h for the rules and pinning).
 * Reference paths are relative to /root/reference/proj/.
 */
#include "pyg_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* hashing                                                             */
/* ------------------------------------------------------------------ */

/* inc/workflow/tokens.hpp:22-28 */
uint64_t o_fnv1a_bytes(const char* s, int64_t n, uint64_t h) {
  for (int64_t i = 0; i < n; ++i) {
    h ^= (unsigned char)s[i];
    h *= O_FNV_PRIME;
  }
  return h;
}

/* inc/workflow/tokens.hpp:30-36: 8 little-endian bytes of the token */
uint64_t o_fnv1a_u64(uint64_t v, uint64_t h) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (i * 8)) & 0xff;
    h *= O_FNV_PRIME;
  }
  return h;
}

/* src/cache/hierarchy.cpp:21-30: one running hash, emitted at every block
   boundary and after the last token. */
int64_t o_chain_hashes(const uint64_t* tokens, int64_t n, int64_t B, uint64_t* out) {
  uint64_t h = O_FNV_OFFSET;
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    h = o_fnv1a_u64(tokens[i], h);
    if ((i + 1) % B == 0 || i + 1 == n) out[k++] = h;
  }
  return k;
}

static int64_t n_hashes(int64_t n, int64_t B) { return (n + B - 1) / B; }

/* ------------------------------------------------------------------ */
/* TierStore                                                           */
/* ------------------------------------------------------------------ */

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  return x;
}

static void map_alloc(o_tier* t, int64_t hcap) {
  t->hcap = hcap;
  t->hused = 0;
  t->hk = (uint64_t*)calloc((size_t)hcap, sizeof(uint64_t));
  t->hv = (int64_t*)calloc((size_t)hcap, sizeof(int64_t));
  t->hs = (uint8_t*)calloc((size_t)hcap, 1);
}

static void map_insert_raw(o_tier* t, uint64_t key, int64_t v) {
  uint64_t m = (uint64_t)t->hcap - 1;
  uint64_t i = mix64(key) & m;
  while (t->hs[i] == 1) i = (i + 1) & m;
  if (t->hs[i] == 0) t->hused++;
  t->hs[i] = 1;
  t->hk[i] = key;
  t->hv[i] = v;
}

static int64_t map_find_slot(const o_tier* t, uint64_t key) {
  uint64_t m = (uint64_t)t->hcap - 1;
  uint64_t i = mix64(key) & m;
  while (t->hs[i] != 0) {
    if (t->hs[i] == 1 && t->hk[i] == key) return (int64_t)i;
    i = (i + 1) & m;
  }
  return -1;
}

/* drops dead log entries and rebuilds the index (internal housekeeping, no semantic effect) */
static void tier_rebuild(o_tier* t, int64_t want_cap) {
  int64_t w = 0;
  for (int64_t i = 0; i < t->n; ++i)
    if (t->b[i].alive) t->b[w++] = t->b[i];
  t->n = w;
  if (want_cap > t->cap) {
    t->b = (o_block*)realloc(t->b, (size_t)want_cap * sizeof(o_block));
    t->cap = want_cap;
  }
  int64_t hcap = 16;
  while (hcap < 2 * t->cap) hcap <<= 1;
  free(t->hk);
  free(t->hv);
  free(t->hs);
  map_alloc(t, hcap);
  for (int64_t i = 0; i < t->n; ++i) map_insert_raw(t, t->b[i].hash, i);
}

void o_tier_init(o_tier* t, int64_t capacity) {
  memset(t, 0, sizeof(*t));
  t->capacity = capacity;
  t->cap = 8;
  t->b = (o_block*)malloc((size_t)t->cap * sizeof(o_block));
  map_alloc(t, 16);
}

void o_tier_free(o_tier* t) {
  free(t->b);
  free(t->hk);
  free(t->hv);
  free(t->hs);
  memset(t, 0, sizeof(*t));
}

void o_tier_copy(o_tier* dst, const o_tier* src) {
  *dst = *src;
  dst->b = (o_block*)malloc((size_t)src->cap * sizeof(o_block));
  memcpy(dst->b, src->b, (size_t)src->n * sizeof(o_block));
  dst->hk = (uint64_t*)malloc((size_t)src->hcap * sizeof(uint64_t));
  dst->hv = (int64_t*)malloc((size_t)src->hcap * sizeof(int64_t));
  dst->hs = (uint8_t*)malloc((size_t)src->hcap);
  memcpy(dst->hk, src->hk, (size_t)src->hcap * sizeof(uint64_t));
  memcpy(dst->hv, src->hv, (size_t)src->hcap * sizeof(int64_t));
  memcpy(dst->hs, src->hs, (size_t)src->hcap);
}

/* hierarchy.cpp:32-42 */
const o_block* o_tier_find(const o_tier* t, uint64_t hash) {
  int64_t s = map_find_slot(t, hash);
  return s < 0 ? NULL : &t->b[t->hv[s]];
}
o_block* o_tier_find_mut(o_tier* t, uint64_t hash) {
  int64_t s = map_find_slot(t, hash);
  return s < 0 ? NULL : &t->b[t->hv[s]];
}

/* std::map::find by id: ids are ascending in the log */
o_block* o_tier_by_id(o_tier* t, uint64_t id) {
  int64_t lo = 0, hi = t->n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    if (t->b[mid].id == id) return t->b[mid].alive ? &t->b[mid] : NULL;
    if (t->b[mid].id < id)
      lo = mid + 1;
    else
      hi = mid - 1;
  }
  return NULL;
}

/* hierarchy.cpp:44-66.  The reference returns blocks_.rbegin()->first for a new block, i.e. the
   largest id in the tier; with the canonical counters (replica counter for L1/L2, L3 counter) the
   new id is always the largest, so it is the new id. */
uint64_t o_tier_put(o_tier* t, uint64_t hash, int64_t s, int64_t e, int32_t wf, int32_t role,
                    double now, int32_t pin_delta, uint64_t* counter) {
  o_block* ex = o_tier_find_mut(t, hash);
  if (ex) {
    ex->la = now;
    ex->pin += pin_delta; /* assert compiled out (NDEBUG) */
    return ex->id;
  }
  if (t->n == t->cap || t->hused + 1 > t->hcap / 2) {
    int64_t want = t->cap;
    if (t->n_alive + 1 > t->cap / 2) want = t->cap * 2;
    tier_rebuild(t, want);
  }
  o_block* b = &t->b[t->n];
  b->id = (*counter)++;
  b->hash = hash;
  b->s = s;
  b->e = e;
  b->wf = wf;
  b->role = role;
  b->la = now;
  b->pin = pin_delta > 0 ? pin_delta : 0;
  b->alive = 1;
  t->occupancy += e - s;
  map_insert_raw(t, hash, t->n);
  t->n++;
  t->n_alive++;
  return b->id;
}

/* hierarchy.cpp:68-82 */
void o_tier_erase(o_tier* t, uint64_t id) {
  o_block* b = o_tier_by_id(t, id);
  if (!b) return;
  t->occupancy -= b->e - b->s;
  int64_t slot = map_find_slot(t, b->hash);
  if (slot >= 0) t->hs[slot] = 2;
  b->alive = 0;
  t->n_alive--;
}

/* hierarchy.cpp:84-104: aligned walk, then the ragged scan over blocks whose
   span_start equals the matched length. */
int64_t o_matched_prefix(const o_tier* t, const uint64_t* tokens, int64_t n,
                         const uint64_t* hashes, int64_t nh, int64_t B) {
  int64_t total = n, matched = 0;
  for (int64_t i = 0; i < nh; ++i) {
    if (!o_tier_find(t, hashes[i])) break;
    int64_t m = (i + 1) * B;
    matched = m < total ? m : total;
  }
  if (matched >= total || matched % B != 0) return matched;
  int64_t best = matched;
  for (int64_t k = 0; k < t->n; ++k) { /* equal_range(by_span_start_, matched) */
    const o_block* b = &t->b[k];
    if (!b->alive || b->s != matched) continue;
    if (b->e > total || b->e % B == 0) continue;
    uint64_t h = O_FNV_OFFSET;
    for (int64_t x = 0; x < b->e; ++x) h = o_fnv1a_u64(tokens[x], h);
    if (h == b->hash && b->e > best) best = b->e;
  }
  return best;
}

int64_t o_tier_dump(const o_tier* t, o_block* out, int64_t cap) {
  int64_t k = 0;
  for (int64_t i = 0; i < t->n; ++i) {
    if (!t->b[i].alive) continue;
    if (out && k < cap) out[k] = t->b[i];
    k++;
  }
  return k;
}

/* ------------------------------------------------------------------ */
/* CacheHierarchy / SharedL3                                           */
/* ------------------------------------------------------------------ */

void o_cache_init(o_cache* c, int64_t l1_cap, int64_t l2_cap) {
  memset(c, 0, sizeof(*c));
  o_tier_init(&c->l1, l1_cap);
  o_tier_init(&c->l2, l2_cap);
  c->next_id = 1; /* hierarchy.hpp:122 */
}
void o_cache_free(o_cache* c) {
  o_tier_free(&c->l1);
  o_tier_free(&c->l2);
}
/* hierarchy.cpp:106-107: every non-L1 tier aliases l2_ */
o_tier* o_cache_tier(o_cache* c, int32_t tier) { return tier == 0 ? &c->l1 : &c->l2; }

void o_l3_init(o_l3* l3) {
  o_tier_init(&l3->store, INT64_MAX); /* hierarchy.hpp:83 */
  l3->next_id = 1;
}
void o_l3_free(o_l3* l3) { o_tier_free(&l3->store); }
void o_l3_copy(o_l3* dst, const o_l3* src) {
  o_tier_copy(&dst->store, &src->store);
  dst->next_id = src->next_id;
}

/* hierarchy.cpp:109-117 */
void o_lookup(const o_cache* c, const o_l3* l3, const uint64_t* tokens, int64_t n, int64_t B,
              int64_t out[3]) {
  uint64_t* h = (uint64_t*)malloc((size_t)(n_hashes(n, B) + 1) * sizeof(uint64_t));
  int64_t nh = o_chain_hashes(tokens, n, B, h);
  out[0] = o_matched_prefix(&c->l1, tokens, n, h, nh, B);
  out[1] = o_matched_prefix(&c->l2, tokens, n, h, nh, B);
  out[2] = l3 ? o_matched_prefix(&l3->store, tokens, n, h, nh, B) : 0;
  free(h);
}

/* hierarchy.cpp:119-130 */
void o_insert_chain(o_cache* c, int32_t tier, const uint64_t* tokens, int64_t n, int64_t upto,
                    int32_t wf, int32_t role, double now, int32_t pin_delta, int64_t B) {
  uint64_t* h = (uint64_t*)malloc((size_t)(n_hashes(n, B) + 1) * sizeof(uint64_t));
  int64_t nh = o_chain_hashes(tokens, n, B, h);
  o_tier* st = o_cache_tier(c, tier);
  for (int64_t i = 0; i < nh; ++i) {
    int64_t s = i * B, e = s + B < n ? s + B : n;
    if (e > upto) break;
    o_tier_put(st, h[i], s, e, wf, role, now, pin_delta, &c->next_id);
  }
  free(h);
}

/* hierarchy.cpp:132-142 (L1 only) */
void o_unpin_chain(o_cache* c, const uint64_t* tokens, int64_t n, int64_t upto, int64_t B) {
  uint64_t* h = (uint64_t*)malloc((size_t)(n_hashes(n, B) + 1) * sizeof(uint64_t));
  int64_t nh = o_chain_hashes(tokens, n, B, h);
  for (int64_t i = 0; i < nh; ++i) {
    int64_t e = (i + 1) * B < n ? (i + 1) * B : n;
    if (e > upto) break;
    o_block* b = o_tier_find_mut(&c->l1, h[i]);
    if (b && b->pin > 0) b->pin -= 1;
  }
  free(h);
}

/* hierarchy.hpp:114 */
int64_t o_l1_occupancy(const o_cache* c) { return c->l1.occupancy + c->decode_tokens; }

/* ------------------------------------------------------------------ */
/* FutureRegistry                                                      */
/* ------------------------------------------------------------------ */

void o_registry_init(o_registry* r) { memset(r, 0, sizeof(*r)); }
void o_registry_free(o_registry* r) {
  free(r->present);
  free(r->mask);
  memset(r, 0, sizeof(*r));
}
static void reg_grow(o_registry* r, int32_t wf) {
  if (wf < r->cap) return;
  int32_t nc = r->cap ? r->cap : 16;
  while (nc <= wf) nc *= 2;
  r->present = (uint8_t*)realloc(r->present, (size_t)nc);
  r->mask = (uint64_t*)realloc(r->mask, (size_t)nc * sizeof(uint64_t));
  memset(r->present + r->cap, 0, (size_t)(nc - r->cap));
  memset(r->mask + r->cap, 0, (size_t)(nc - r->cap) * sizeof(uint64_t));
  r->cap = nc;
}
/* manager.cpp:13-15 */
void o_registry_update(o_registry* r, int32_t wf, uint64_t role_mask) {
  reg_grow(r, wf);
  r->present[wf] = 1;
  r->mask[wf] = role_mask;
}
/* manager.cpp:17 */
void o_registry_drop(o_registry* r, int32_t wf) {
  if (wf < r->cap) {
    r->present[wf] = 0;
    r->mask[wf] = 0;
  }
}
/* manager.cpp:19-23 */
int o_lineage_live(const o_registry* r, int32_t wf, int32_t role) {
  if (wf < 0 || wf >= r->cap || !r->present[wf]) return 0;
  if (role < 0 || role >= 64) return 0;
  return (int)((r->mask[wf] >> role) & 1u);
}

/* ------------------------------------------------------------------ */
/* evict_for_space                                                     */
/* ------------------------------------------------------------------ */

typedef struct {
  int dead;
  double la;
  uint64_t id;
  int64_t size;
} victim;

/* manager.cpp:125-129 */
static int victim_cmp(const void* pa, const void* pb) {
  const victim* a = (const victim*)pa;
  const victim* b = (const victim*)pb;
  if (a->dead != b->dead) return a->dead ? -1 : 1;
  if (a->la != b->la) return a->la < b->la ? -1 : 1;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return 0;
}

/* manager.cpp:102-138 */
int o_evict_for_space(o_cache* c, int32_t tier, int64_t needed, const o_registry* reg,
                      int speculative, uint64_t* out_ids, int64_t cap, int64_t* n_freed,
                      int64_t* freed_tokens) {
  o_tier* st = o_cache_tier(c, tier);
  int64_t base = tier == 0 ? o_l1_occupancy(c) : st->occupancy;
  int64_t excess = base + needed - st->capacity;
  *n_freed = 0;
  *freed_tokens = 0;
  if (excess <= 0) return 1;
  victim* v = (victim*)malloc((size_t)(st->n + 1) * sizeof(victim));
  int64_t nv = 0;
  for (int64_t i = 0; i < st->n; ++i) {
    const o_block* b = &st->b[i];
    if (!b->alive || b->pin > 0) continue;
    v[nv].dead = speculative && !o_lineage_live(reg, b->wf, b->role);
    v[nv].la = b->la;
    v[nv].id = b->id;
    v[nv].size = b->e - b->s;
    nv++;
  }
  qsort(v, (size_t)nv, sizeof(victim), victim_cmp);
  int64_t freed = 0, k = 0;
  for (int64_t i = 0; i < nv; ++i) {
    if (freed >= excess) break;
    o_tier_erase(st, v[i].id);
    if (out_ids && k < cap) out_ids[k] = v[i].id;
    k++;
    freed += v[i].size;
  }
  free(v);
  *n_freed = k;
  *freed_tokens = freed;
  return freed >= excess;
}

/* ------------------------------------------------------------------ */
/* completion                                                          */
/* ------------------------------------------------------------------ */

/* manager.cpp:25-42 (req.unprofiled() || !req.position => no actions) */
int64_t o_on_request_complete(const o_cache* c, int32_t wf, uint64_t future_mask, int profiled,
                              o_action* out, int64_t cap) {
  int64_t k = 0;
  if (!profiled) return 0;
  for (int32_t tier = 0; tier < 2; ++tier) {
    const o_tier* st = tier == 0 ? &c->l1 : &c->l2;
    for (int64_t i = 0; i < st->n; ++i) {
      const o_block* b = &st->b[i];
      if (!b->alive || b->pin > 0) continue;
      if (b->wf != wf) continue;
      int live = b->role >= 0 && b->role < 64 && ((future_mask >> b->role) & 1u);
      if (out && k < cap) {
        out[k].kind = live ? 1 : 0;
        out[k].tier = tier;
        out[k].id = b->id;
      }
      k++;
    }
  }
  return k;
}

/* manager.cpp:44-58 */
void o_apply_completion(const o_action* acts, int64_t n, o_cache* c, o_l3* l3, double now) {
  for (int64_t i = 0; i < n; ++i) {
    o_tier* st = o_cache_tier(c, acts[i].tier);
    o_block* b = o_tier_by_id(st, acts[i].id);
    if (!b) continue;
    if (acts[i].kind == 0) {
      o_tier_erase(st, acts[i].id);
    } else {
      o_block cp = *b;
      o_tier_put(&l3->store, cp.hash, cp.s, cp.e, cp.wf, cp.role, now, 0, &l3->next_id);
    }
  }
}

/* ------------------------------------------------------------------ */
/* router                                                              */
/* ------------------------------------------------------------------ */

/* router.hpp:21 */
int64_t o_res_tokens(const o_res* r) {
  return r->prompt_len + (r->upper > r->tokens_generated ? r->upper : r->tokens_generated);
}

/* router.cpp:7-11 */
int o_capacity_holds(int64_t kv_capacity, const o_res* asg, int64_t na, const o_res* req) {
  int64_t total = o_res_tokens(req);
  for (int64_t i = 0; i < na; ++i) total += o_res_tokens(&asg[i]);
  return total <= kv_capacity;
}

/* router.cpp:13-17: ordered double sum, request alpha first */
double o_oom_bound(const o_res* asg, int64_t na, const o_res* req) {
  double sum = req->alpha;
  for (int64_t i = 0; i < na; ++i) sum += asg[i].alpha;
  return sum;
}

/* router.cpp:19-50 */
o_decision o_route(int32_t n_nodes, const int32_t* replica_id, const int64_t* kv_capacity,
                   const int64_t* asg_off, const o_res* asg, const int64_t* staged,
                   const o_res* req, double epsilon) {
  o_decision d;
  d.target = -1;
  d.tiebreak = 0;
  d.headroom = 0;
  d.oom_bound = 0.0;
  int32_t best = -1;
  int64_t best_headroom = 0;
  for (int32_t n = 0; n < n_nodes; ++n) {
    const o_res* a = asg + asg_off[n];
    int64_t na = asg_off[n + 1] - asg_off[n];
    if (!o_capacity_holds(kv_capacity[n], a, na, req)) continue;
    double bound = o_oom_bound(a, na, req);
    if (bound > epsilon) continue;
    int64_t reserved = o_res_tokens(req);
    for (int64_t i = 0; i < na; ++i) reserved += o_res_tokens(&a[i]);
    int64_t headroom = kv_capacity[n] - reserved;
    if (best < 0 || headroom > best_headroom ||
        (headroom == best_headroom && staged[n] > staged[best]) ||
        (headroom == best_headroom && staged[n] == staged[best] &&
         replica_id[n] < replica_id[best])) {
      if (best >= 0 && headroom == best_headroom && staged[n] > staged[best]) {
        d.tiebreak = 1;
      } else if (best < 0 || headroom > best_headroom) {
        d.tiebreak = 0;
      }
      best = n;
      best_headroom = headroom;
    }
  }
  if (best >= 0) {
    d.target = replica_id[best];
    d.headroom = best_headroom;
    d.oom_bound = o_oom_bound(asg + asg_off[best], asg_off[best + 1] - asg_off[best], req);
  }
  return d;
}

/* router.cpp:52-62 */
int32_t o_route_least_outstanding(int32_t n_nodes, const int32_t* replica_id,
                                  const int64_t* asg_off) {
  int32_t best = -1;
  for (int32_t n = 0; n < n_nodes; ++n) {
    int64_t sz = asg_off[n + 1] - asg_off[n];
    int64_t bsz = best >= 0 ? asg_off[best + 1] - asg_off[best] : 0;
    if (best < 0 || sz < bsz || (sz == bsz && replica_id[n] < replica_id[best])) best = n;
  }
  return best < 0 ? -1 : replica_id[best];
}

/* ------------------------------------------------------------------ */
/* engine composition                                                  */
/* ------------------------------------------------------------------ */

/* sim/engine.cpp:849-861 */
void o_erase_chain_span(o_tier* t, const uint64_t* tokens, int64_t n, int64_t from, int64_t to,
                        int64_t B) {
  uint64_t* h = (uint64_t*)malloc((size_t)(n_hashes(n, B) + 1) * sizeof(uint64_t));
  int64_t nh = o_chain_hashes(tokens, n, B, h);
  for (int64_t i = 0; i < nh; ++i) {
    int64_t e = (i + 1) * B < n ? (i + 1) * B : n;
    if (e <= from || e > to) continue;
    const o_block* b = o_tier_find(t, h[i]);
    if (b && !(b->pin > 0)) o_tier_erase(t, b->id);
  }
  free(h);
}

static int64_t max3(int64_t a, int64_t b, int64_t c) {
  int64_t m = a > b ? a : b;
  return m > c ? m : c;
}

/* sim/engine.cpp:799-829 (cache side of start_prefill; prefill timing is out of scope) */
int o_admit(o_cache* c, const o_l3* l3_lookup, o_l3* l3_live, const o_registry* reg,
            int speculative, const uint64_t* seq, int64_t len, int32_t wf, int32_t role, double now,
            int64_t B, int64_t match[3]) {
  o_lookup(c, l3_lookup ? l3_lookup : l3_live, seq, len, B, match);
  int64_t needed = len - match[0];
  int64_t nf, ft;
  int ok = o_evict_for_space(c, 0, needed, reg, speculative, NULL, 0, &nf, &ft);
  if (!ok) return 0;
  int64_t reusable = max3(match[0], match[1], match[2]);
  int64_t l2m = reusable < match[1] ? reusable : match[1];
  int64_t l2_part = l2m - match[0] > 0 ? l2m - match[0] : 0;
  int64_t l12 = match[0] > match[1] ? match[0] : match[1];
  int64_t l3_part = reusable - l12 > 0 ? reusable - l12 : 0;
  if (l2_part > 0) o_erase_chain_span(&c->l2, seq, len, match[0], match[0] + l2_part, B);
  if (l3_part > 0) o_erase_chain_span(&l3_live->store, seq, len, l12, reusable, B);
  o_insert_chain(c, 0, seq, len, len, wf, role, now, +1, B);
  return 1;
}

/* sim/engine.cpp:1063-1080 */
void o_completion_policy(o_cache* caches, int32_t n_rep, o_l3* l3, o_registry* reg, int32_t wf,
                         uint64_t future_mask, double now) {
  o_registry_update(reg, wf, future_mask);
  for (int32_t r = 0; r < n_rep; ++r) {
    if (caches[r].off) continue;
    int64_t na = o_on_request_complete(&caches[r], wf, future_mask, 1, NULL, 0);
    o_action* a = (o_action*)malloc((size_t)(na + 1) * sizeof(o_action));
    o_on_request_complete(&caches[r], wf, future_mask, 1, a, na);
    o_apply_completion(a, na, &caches[r], l3, now);
    free(a);
  }
  o_tier* st = &l3->store;
  int64_t n = st->n;
  uint64_t* dead = (uint64_t*)malloc((size_t)(n + 1) * sizeof(uint64_t));
  int64_t nd = 0;
  for (int64_t i = 0; i < n; ++i) {
    const o_block* b = &st->b[i];
    if (!b->alive) continue;
    int live = b->role >= 0 && b->role < 64 && ((future_mask >> b->role) & 1u);
    if (b->wf == wf && !live) dead[nd++] = b->id;
  }
  for (int64_t i = 0; i < nd; ++i) o_tier_erase(st, dead[i]);
  free(dead);
}

/* ------------------------------------------------------------------ */
/* heap constructors for FFI callers (tests / bench)                   */
/* ------------------------------------------------------------------ */

o_cache* o_cache_new(int64_t l1_cap, int64_t l2_cap) {
  o_cache* c = (o_cache*)malloc(sizeof(o_cache));
  o_cache_init(c, l1_cap, l2_cap);
  return c;
}
void o_cache_delete(o_cache* c) {
  o_cache_free(c);
  free(c);
}
o_cache* o_cache_clone(const o_cache* c) {
  o_cache* d = (o_cache*)malloc(sizeof(o_cache));
  *d = *c;
  o_tier_copy(&d->l1, &c->l1);
  o_tier_copy(&d->l2, &c->l2);
  return d;
}
void o_cache_set_off(o_cache* c, int32_t off) { c->off = off; }
void o_add_decode_tokens(o_cache* c, int64_t n) { c->decode_tokens += n; }
o_l3* o_l3_new(void) {
  o_l3* l = (o_l3*)malloc(sizeof(o_l3));
  o_l3_init(l);
  return l;
}
void o_l3_delete(o_l3* l) {
  o_l3_free(l);
  free(l);
}
o_l3* o_l3_clone(const o_l3* l) {
  o_l3* d = (o_l3*)malloc(sizeof(o_l3));
  o_l3_copy(d, l);
  return d;
}
o_registry* o_registry_new(void) {
  o_registry* r = (o_registry*)malloc(sizeof(o_registry));
  o_registry_init(r);
  return r;
}
void o_registry_delete(o_registry* r) {
  o_registry_free(r);
  free(r);
}
/* tier handle for TierStore-level calls: 0 L1, 1 L2, 2 L3 (needs l3) */
o_tier* o_store_of(o_cache* c, o_l3* l3, int32_t tier) {
  if (tier == 2 && l3) return &l3->store;
  return o_cache_tier(c, tier);
}
uint64_t* o_counter_of(o_cache* c, o_l3* l3, int32_t tier) {
  if (tier == 2 && l3) return &l3->next_id;
  return &c->next_id;
}
