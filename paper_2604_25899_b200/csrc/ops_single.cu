// ops_single.cu -- the drop-in, one-call-per-reference-call API.  Each entry
// point copies its (small) host inputs to the device, runs the kernel that
// restates the reference function, and copies the result back.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

namespace {

// ---------------------------------------------------------------- kernels
struct ChainGet {
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

// CacheHierarchy::insert_chain (hierarchy.cpp:119-130), one warp.
__global__ void k_insert_chain(CtxDev c, int ti, const uint64_t* hashes, int64_t n, int64_t nput,
                               int32_t wf, int32_t role, double now, int32_t pin) {
  ChainGet g{hashes, n, c.B, wf, role};
  warp_put_ordered(c, c.tiers + ti, nput, g, now, pin);
}

struct OneGet {
  PutItem it;
  __device__ PutItem operator()(int64_t) const { return it; }
};

// TierStore::put (hierarchy.cpp:44-66), one warp.
__global__ void k_put(CtxDev c, int ti, PutItem it, double now, int32_t pin, uint64_t* out) {
  OneGet g{it};
  const uint64_t id = warp_put_ordered(c, c.tiers + ti, 1, g, now, pin);
  if (threadIdx.x == 0) *out = id;
}

// TierStore::erase (hierarchy.cpp:68-82): binary search of the id-ordered log.
__global__ void k_erase_id(CtxDev c, int ti, uint64_t id) {
  TierDev* tp = c.tiers + ti;
  const TierDev t = *tp;
  int64_t lo = 0, hi = t.log_len - 1;
  while (lo <= hi) {
    const int64_t mid = (lo + hi) / 2;
    const uint64_t v = t.log[mid].id;
    if (v == id) {
      if (t.log[mid].flags & kAlive) {
        tp->occupancy -= erase_at(t, mid);
        tp->n_alive -= 1;
      }
      return;
    }
    if (v < id)
      lo = mid + 1;
    else
      hi = mid - 1;
  }
}

// TierStore::erase of a list of ids, in order (one thread: each is a binary search)
__global__ void k_erase_ids(CtxDev c, int ti, const uint64_t* ids, int64_t n) {
  TierDev* tp = c.tiers + ti;
  const TierDev t = *tp;
  int64_t occ = 0, cnt = 0;
  for (int64_t k = 0; k < n; ++k) {
    const uint64_t id = ids[k];
    int64_t lo = 0, hi = t.log_len - 1;
    while (lo <= hi) {
      const int64_t mid = (lo + hi) / 2;
      const uint64_t v = t.log[mid].id;
      if (v == id) {
        if (t.log[mid].flags & kAlive) {
          occ += erase_at(t, mid);
          cnt += 1;
        }
        break;
      }
      if (v < id)
        lo = mid + 1;
      else
        hi = mid - 1;
    }
  }
  tp->occupancy -= occ;
  tp->n_alive -= cnt;
}

struct PutListGet {
  const pyg_put_item* items;
  __device__ PutItem operator()(int64_t i) const {
    const pyg_put_item x = items[i];
    return PutItem{x.chain_hash, 0, x.span_start, x.span_end, x.workflow, x.role, 1};
  }
};

// TierStore::put of a list of blocks, in order (one warp, warp_put_ordered)
__global__ void k_put_list(CtxDev c, int ti, const pyg_put_item* items, int64_t n, double now,
                           int32_t pin) {
  warp_put_ordered(c, c.tiers + ti, n, PutListGet{items}, now, pin);
}

__global__ void k_find(CtxDev c, int ti, uint64_t hash, pyg_block* out, int32_t* found) {
  const TierDev t = c.tiers[ti];
  const int64_t li = idx_find(t, hash);
  *found = li >= 0;
  if (li >= 0) {
    const Block& b = t.log[li];
    *out = pyg_block{b.id, b.hash, b.s, b.e, b.wf, b.role, b.la, b.pin, 1};
  }
}

// Applies f(leader lane, log index, multiplicity) to the blocks of a chain
// whose span_end <= upto (or in (from, to]), deduplicated per chunk.
// unpin_chain (hierarchy.cpp:132-142): L1 only, pin-- if pin > 0, per occurrence.
__global__ void k_unpin(CtxDev c, int ti, const uint64_t* hashes, int64_t nput) {
  const TierDev t = c.tiers[ti];
  const int lane = threadIdx.x & 31;
  for (int64_t base = 0; base < nput; base += 32) {
    const int64_t i = base + lane;
    const bool active = i < nput;
    const uint64_t key = active ? hashes[i] : 0;
    const unsigned am = __ballot_sync(kFull, active);
    const unsigned grp = __match_any_sync(kFull, key) & am;
    if (active && (__ffs(grp) - 1) == lane) {
      const int64_t li = idx_find(t, key);
      if (li >= 0) {
        int32_t p = t.log[li].pin;
        for (int k = __popc(grp); k > 0 && p > 0; --k) --p;
        t.log[li].pin = p;
      }
    }
    __syncwarp();
  }
}

// Engine::erase_chain_span (engine.cpp:849-861): blocks with from < span_end <= to,
// erased if present and unpinned.
__global__ void k_erase_span(CtxDev c, int ti, const uint64_t* hashes, int64_t n, int64_t from,
                             int64_t to) {
  TierDev* tp = c.tiers + ti;
  const TierDev t = *tp;
  const int lane = threadIdx.x & 31;
  const int64_t nh = blocks_of(n, c.B);
  int64_t freed = 0, cnt = 0;
  for (int64_t base = 0; base < nh; base += 32) {
    const int64_t i = base + lane;
    bool active = false;
    uint64_t key = 0;
    if (i < nh) {
      const int64_t e = min((i + 1) * c.B, n);
      active = !(e <= from || e > to);
      key = hashes[i];
    }
    const unsigned am = __ballot_sync(kFull, active);
    const unsigned grp = __match_any_sync(kFull, key) & am;
    if (active && (__ffs(grp) - 1) == lane) {
      const int64_t li = idx_find(t, key);
      if (li >= 0 && !(t.log[li].pin > 0)) {
        freed += erase_at(t, li);
        cnt += 1;
      }
    }
    __syncwarp();
  }
  freed = warp_sum(freed);
  cnt = warp_sum(cnt);
  if (lane == 0) {
    tp->occupancy -= freed;
    tp->n_alive -= cnt;
  }
}

// TierStore::matched_prefix (hierarchy.cpp:84-104) on up to 3 tiers, one warp.
__global__ void k_lookup(CtxDev c, int t0, int t1, int t2, const uint64_t* tokens, int64_t n,
                         const uint64_t* hashes, int64_t* out) {
  const int lane = threadIdx.x & 31;
  const int tis[3] = {t0, t1, t2};
  for (int k = 0; k < 3; ++k) {
    if (tis[k] < 0) {
      if (lane == 0) out[k] = 0;
      continue;
    }
    const TierDev t = c.tiers[tis[k]];
    const int64_t nh = blocks_of(n, c.B);
    const int64_t kb = warp_walk(t, hashes, nh);
    int64_t m = kb ? matched_from_blocks(kb, n, c.B) : 0;
    if (lane == 0) out[k] = ragged_extend(t, t.log, tokens, n, hashes, m, c.B);
    __syncwarp();
  }
}

// CacheHierarchy::lookup (hierarchy.cpp:109-117) of ONE prompt on replicas [0, n_rep): a
// warp per (replica, tier) -- the engine's node_view loop (engine.cpp:640-648) in one launch.
__global__ void k_lookup_all(CtxDev c, int n_rep, int with_l3, const uint64_t* tokens, int64_t n,
                             const uint64_t* hashes, int64_t* out) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= 3 * n_rep) return;
  const int rep = w / 3, k = w % 3;
  if (k == 2 && !with_l3) {
    if (lane == 0) out[3 * rep + 2] = 0;
    return;
  }
  const TierDev t = c.tiers[k < 2 ? 2 * rep + k : 2 * c.n_rep];
  const int64_t nh = blocks_of(n, c.B);
  const int64_t kb = warp_walk(t, hashes, nh);
  const int64_t m = kb ? matched_from_blocks(kb, n, c.B) : 0;
  if (lane == 0) out[3 * rep + k] = ragged_extend(t, t.log, tokens, n, hashes, m, c.B);
}

__global__ void __launch_bounds__(512) k_evict(CtxDev c, int ti, int rep_for_decode, int64_t needed, int spec,
                        uint64_t* out_ids, int64_t cap, int64_t* out_stats) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t sm[64];
  TierDev* tp = c.tiers + ti;
  // evict_for_space: base = l1_occupancy() for L1, occupancy() otherwise (manager.cpp:106-107)
  const int64_t base = tp->occupancy + (rep_for_decode >= 0 ? c.decode[rep_for_decode] : 0);
  const int64_t excess = base + needed - tp->capacity;
  __syncthreads();
  const EvictOut r = block_evict(c, tp, excess, spec, out_ids, cap, smem, sm);
  if (threadIdx.x == 0) {
    out_stats[0] = r.n_freed;
    out_stats[1] = r.freed_tokens;
    out_stats[2] = r.satisfied;
  }
}

__global__ void k_add_decode(CtxDev c, int rep, int64_t n) { c.decode[rep] += n; }

// on_request_complete (manager.cpp:25-42), first half: per replica, Free
// actions are applied (erase) and Retain actions are appended, in action
// order (L1 then L2, ascending id), to the replica's retain list.
__global__ void k_complete_collect(CtxDev c, int32_t wf, uint64_t future, const int32_t* reps,
                                   int nreps, PutItem* lists, const int64_t* list_off,
                                   int64_t* list_len, int64_t* n_actions) {
  __shared__ int64_t sm[64];
  const int rep = reps[blockIdx.x];
  int64_t nret = 0, nact = 0;
  for (int tier = 0; tier < 2; ++tier) {
    TierDev* tp = c.tiers + 2 * rep + tier;
    const TierDev t = *tp;
    int64_t freed = 0, nfree = 0;
    for (int64_t base = 0; base < t.log_len; base += blockDim.x) {
      const int64_t i = base + threadIdx.x;
      bool act = false, keep = false;
      if (i < t.log_len) {
        const Block& b = t.log[i];
        act = (b.flags & kAlive) && !(b.pin > 0) && b.wf == wf;
        keep = act && b.role >= 0 && b.role < 64 && ((future >> b.role) & 1ULL);
      }
      int64_t tot;
      const int64_t pos = nret + block_exscan(keep ? 1 : 0, sm, &tot);
      int64_t tact;
      block_exscan(act ? 1 : 0, sm, &tact);
      if (keep) {
        const Block& b = t.log[i];
        PutItem it;
        it.hash = b.hash;
        it.parent = b.parent;
        it.s = b.s;
        it.e = b.e;
        it.wf = b.wf;
        it.role = b.role;
        it.orphan = (b.flags & kOrphan) ? 1 : 0;
        lists[list_off[blockIdx.x] + pos] = it;
      } else if (act) {
        freed += erase_at(t, i);
        nfree += 1;
      }
      nret += tot;
      nact += tact;
    }
    int64_t ft, nf;
    block_exscan(freed, sm, &ft);
    block_exscan(nfree, sm, &nf);
    if (threadIdx.x == 0) {
      tp->occupancy -= ft;
      tp->n_alive -= nf;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    list_len[blockIdx.x] = nret;
    n_actions[blockIdx.x] = nact;
  }
}

struct ListGet {
  const PutItem* items;
  __device__ PutItem operator()(int64_t i) const { return items[i]; }
};

// apply_completion's RetainAndWriteL3 (manager.cpp:51-56): L3 puts in replica
// order then action order (the engine sweeps replicas in order,
// engine.cpp:1068-1073), one warp.
__global__ void k_complete_l3put(CtxDev c, const PutItem* lists, const int64_t* list_off,
                                 const int64_t* list_len, int nreps, double now) {
  for (int k = 0; k < nreps; ++k) {
    ListGet g{lists + list_off[k]};
    warp_put_ordered(c, c.tiers + 2 * c.n_rep, list_len[k], g, now, 0);
  }
}

// L3 dead-lineage erase (engine.cpp:1074-1080); erasures commute.
__global__ void k_l3_dead_sweep(CtxDev c, int32_t wf, uint64_t future) {
  TierDev* tp = c.tiers + 2 * c.n_rep;
  const TierDev t = *tp;
  int64_t freed = 0, cnt = 0;
  for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < t.log_len;
       i += gridDim.x * blockDim.x) {
    const Block& b = t.log[i];
    if (!(b.flags & kAlive) || b.wf != wf) continue;
    const bool live = b.role >= 0 && b.role < 64 && ((future >> b.role) & 1ULL);
    if (!live) {
      freed += erase_at(t, i);
      cnt += 1;
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

__global__ void k_reg_set(CtxDev c, int32_t wf, uint8_t present, uint64_t mask) {
  c.reg_present[wf] = present;
  c.reg_mask[wf] = mask;
}

// FutureRegistry::update for a batch of distinct workflows (a burst's issue-time updates,
// engine.cpp:605-609, last write per workflow).  Out-of-range ids set the error flag.
__global__ void k_reg_set_batch(CtxDev c, int32_t n, const int32_t* wf, const uint64_t* mask) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t w = wf[i];
  if (w < 0 || w >= c.reg_cap) {
    atomicExch(c.error, 6);
    return;
  }
  c.reg_mask[w] = mask[i];
  c.reg_present[w] = 1;
}

__global__ void k_dump(CtxDev c, int ti, pyg_block* out, int64_t cap, int64_t* count) {
  __shared__ int64_t sm[64];
  const TierDev t = c.tiers[ti];
  int64_t write = 0;
  for (int64_t base = 0; base < t.log_len; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool alive = i < t.log_len && (t.log[i].flags & kAlive);
    int64_t tot;
    const int64_t pos = write + block_exscan(alive ? 1 : 0, sm, &tot);
    if (alive && pos < cap) {
      const Block& b = t.log[i];
      out[pos] = pyg_block{b.id, b.hash, b.s, b.e, b.wf, b.role, b.la, b.pin, 1};
    }
    write += tot;
  }
  if (threadIdx.x == 0) *count = write;
}

// sched::route (router.cpp:19-50) for one request; one warp, lanes over nodes.
__global__ void k_route_one(int32_t nn, const int32_t* rid, const int64_t* cap,
                            const int64_t* off, const pyg_reservation* asg, const int64_t* staged,
                            pyg_reservation req, double eps, pyg_decision* out) {
  const int lane = threadIdx.x;
  const int64_t treq = res_tokens(req.prompt_len, req.upper, req.tokens_generated);
  RouteAcc best{0, 0, 0, -1};
  for (int32_t n = lane; n < nn; n += 32) {
    int64_t total = treq;
    double bound = req.alpha;
    for (int64_t k = off[n]; k < off[n + 1]; ++k) {
      total += res_tokens(asg[k].prompt_len, asg[k].upper, asg[k].tokens_generated);
      bound += asg[k].alpha;
    }
    if (total > cap[n]) continue;  // capacity_holds
    if (bound > eps) continue;
    RouteAcc a{cap[n] - total, staged[n], rid[n], n};
    if (acc_better(a, best)) best = a;
  }
  best = warp_best(best);
  // tiebreak flag: first position with headroom H vs first with (H, S)
  int32_t p1 = 0x7fffffff, p2 = 0x7fffffff;
  if (best.pos >= 0) {
    for (int32_t n = lane; n < nn; n += 32) {
      int64_t total = treq;
      double bound = req.alpha;
      for (int64_t k = off[n]; k < off[n + 1]; ++k) {
        total += res_tokens(asg[k].prompt_len, asg[k].upper, asg[k].tokens_generated);
        bound += asg[k].alpha;
      }
      if (total > cap[n] || bound > eps) continue;
      if (cap[n] - total == best.h) {
        p1 = min(p1, n);
        if (staged[n] == best.s) p2 = min(p2, n);
      }
    }
  }
  p1 = warp_min_i32(p1);
  p2 = warp_min_i32(p2);
  if (lane == 0) {
    pyg_decision d{-1, 0, 0, 0.0};
    if (best.pos >= 0) {
      d.target = best.id;
      d.headroom = best.h;
      double bound = req.alpha;
      for (int64_t k = off[best.pos]; k < off[best.pos + 1]; ++k) bound += asg[k].alpha;
      d.oom_bound = bound;
      d.tiebreak = p1 < p2 ? 1 : 0;
    }
    *out = d;
  }
}

// ------------------------------------------------------------ host helpers
// The sequence on the device + its boundary hashes, with room for 64 int64 of outputs
// after the hashes (at *d_hash + nh + 1).  Memoized: the same tokens as the last call reuse
// the device copy (no upload, no hashing).
int upload_tokens(pyg_ctx* c, const uint64_t* tokens, int64_t n, uint64_t** d_tok,
                  uint64_t** d_hash) {
  const int64_t nh = (n + c->B - 1) / c->B;
  const size_t need = static_cast<size_t>(n + nh + 8 + 64) * sizeof(uint64_t) + 64;
  if (c->memo_valid && static_cast<int64_t>(c->memo_tokens.size()) == n &&
      (n == 0 || std::memcmp(c->memo_tokens.data(), tokens, n * sizeof(uint64_t)) == 0)) {
    *d_tok = static_cast<uint64_t*>(c->memo);
    *d_hash = *d_tok + n + 4;
    return PYG_OK;
  }
  if (need > c->memo_size) {
    if (c->memo) {
      PYG_CUDA(cudaStreamSynchronize(c->stream));
      PYG_CUDA(cudaFree(c->memo));
      c->memo = nullptr;
    }
    const size_t sz = std::max<size_t>(need * 2, 1 << 16);
    PYG_CUDA(cudaMalloc(&c->memo, sz));
    c->memo_size = sz;
  }
  c->memo_valid = false;
  *d_tok = static_cast<uint64_t*>(c->memo);
  *d_hash = *d_tok + n + 4;
  if (n) {
    PYG_CUDA(cudaMemcpyAsync(*d_tok, tokens, n * sizeof(uint64_t), cudaMemcpyHostToDevice,
                             c->stream));
    int rc = hash_seq_launch(c, *d_tok, n, *d_hash);
    if (rc) return rc;
  }
  c->memo_tokens.assign(tokens, tokens + n);
  c->memo_valid = true;
  return PYG_OK;
}

// number of chain blocks with span_end <= upto (hierarchy.cpp:125-127)
int64_t blocks_upto(int64_t n, int64_t upto, int B) {
  const int64_t nh = (n + B - 1) / B;
  if (upto >= n) return nh;
  if (upto <= 0) return 0;
  return std::min<int64_t>(nh, upto / B);
}

}  // namespace

// ------------------------------------------------------------------- C-ABI
extern "C" {

int pyg_chain_hashes(pyg_ctx* c, const uint64_t* tokens, int64_t n, uint64_t* out,
                     int64_t* n_out) {
  PYG_ON_DEVICE(c);
  if (!c || n < 0 || (n && (!tokens || !out))) return PYG_EINVAL;
  uint64_t *dt, *dh;
  int rc = upload_tokens(c, tokens, n, &dt, &dh);
  if (rc) return rc;
  const int64_t nh = (n + c->B - 1) / c->B;
  if (nh)
    PYG_CUDA(cudaMemcpyAsync(out, dh, nh * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  if (n_out) *n_out = nh;
  return PYG_OK;
}

int pyg_tier_put(pyg_ctx* c, int32_t replica, int32_t tier, uint64_t hash, int64_t s, int64_t e,
                 int32_t wf, int32_t role, double now, int32_t pin, uint64_t* out_id) {
  PYG_ON_DEVICE(c);
  if (c) dir_touch(c);  // may change an L2 tier: the directory is rebuilt before use
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  if (e < s) {
    set_error("span_end < span_start");
    return PYG_EINVAL;
  }
  if ((rc = ensure_capacity(c, ti, 1))) return rc;
  void* sp;
  if ((rc = scratch(c, 64, &sp))) return rc;
  PutItem it{hash, 0, s, e, wf, role, 1};
  k_put<<<1, 32, 0, c->stream>>>(c->hd, ti, it, now, pin, static_cast<uint64_t*>(sp));
  PYG_LAUNCHED(c);
  uint64_t id = 0;
  PYG_CUDA(cudaMemcpyAsync(&id, sp, 8, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  if (out_id) *out_id = id;
  return PYG_OK;
}

int pyg_tier_erase(pyg_ctx* c, int32_t replica, int32_t tier, uint64_t id) {
  PYG_ON_DEVICE(c);
  if (c) dir_touch(c);  // may change an L2 tier: the directory is rebuilt before use
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  k_erase_id<<<1, 1, 0, c->stream>>>(c->hd, ti, id);
  PYG_LAUNCHED(c);
  return PYG_OK;  // stream-ordered: nothing to return, later calls see the erase
}

int pyg_tier_erase_many(pyg_ctx* c, int32_t replica, int32_t tier, const uint64_t* ids,
                        int64_t n) {
  PYG_ON_DEVICE(c);
  if (c) dir_touch(c);
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  if (n < 0 || (n && !ids)) return PYG_EINVAL;
  if (!n) return PYG_OK;
  void* sp;
  if ((rc = aux(c, static_cast<size_t>(n) * 8 + 64, &sp))) return rc;
  // pageable source: the copy is staged before the call returns, the host list may go
  PYG_CUDA(cudaMemcpyAsync(sp, ids, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice,
                           c->stream));
  k_erase_ids<<<1, 1, 0, c->stream>>>(c->hd, ti, static_cast<const uint64_t*>(sp), n);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_tier_put_many(pyg_ctx* c, int32_t replica, int32_t tier, const pyg_put_item* items,
                      int64_t n, double now, int32_t pin) {
  PYG_ON_DEVICE(c);
  if (c) dir_touch(c);
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  if (n < 0 || (n && !items)) return PYG_EINVAL;
  if (!n) return PYG_OK;
  for (int64_t k = 0; k < n; ++k)
    if (items[k].span_end < items[k].span_start) {
      set_error("span_end < span_start");
      return PYG_EINVAL;
    }
  if ((rc = ensure_capacity(c, ti, n))) return rc;
  void* sp;
  if ((rc = aux(c, static_cast<size_t>(n) * sizeof(pyg_put_item) + 64, &sp))) return rc;
  PYG_CUDA(cudaMemcpyAsync(sp, items, static_cast<size_t>(n) * sizeof(pyg_put_item),
                           cudaMemcpyHostToDevice, c->stream));
  k_put_list<<<1, 32, 0, c->stream>>>(c->hd, ti, static_cast<const pyg_put_item*>(sp), n, now,
                                      pin);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_tier_find(pyg_ctx* c, int32_t replica, int32_t tier, uint64_t hash, pyg_block* out,
                  int32_t* found) {
  PYG_ON_DEVICE(c);
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  void* sp;
  if ((rc = scratch(c, sizeof(pyg_block) + 16, &sp))) return rc;
  auto* db = static_cast<pyg_block*>(sp);
  auto* df = reinterpret_cast<int32_t*>(db + 1);
  k_find<<<1, 1, 0, c->stream>>>(c->hd, ti, hash, db, df);
  PYG_LAUNCHED(c);
  pyg_block b{};
  int32_t f = 0;
  PYG_CUDA(cudaMemcpyAsync(&b, db, sizeof(b), cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaMemcpyAsync(&f, df, 4, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  if (found) *found = f;
  if (out && f) *out = b;
  return PYG_OK;
}

int pyg_tier_stats(pyg_ctx* c, int32_t replica, int32_t tier, int64_t* occ, int64_t* cap,
                   int64_t* nb) {
  PYG_ON_DEVICE(c);
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  TierDev t;
  if ((rc = read_tier(c, ti, &t))) return rc;
  if (occ) *occ = t.occupancy;
  if (cap) *cap = t.capacity;
  if (nb) *nb = t.n_alive;
  return PYG_OK;
}

int pyg_tier_dump(pyg_ctx* c, int32_t replica, int32_t tier, pyg_block* out, int64_t cap,
                  int64_t* n) {
  PYG_ON_DEVICE(c);
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  TierDev t;
  if ((rc = read_tier(c, ti, &t))) return rc;
  const int64_t want = std::min<int64_t>(std::max<int64_t>(cap, 0), t.n_alive);
  void* sp;
  if ((rc = scratch(c, (want + 1) * sizeof(pyg_block) + 16, &sp))) return rc;
  auto* db = static_cast<pyg_block*>(sp);
  auto* dn = reinterpret_cast<int64_t*>(db + want + 1);
  k_dump<<<1, 1024, 0, c->stream>>>(c->hd, ti, db, want, dn);
  PYG_LAUNCHED(c);
  int64_t cnt = 0;
  PYG_CUDA(cudaMemcpyAsync(&cnt, dn, 8, cudaMemcpyDeviceToHost, c->stream));
  if (want && out)
    PYG_CUDA(cudaMemcpyAsync(out, db, want * sizeof(pyg_block), cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  if (n) *n = cnt;
  return PYG_OK;
}

int pyg_matched_prefix(pyg_ctx* c, int32_t replica, int32_t tier, const uint64_t* tokens,
                       int64_t n, int64_t* out) {
  PYG_ON_DEVICE(c);
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  if (n < 0 || (n && !tokens) || !out) return PYG_EINVAL;
  uint64_t *dt, *dh;
  if ((rc = upload_tokens(c, tokens, n, &dt, &dh))) return rc;
  int64_t* dout = reinterpret_cast<int64_t*>(dh + (n + c->B - 1) / c->B + 1);
  k_lookup<<<1, 32, 0, c->stream>>>(c->hd, ti, -1, -1, dt, n, dh, dout);
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaMemcpyAsync(out, dout, 8, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int pyg_lookup(pyg_ctx* c, int32_t replica, const uint64_t* tokens, int64_t n, int32_t with_l3,
               int64_t out[3]) {
  PYG_ON_DEVICE(c);
  if (!c || replica < 0 || replica >= c->n_rep || n < 0 || (n && !tokens) || !out) {
    set_error("pyg_lookup: bad arguments");
    return PYG_EINVAL;
  }
  uint64_t *dt, *dh;
  int rc = upload_tokens(c, tokens, n, &dt, &dh);
  if (rc) return rc;
  int64_t* dout = reinterpret_cast<int64_t*>(dh + (n + c->B - 1) / c->B + 1);
  k_lookup<<<1, 32, 0, c->stream>>>(c->hd, 2 * replica, 2 * replica + 1,
                                    with_l3 ? 2 * c->n_rep : -1, dt, n, dh, dout);
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaMemcpyAsync(out, dout, 24, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int pyg_lookup_all(pyg_ctx* c, const uint64_t* tokens, int64_t n, int32_t with_l3,
                   int32_t n_rep, int64_t* out) {
  PYG_ON_DEVICE(c);
  if (!c || n < 0 || (n && !tokens) || !out || n_rep < 0 || n_rep > c->n_rep) {
    set_error("pyg_lookup_all: bad arguments");
    return PYG_EINVAL;
  }
  if (!n_rep) return PYG_OK;
  uint64_t *dt, *dh;
  int rc = upload_tokens(c, tokens, n, &dt, &dh);
  if (rc) return rc;
  void* sp;
  if ((rc = scratch(c, static_cast<size_t>(n_rep) * 24 + 64, &sp))) return rc;
  auto* dout = static_cast<int64_t*>(sp);
  const int warps = 3 * n_rep;
  k_lookup_all<<<(warps + 3) / 4, 128, 0, c->stream>>>(c->hd, n_rep, with_l3, dt, n, dh, dout);
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaMemcpyAsync(out, dout, static_cast<size_t>(n_rep) * 24, cudaMemcpyDeviceToHost,
                           c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int pyg_insert_chain(pyg_ctx* c, int32_t replica, int32_t tier, const uint64_t* tokens, int64_t n,
                     int64_t upto, int32_t wf, int32_t role, double now, int32_t pin) {
  PYG_ON_DEVICE(c);
  if (c) dir_touch(c);  // may change an L2 tier: the directory is rebuilt before use
  int ti;
  int rc = tier_index(c, replica, tier, true, &ti);
  if (rc) return rc;
  if (n < 0 || (n && !tokens)) return PYG_EINVAL;
  const int64_t nput = blocks_upto(n, upto, c->B);
  if (nput == 0) return PYG_OK;
  if ((rc = ensure_capacity(c, ti, nput))) return rc;
  uint64_t *dt, *dh;
  if ((rc = upload_tokens(c, tokens, n, &dt, &dh))) return rc;
  k_insert_chain<<<1, 32, 0, c->stream>>>(c->hd, ti, dh, n, nput, wf, role, now, pin);
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int pyg_unpin_chain(pyg_ctx* c, int32_t replica, const uint64_t* tokens, int64_t n,
                    int64_t upto) {
  PYG_ON_DEVICE(c);
  if (!c || replica < 0 || replica >= c->n_rep || n < 0 || (n && !tokens)) return PYG_EINVAL;
  const int64_t nput = blocks_upto(n, upto, c->B);
  if (nput == 0) return PYG_OK;
  uint64_t *dt, *dh;
  int rc = upload_tokens(c, tokens, n, &dt, &dh);
  if (rc) return rc;
  k_unpin<<<1, 32, 0, c->stream>>>(c->hd, 2 * replica, dh, nput);
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int pyg_erase_chain_span(pyg_ctx* c, int32_t replica, int32_t tier, const uint64_t* tokens,
                         int64_t n, int64_t from, int64_t to) {
  PYG_ON_DEVICE(c);
  if (c) dir_touch(c);  // may change an L2 tier: the directory is rebuilt before use
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  if (n < 0 || (n && !tokens)) return PYG_EINVAL;
  if (n == 0) return PYG_OK;
  uint64_t *dt, *dh;
  if ((rc = upload_tokens(c, tokens, n, &dt, &dh))) return rc;
  k_erase_span<<<1, 32, 0, c->stream>>>(c->hd, ti, dh, n, from, to);
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int pyg_add_decode_tokens(pyg_ctx* c, int32_t replica, int64_t n) {
  PYG_ON_DEVICE(c);
  if (!c || replica < 0 || replica >= c->n_rep) return PYG_EINVAL;
  k_add_decode<<<1, 1, 0, c->stream>>>(c->hd, replica, n);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_l1_occupancy(pyg_ctx* c, int32_t replica, int64_t* out) {
  PYG_ON_DEVICE(c);
  if (!c || replica < 0 || replica >= c->n_rep || !out) return PYG_EINVAL;
  TierDev t;
  int rc = read_tier(c, 2 * replica, &t);
  if (rc) return rc;
  int64_t dec = 0;
  PYG_CUDA(cudaMemcpy(&dec, c->hd.decode + replica, 8, cudaMemcpyDeviceToHost));
  *out = t.occupancy + dec;  // hierarchy.hpp:114
  return PYG_OK;
}

int pyg_set_replica_off(pyg_ctx* c, int32_t replica, int32_t off) {
  PYG_ON_DEVICE(c);
  if (!c || replica < 0 || replica >= c->n_rep) return PYG_EINVAL;
  int32_t v = off ? 1 : 0;
  PYG_CUDA(cudaMemcpyAsync(c->hd.off + replica, &v, 4, cudaMemcpyHostToDevice, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

static int reg_grow(pyg_ctx* c, int32_t wf) {
  if (wf < c->hd.reg_cap) return PYG_OK;
  int32_t nc = c->hd.reg_cap;
  while (nc <= wf) nc *= 2;
  uint8_t* np = nullptr;
  uint64_t* nm = nullptr;
  PYG_CUDA(cudaMalloc(&np, nc));
  PYG_CUDA(cudaMalloc(&nm, nc * sizeof(uint64_t)));
  PYG_CUDA(cudaMemsetAsync(np, 0, nc, c->stream));
  PYG_CUDA(cudaMemsetAsync(nm, 0, nc * sizeof(uint64_t), c->stream));
  PYG_CUDA(cudaMemcpyAsync(np, c->hd.reg_present, c->hd.reg_cap, cudaMemcpyDeviceToDevice,
                           c->stream));
  PYG_CUDA(cudaMemcpyAsync(nm, c->hd.reg_mask, c->hd.reg_cap * sizeof(uint64_t),
                           cudaMemcpyDeviceToDevice, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  cudaFree(c->hd.reg_present);
  cudaFree(c->hd.reg_mask);
  c->hd.reg_present = np;
  c->hd.reg_mask = nm;
  c->hd.reg_cap = nc;
  return PYG_OK;
}


int pyg_registry_update(pyg_ctx* c, int32_t wf, uint64_t mask) {
  PYG_ON_DEVICE(c);
  if (!c || wf < 0) return PYG_EINVAL;
  int rc = reg_grow(c, wf);
  if (rc) return rc;
  k_reg_set<<<1, 1, 0, c->stream>>>(c->hd, wf, 1, mask);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_registry_update_batch_dev(pyg_ctx* c, int32_t n, const int32_t* d_wf,
                                  const uint64_t* d_mask, int32_t max_wf) {
  PYG_ON_DEVICE(c);
  if (!c || n < 0 || max_wf < 0) return PYG_EINVAL;
  if (!n) return PYG_OK;
  PYG_CUDA(cudaSetDevice(c->device));
  int rc = reg_grow(c, max_wf);
  if (rc) return rc;
  k_reg_set_batch<<<(n + 255) / 256, 256, 0, c->stream>>>(c->hd, n, d_wf, d_mask);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_registry_reserve(pyg_ctx* c, int32_t max_wf) {
  PYG_ON_DEVICE(c);
  if (!c || max_wf < 0) return PYG_EINVAL;
  return reg_grow(c, max_wf);
}

int pyg_registry_drop(pyg_ctx* c, int32_t wf) {
  PYG_ON_DEVICE(c);
  if (!c || wf < 0) return PYG_EINVAL;
  if (wf >= c->hd.reg_cap) return PYG_OK;
  k_reg_set<<<1, 1, 0, c->stream>>>(c->hd, wf, 0, 0);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_evict_for_space(pyg_ctx* c, int32_t replica, int32_t tier, int64_t needed,
                        int32_t speculative, uint64_t* freed, int64_t cap, int64_t* n_freed,
                        int64_t* freed_tokens, int32_t* satisfied) {
  PYG_ON_DEVICE(c);
  if (c) dir_touch(c);  // may change an L2 tier: the directory is rebuilt before use
  int ti;
  int rc = tier_index(c, replica, tier, true, &ti);
  if (rc) return rc;
  TierDev t;
  if ((rc = read_tier(c, ti, &t))) return rc;
  const int64_t room = std::max<int64_t>(cap, 0);
  void* sp;
  if ((rc = scratch(c, (room + 8) * sizeof(uint64_t), &sp))) return rc;
  auto* dstats = static_cast<int64_t*>(sp);
  auto* dids = reinterpret_cast<uint64_t*>(dstats + 4);
  const size_t smem = kSmemSortCap * 12;
  PYG_CUDA(cudaFuncSetAttribute(k_evict, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_evict<<<1, 512, smem, c->stream>>>(c->hd, ti, tier == 0 ? replica : -1, needed,
                                        speculative, dids, room, dstats);
  PYG_LAUNCHED(c);
  int64_t st[3];
  PYG_CUDA(cudaMemcpyAsync(st, dstats, 24, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  const int64_t k = std::min(st[0], room);
  if (k && freed)
    PYG_CUDA(cudaMemcpyAsync(freed, dids, k * 8, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  if (n_freed) *n_freed = st[0];
  if (freed_tokens) *freed_tokens = st[1];
  if (satisfied) *satisfied = static_cast<int32_t>(st[2]);
  return PYG_OK;
}

static int complete_reps(pyg_ctx* c, const std::vector<int32_t>& reps, int32_t wf,
                         uint64_t future, double now, int64_t* n_actions) {
  const int nr = static_cast<int>(reps.size());
  if (nr == 0) {
    if (n_actions) *n_actions = 0;
    return PYG_OK;
  }
  std::vector<int64_t> off(nr + 1, 0);
  for (int k = 0; k < nr; ++k) {
    TierDev a, b;
    int rc = read_tier(c, 2 * reps[k], &a);
    if (rc) return rc;
    if ((rc = read_tier(c, 2 * reps[k] + 1, &b))) return rc;
    off[k + 1] = off[k] + a.log_len + b.log_len;
  }
  const size_t need = off[nr] * sizeof(PutItem) + (3 * nr + 8) * sizeof(int64_t) + nr * 4 + 64;
  if (need > c->d_list_size) {
    if (c->d_list) {
      PYG_CUDA(cudaStreamSynchronize(c->stream));
      cudaFree(c->d_list);
    }
    PYG_CUDA(cudaMalloc(&c->d_list, need * 2));
    c->d_list_size = need * 2;
  }
  auto* items = static_cast<PutItem*>(c->d_list);
  auto* doff = reinterpret_cast<int64_t*>(items + off[nr]);
  auto* dlen = doff + nr + 1;
  auto* dact = dlen + nr;
  auto* dreps = reinterpret_cast<int32_t*>(dact + nr);
  PYG_CUDA(cudaMemcpyAsync(doff, off.data(), (nr + 1) * 8, cudaMemcpyHostToDevice, c->stream));
  PYG_CUDA(cudaMemcpyAsync(dreps, reps.data(), nr * 4, cudaMemcpyHostToDevice, c->stream));
  k_complete_collect<<<nr, 1024, 0, c->stream>>>(c->hd, wf, future, dreps, nr, items, doff, dlen,
                                                 dact);
  PYG_LAUNCHED(c);
  std::vector<int64_t> len(nr), act(nr);
  PYG_CUDA(cudaMemcpyAsync(len.data(), dlen, nr * 8, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaMemcpyAsync(act.data(), dact, nr * 8, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  int64_t tot = 0, tact = 0;
  for (int k = 0; k < nr; ++k) {
    tot += len[k];
    tact += act[k];
  }
  if (tot) {
    int rc = ensure_capacity(c, 2 * c->n_rep, tot);
    if (rc) return rc;
    k_complete_l3put<<<1, 32, 0, c->stream>>>(c->hd, items, doff, dlen, nr, now);
    PYG_LAUNCHED(c);
  }
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  if (n_actions) *n_actions = tact;
  return PYG_OK;
}

int pyg_complete(pyg_ctx* c, int32_t replica, int32_t wf, uint64_t future, int32_t profiled,
                 double now, int64_t* n_actions) {
  PYG_ON_DEVICE(c);
  if (c) dir_touch(c);  // may change an L2 tier: the directory is rebuilt before use
  if (!c || replica < 0 || replica >= c->n_rep) return PYG_EINVAL;
  if (!profiled) {  // req.unprofiled() => no actions (manager.cpp:28)
    if (n_actions) *n_actions = 0;
    return PYG_OK;
  }
  return complete_reps(c, {replica}, wf, future, now, n_actions);
}

int pyg_l3_dead_sweep(pyg_ctx* c, int32_t wf, uint64_t future) {
  PYG_ON_DEVICE(c);
  if (!c) return PYG_EINVAL;
  k_l3_dead_sweep<<<148, 256, 0, c->stream>>>(c->hd, wf, future);
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int pyg_completion_policy(pyg_ctx* c, int32_t wf, uint64_t future, double now) {
  PYG_ON_DEVICE(c);
  if (c) dir_touch(c);  // may change an L2 tier: the directory is rebuilt before use
  if (!c || wf < 0) return PYG_EINVAL;
  int rc = pyg_registry_update(c, wf, future);  // engine.cpp:1064-1065
  if (rc) return rc;
  std::vector<int32_t> off(c->n_rep);
  if (c->n_rep)
    PYG_CUDA(cudaMemcpy(off.data(), c->hd.off, c->n_rep * 4, cudaMemcpyDeviceToHost));
  std::vector<int32_t> reps;
  for (int r = 0; r < c->n_rep; ++r)
    if (!off[r]) reps.push_back(r);  // engine.cpp:1069
  int64_t na;
  if ((rc = complete_reps(c, reps, wf, future, now, &na))) return rc;
  return pyg_l3_dead_sweep(c, wf, future);
}

int pyg_route(pyg_ctx* c, int32_t nn, const int32_t* rid, const int64_t* kv, const int64_t* off,
              const pyg_reservation* asg, const int64_t* staged, const pyg_reservation* req,
              double eps, pyg_decision* out) {
  PYG_ON_DEVICE(c);
  if (!c || nn < 0 || !req || !out || (nn && (!rid || !kv || !off || !staged))) return PYG_EINVAL;
  const int64_t na = nn ? off[nn] : 0;
  const size_t bytes = nn * 4 + nn * 8 * 3 + 8 + na * sizeof(pyg_reservation) + 64 + 256;
  void* sp;
  int rc = scratch(c, bytes, &sp);
  if (rc) return rc;
  char* p = static_cast<char*>(sp);
  auto* d_dec = reinterpret_cast<pyg_decision*>(p);
  p += 64;
  auto* d_asg = reinterpret_cast<pyg_reservation*>(p);
  p += na * sizeof(pyg_reservation);
  auto* d_cap = reinterpret_cast<int64_t*>(p);
  p += nn * 8;
  auto* d_off = reinterpret_cast<int64_t*>(p);
  p += (nn + 1) * 8;
  auto* d_st = reinterpret_cast<int64_t*>(p);
  p += nn * 8;
  auto* d_rid = reinterpret_cast<int32_t*>(p);
  if (nn) {
    if (na) PYG_CUDA(cudaMemcpyAsync(d_asg, asg, na * sizeof(pyg_reservation), cudaMemcpyHostToDevice, c->stream));
    PYG_CUDA(cudaMemcpyAsync(d_cap, kv, nn * 8, cudaMemcpyHostToDevice, c->stream));
    PYG_CUDA(cudaMemcpyAsync(d_off, off, (nn + 1) * 8, cudaMemcpyHostToDevice, c->stream));
    PYG_CUDA(cudaMemcpyAsync(d_st, staged, nn * 8, cudaMemcpyHostToDevice, c->stream));
    PYG_CUDA(cudaMemcpyAsync(d_rid, rid, nn * 4, cudaMemcpyHostToDevice, c->stream));
  }
  k_route_one<<<1, 32, 0, c->stream>>>(nn, d_rid, d_cap, d_off, d_asg, d_st, *req, eps, d_dec);
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaMemcpyAsync(out, d_dec, sizeof(pyg_decision), cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int pyg_route_least_outstanding(pyg_ctx* c, int32_t nn, const int32_t* rid, const int64_t* off,
                                int32_t* out) {
  PYG_ON_DEVICE(c);
  // route_least_outstanding (router.cpp:52-62): fewest assigned, ties to lowest id.
  // Evaluated with the route kernel: headroom = -assigned count, staged 0.
  if (!c || nn < 0 || !out) return PYG_EINVAL;
  std::vector<int64_t> kv(nn), zoff(nn + 1, 0), st(nn, 0);
  for (int n = 0; n < nn; ++n) kv[n] = -(off[n + 1] - off[n]) + (int64_t{1} << 40);
  pyg_reservation req{0, 0, 0.0, 0};
  pyg_decision d;
  int rc = pyg_route(c, nn, rid, kv.data(), zoff.data(), nullptr, st.data(), &req, 1.0, &d);
  if (rc) return rc;
  *out = d.target;
  return PYG_OK;
}

}  // extern "C"

namespace pyg_host {
int reg_ensure(pyg_ctx* c, int32_t max_wf) { return reg_grow(c, max_wf); }
}  // namespace pyg_host
