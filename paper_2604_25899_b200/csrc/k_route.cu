// k_route.cu -- K3: sched::route (router.cpp:19-50) over a batch.
//
// Node aggregates are built once per batch (capacity_holds is an integer sum,
// router.cpp:7-11; oom_bound an ordered double sum, router.cpp:13-17, kept
// bit-exact by evaluating it in the reference order: request alpha first, then
// the assigned alphas, then -- in SEQ_COMMIT -- the alphas appended by this
// batch's placements).
//
// SNAPSHOT: one warp per request, every request against the same state.
// SEQ_COMMIT (engine.cpp:650-692): requests of one candidate group (model) in
// issue order, each placement committed before the next request.  Requests are
// stably partitioned by group (radix sort); one warp per group keeps its
// candidates' state in shared memory and scans 128 requests per iteration.  A
// request with alpha == +0.0 or alpha == a* (the group's first non-zero
// alpha) is placeable iff its reservation fits the largest free capacity among
// nodes whose bound admits that alpha (F0 / Fa) -- an exact test, so requests
// that fail it wait without a full evaluation; all others are evaluated fully.
// Per-replica placed lists come from a stable radix sort of the targets.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

namespace {

constexpr int kMaxSeqCand = 1024;  // candidates per group held in shared memory

struct NodeScratch {
  int64_t* free_;     // kv_capacity - sum of assigned tokens()
  double* b0;         // oom_bound(node, +0.0) = 0.0 + a_1 + ... (+ appended)
  double* app_alpha;  // [R] appended placement alphas (seq-commit)
  int32_t* app_next;  // [R]
  int32_t* head;      // [n]
  int32_t* tail;      // [n]
};

__device__ __forceinline__ bool same_bits(double a, double b) {
  return __double_as_longlong(a) == __double_as_longlong(b);
}

__global__ void k_node_prep(int n, const pyg_nodes_dev nodes, NodeScratch ns) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t sum = 0;
  double b = 0.0;
  for (int64_t k = nodes.asg_off[i]; k < nodes.asg_off[i + 1]; ++k) {
    const pyg_reservation& a = nodes.asg[k];
    sum += res_tokens(a.prompt_len, a.upper, a.tokens_generated);
    b += a.alpha;
  }
  ns.free_[i] = nodes.kv_capacity[i] - sum;
  ns.b0[i] = b;
  ns.head[i] = -1;
  ns.tail[i] = -1;
}

// alpha + assigned alphas in order + appended placements (router.cpp:13-17)
__device__ __forceinline__ double bound_loop(const pyg_nodes_dev& nodes, const NodeScratch& ns,
                                             int i, double alpha) {
  double b = alpha;
  for (int64_t k = nodes.asg_off[i]; k < nodes.asg_off[i + 1]; ++k) b += nodes.asg[k].alpha;
  for (int32_t q = ns.head[i]; q >= 0; q = ns.app_next[q]) b += ns.app_alpha[q];
  return b;
}

// ---------------------------------------------------------------- SNAPSHOT
__global__ void k_route_snapshot(const pyg_nodes_dev nodes, const NodeScratch ns,
                                 const int32_t* cand_off, const int32_t* cand, int max_cand,
                                 const int32_t* staged, double eps, const pyg_reservation* req,
                                 const int32_t* group, int R, pyg_decision* out, int32_t* t_idx) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= R) return;
  const pyg_reservation q = req[r];
  const int g = group[r];
  const int c0 = cand_off[g], nc = cand_off[g + 1] - c0;
  const int64_t t = res_tokens(q.prompt_len, q.upper, q.tokens_generated);
  const bool z = same_bits(q.alpha, 0.0);
  RouteAcc best{0, 0, 0, -1};
  for (int j = lane; j < nc; j += 32) {
    const int n = cand[c0 + j];
    const int64_t fr = ns.free_[n];
    if (t > fr) continue;
    const double b = z ? ns.b0[n] : bound_loop(nodes, ns, n, q.alpha);
    if (b > eps) continue;
    RouteAcc a{fr - t, staged[static_cast<int64_t>(r) * max_cand + j], nodes.replica_id[n], j};
    if (acc_better(a, best)) best = a;
  }
  best = warp_best(best);
  int32_t p1 = 0x7fffffff, p2 = 0x7fffffff;
  if (best.pos >= 0) {
    for (int j = lane; j < nc; j += 32) {
      const int n = cand[c0 + j];
      const int64_t fr = ns.free_[n];
      if (t > fr || fr - t != best.h) continue;
      const double b = z ? ns.b0[n] : bound_loop(nodes, ns, n, q.alpha);
      if (b > eps) continue;
      p1 = min(p1, j);
      if (staged[static_cast<int64_t>(r) * max_cand + j] == best.s) p2 = min(p2, j);
    }
  }
  p1 = warp_min_i32(p1);
  p2 = warp_min_i32(p2);
  if (lane == 0) {
    pyg_decision d{-1, 0, 0, 0.0};
    int32_t ti = -1;
    if (best.pos >= 0) {
      const int n = cand[c0 + best.pos];
      d.target = best.id;
      d.headroom = best.h;
      d.oom_bound = z ? ns.b0[n] : bound_loop(nodes, ns, n, q.alpha);
      d.tiebreak = p1 < p2 ? 1 : 0;
      ti = n;
    }
    out[r] = d;
    t_idx[r] = ti;
  }
}

// -------------------------------------------------------------- SEQ_COMMIT
struct GroupStat {
  int32_t first_nz;   // smallest request index with alpha != +0.0 (defines a*; INT32_MAX none)
  int32_t count;      // requests in the group
  int32_t n_other;    // requests whose alpha is neither +0.0 nor a*
  int32_t nplaced;    // placements (written by the group's warp)
  int64_t min_t0;     // smallest tokens() among alpha == +0.0 requests
  int64_t min_t1;     // smallest tokens() among alpha == a* requests
};

__global__ void k_gs_init(GroupStat* gs, int G, int32_t* rcount, int32_t* rcur, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < G) gs[i] = GroupStat{INT32_MAX, 0, 0, 0, INT64_MAX, INT64_MAX};
  if (i < n) {
    rcount[i] = 0;
    rcur[i] = 0;
  }
}

// pass 1 (parallel): every decision starts as "wait"; per-group request count
// and first non-zero alpha, reduced in shared memory then once per CTA.
__global__ void k_seq_stats1(const pyg_reservation* req, const int32_t* group, int R, int G,
                             GroupStat* gs, pyg_decision* out, int32_t* t_idx) {
  extern __shared__ int32_t sh[];  // [2G]: first_nz, count
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    sh[g] = INT32_MAX;
    sh[G + g] = 0;
  }
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) {
    const int g = group[r];
    out[r] = pyg_decision{-1, 0, 0, 0.0};
    t_idx[r] = -1;
    atomicAdd(&sh[G + g], 1);
    if (!same_bits(req[r].alpha, 0.0)) atomicMin(&sh[g], r);
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    if (sh[g] != INT32_MAX) atomicMin(&gs[g].first_nz, sh[g]);
    if (sh[G + g]) atomicAdd(&gs[g].count, sh[G + g]);
  }
}

// pass 2 (parallel, one CTA per 128-request chunk): with a* known, per chunk
// and group the smallest tokens() of alpha == +0.0 and alpha == a* requests and
// the count of other alphas.  A chunk can hold a placement only if one of its
// minima fits the current largest free capacity F0 / Fa (exact for those
// classes), so the group's warp skips every other chunk.
__global__ void k_chunk_stats(const pyg_reservation* req, const int32_t* group, int R, int G,
                              GroupStat* gs, int64_t* cmin0, int64_t* cmin1, int32_t* cother,
                              int64_t* smin0, int64_t* smin1, int32_t* sother, int64_t* rt,
                              int32_t* rcls) {
  extern __shared__ int64_t sh64[];  // [2G] minima, then [G] int32 counts
  int32_t* shc = reinterpret_cast<int32_t*>(sh64 + 2 * G);
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    sh64[g] = INT64_MAX;
    sh64[G + g] = INT64_MAX;
    shc[g] = 0;
  }
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) {
    const int g = group[r];
    const pyg_reservation q = req[r];
    const int64_t t = res_tokens(q.prompt_len, q.upper, q.tokens_generated);
    const int32_t f = gs[g].first_nz;
    int cls;
    if (same_bits(q.alpha, 0.0)) {
      cls = 0;
      atomicMin(reinterpret_cast<long long*>(&sh64[g]), t);
    } else if (f != INT32_MAX && same_bits(q.alpha, req[f].alpha)) {
      cls = 1;
      atomicMin(reinterpret_cast<long long*>(&sh64[G + g]), t);
    } else {
      cls = 2;
      atomicAdd(&shc[g], 1);
    }
    rt[r] = t;
    rcls[r] = (g << 2) | cls;  // group and alpha class of the request
  }
  __syncthreads();
  const int sup = blockIdx.x / 32;  // level-2 summary: 32 chunks
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const size_t k = static_cast<size_t>(blockIdx.x) * G + g;
    const size_t k2 = static_cast<size_t>(sup) * G + g;
    cmin0[k] = sh64[g];
    cmin1[k] = sh64[G + g];
    cother[k] = shc[g];
    if (shc[g]) {
      atomicAdd(&gs[g].n_other, shc[g]);
      atomicAdd(&sother[k2], shc[g]);
    }
    if (sh64[g] != INT64_MAX) atomicMin(reinterpret_cast<long long*>(&smin0[k2]), sh64[g]);
    if (sh64[G + g] != INT64_MAX) atomicMin(reinterpret_cast<long long*>(&smin1[k2]), sh64[G + g]);
  }
}

__global__ void k_super_init(int64_t* smin0, int64_t* smin1, int32_t* sother, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    smin0[i] = INT64_MAX;
    smin1[i] = INT64_MAX;
    sother[i] = 0;
  }
}

// group list offsets (exclusive scan of counts); tiny
__global__ void k_group_off(const GroupStat* gs, int G, int32_t* goff) {
  if (threadIdx.x || blockIdx.x) return;
  int32_t a = 0;
  for (int g = 0; g < G; ++g) {
    goff[g] = a;
    a += gs[g].count;
  }
  goff[G] = a;
}

struct SeqArgs {
  pyg_nodes_dev nodes;
  NodeScratch ns;
  const int32_t* cand_off;
  const int32_t* cand;
  int max_cand;
  const int32_t* staged;
  double eps;
  const pyg_reservation* req;
  const int32_t* group;
  int R;
  GroupStat* gs;
  const int32_t* goff;
  int32_t* glist;   // placements per group, in order: request index
  int32_t* rcount;  // placements per replica
  const int64_t* cmin0;  // [nchunks][G] chunk summaries (k_chunk_stats)
  const int64_t* cmin1;
  const int32_t* cother;
  const int64_t* smin0;  // [nchunks/32][G] level-2 summaries
  const int64_t* smin1;
  const int32_t* sother;
  const int64_t* rt;     // [R] tokens()
  const int32_t* rcls;   // [R] group << 2 | alpha class
  int G;
  pyg_decision* out;
  int32_t* t_idx;
};

constexpr int kPer = 4;                 // requests per lane per scan step
constexpr int kScan = 32 * kPer;        // requests per scan step

__global__ void __launch_bounds__(32) k_route_seq(SeqArgs A) {
  __shared__ int64_t s_free[kMaxSeqCand];
  __shared__ double s_b0[kMaxSeqCand];
  __shared__ double s_ba[kMaxSeqCand];
  __shared__ int32_t s_rid[kMaxSeqCand];
  __shared__ int32_t s_node[kMaxSeqCand];
  __shared__ int32_t s_cnt[kMaxSeqCand];
  // wide groups (nc > 32): staged rows of the evaluated request and of the next one,
  // prefetched with cp.async one evaluation ahead
  __shared__ int32_t s_stg[2][kMaxSeqCand];
  int wide_buf = 0, wide_pre = -1;
  const int g = blockIdx.x;
  const int lane = threadIdx.x;
  const int c0 = A.cand_off[g], nc = min(A.cand_off[g + 1] - c0, kMaxSeqCand);
  const GroupStat st = A.gs[g];
  if (st.count == 0) return;
  for (int j = lane; j < nc; j += 32) {
    const int n = A.cand[c0 + j];
    s_node[j] = n;
    s_free[j] = A.ns.free_[n];
    s_b0[j] = A.ns.b0[n];
    s_rid[j] = A.nodes.replica_id[n];
    s_cnt[j] = 0;
  }
  __syncwarp();
  const bool have_star = st.first_nz != INT32_MAX;
  const double astar = have_star ? A.req[st.first_nz].alpha : 0.0;
  if (have_star) {
    for (int j = lane; j < nc; j += 32) s_ba[j] = bound_loop(A.nodes, A.ns, s_node[j], astar);
    __syncwarp();
  }
  // class maxima F0 / Fa of the free capacity over the bound-feasible nodes, and the node
  // holding it when it is unique (u0 / ua, else -1)
  int64_t F0 = INT64_MIN, Fa = INT64_MIN;
  int u0 = -1, ua = -1;
  auto refresh = [&]() {
    int64_t f0 = INT64_MIN, fa = INT64_MIN;
    for (int j = lane; j < nc; j += 32) {
      if (!(s_b0[j] > A.eps)) f0 = max(f0, s_free[j]);
      if (have_star && !(s_ba[j] > A.eps)) fa = max(fa, s_free[j]);
    }
    F0 = redux_max_i64(f0);
    Fa = redux_max_i64(fa);
    int n0 = 0, na = 0, w0 = -1, wa = -1;
    for (int jb = 0; jb < nc; jb += 32) {
      const int j = jb + lane;
      const unsigned m0 = __ballot_sync(kFull, j < nc && !(s_b0[j] > A.eps) && s_free[j] == F0);
      const unsigned ma = __ballot_sync(
          kFull, have_star && j < nc && !(s_ba[j] > A.eps) && s_free[j] == Fa);
      if (m0 && w0 < 0) w0 = jb + __ffs(m0) - 1;
      if (ma && wa < 0) wa = jb + __ffs(ma) - 1;
      n0 += __popc(m0);
      na += __popc(ma);
    }
    u0 = n0 == 1 ? w0 : -1;
    ua = na == 1 ? wa : -1;
  };
  refresh();
  auto bound_of = [&](int j, int cls, double al) -> double {
    if (cls == 0) return s_b0[j];
    if (cls == 1) return s_ba[j];
    return bound_loop(A.nodes, A.ns, s_node[j], al);
  };
  int32_t nplaced = 0;
  const int32_t lbase = A.goff[g];
  const int nchunks = (A.R + kScan - 1) / kScan;
  int next = 0;
  for (;;) {
    // next chunk that can hold a placement under the current state: level-2 summaries
    // (32 chunks each) first, then the 32 chunks of the first promising super-chunk
    int found = -1;
    auto pot = [&](const int64_t* m0, const int64_t* m1, const int32_t* ot, size_t e) {
      return ot[e] > 0 || m0[e] <= F0 || (have_star && m1[e] <= Fa);
    };
    const int nsup = (nchunks + 31) / 32;
    for (int sb = next / 32; sb < nsup && found < 0; sb += 32) {
      const int k2 = sb + lane;
      const bool p2 = k2 < nsup && pot(A.smin0, A.smin1, A.sother, static_cast<size_t>(k2) * A.G + g);
      unsigned m2 = __ballot_sync(kFull, p2);
      while (m2 && found < 0) {
        const int sc = sb + __ffs(m2) - 1;
        m2 &= m2 - 1;
        const int k = sc * 32 + lane;
        const bool p = k >= next && k < nchunks &&
                       pot(A.cmin0, A.cmin1, A.cother, static_cast<size_t>(k) * A.G + g);
        const unsigned m = __ballot_sync(kFull, p);
        if (m) found = sc * 32 + __ffs(m) - 1;
      }
    }
    if (found < 0) break;  // no later request of this group can be placed: all wait
    next = found + 1;
    const int base = found * kScan;
    int64_t t[kPer];
    bool mine[kPer];
    int cl4[kPer];
    {
      const int r0 = base + lane * kPer;
      int32_t cc[kPer];
      int64_t tt4[kPer];
      if (r0 + kPer <= A.R) {
        const int4 c4 = *reinterpret_cast<const int4*>(A.rcls + r0);
        const longlong2 ta = *reinterpret_cast<const longlong2*>(A.rt + r0);
        const longlong2 tb = *reinterpret_cast<const longlong2*>(A.rt + r0 + 2);
        cc[0] = c4.x; cc[1] = c4.y; cc[2] = c4.z; cc[3] = c4.w;
        tt4[0] = ta.x; tt4[1] = ta.y; tt4[2] = tb.x; tt4[3] = tb.y;
      } else {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          cc[u] = r0 + u < A.R ? A.rcls[r0 + u] : -1;
          tt4[u] = r0 + u < A.R ? A.rt[r0 + u] : INT64_MAX;
        }
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        mine[u] = cc[u] >= 0 && (cc[u] >> 2) == g;
        cl4[u] = cc[u] & 3;
        t[u] = mine[u] ? tt4[u] : INT64_MAX;
      }
    }
    int done = base - 1;
    // staged value of candidate `lane` for request pre_r, loaded one evaluation ahead
    int pre_r = -1;
    int32_t pre_v = 0;
    for (;;) {
      int first = INT32_MAX;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int r = base + lane * kPer + u;
        if (!mine[u] || r <= done) continue;
        const int cls = cl4[u];
        const bool could = cls == 0 ? t[u] <= F0 : (cls == 1 ? t[u] <= Fa : true);
        if (could) first = min(first, r);
      }
      first = __reduce_min_sync(kFull, first);
      if (first == INT32_MAX) break;
      const int owner = (first - base) / kPer, uu = (first - base) % kPer;
      int64_t tt = 0;
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if (u == uu) tt = __shfl_sync(kFull, t[u], owner);
      int cl = 0;
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if (u == uu) cl = __shfl_sync(kFull, cl4[u], owner);
      // classes 0 / 1 are bit-identical to +0.0 / a*; only "other" alphas are fetched
      const double a = cl == 0 ? 0.0 : (cl == 1 ? astar : A.req[first].alpha);
      // classes 0 / 1 whose maximum is held by ONE bound-feasible node: that node alone has
      // the largest headroom, so it wins whatever the staged values and p1 == p2 (no
      // tiebreak) -- no staged row, no reductions
      const int uniq = cl == 0 ? u0 : (cl == 1 ? ua : -1);
      RouteAcc best{0, 0, 0, -1};
      int tb = 0;
      if (uniq >= 0) {
        best = RouteAcc{(cl == 0 ? F0 : Fa) - tt, 0, s_rid[uniq], uniq};
      } else {
        // the staged row is read where it is needed (one L2 line per evaluated request);
        // staging every visited chunk's rows in shared memory cost more than it saved once
        // groups interleave (probe: tools/route_probe.py)
        int32_t own_v = 0;
        // the next request of this group in the chunk (narrow groups) / the next one that
        // could fit under the current state (wide groups: a mispredicted row costs a full
        // L2 round trip there)
        int nx = INT32_MAX;
  #pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int r = base + lane * kPer + u;
          if (!mine[u] || r <= first) continue;
          const int cls = cl4[u];
          if (nc <= 32 || (cls == 0 ? t[u] <= F0 : (cls == 1 ? t[u] <= Fa : true))) nx = min(nx, r);
        }
        nx = __reduce_min_sync(kFull, nx);
        if (nc <= 32) {
          // load the next request's value now: its evaluation (usually the next one) then
          // finds its staged value in a register instead of waiting on L2
          own_v = (first == pre_r)
                      ? pre_v
                      : (lane < nc ? A.staged[static_cast<int64_t>(first) * A.max_cand + lane] : 0);
          pre_r = nx;
          if (nx != INT32_MAX && lane < nc) pre_v = A.staged[static_cast<int64_t>(nx) * A.max_cand + lane];
        } else {
          // wide groups: the row was prefetched into s_stg[wide_buf] if `first` is the
          // request predicted last time, else it is loaded now (8 loads in flight per lane)
          asm volatile("cp.async.wait_all;\n" ::);
          __syncwarp();
          if (first != wide_pre) {
            const int32_t* row = A.staged + static_cast<int64_t>(first) * A.max_cand;
            for (int jb = 0; jb < nc; jb += 256) {
              int32_t v[8];
  #pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int j = jb + lane + 32 * i;
                v[i] = j < nc ? row[j] : 0;
              }
  #pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int j = jb + lane + 32 * i;
                if (j < nc) s_stg[wide_buf][j] = v[i];
              }
            }
          }
          __syncwarp();
          // prefetch the next request's row into the other buffer (read one evaluation ago)
          wide_pre = nx;
          if (nx != INT32_MAX) {
            const int32_t* row = A.staged + static_cast<int64_t>(nx) * A.max_cand;
            int32_t* dst = s_stg[wide_buf ^ 1];
            for (int j = lane; j < nc; j += 32) {
              const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + j));
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(row + j));
            }
            asm volatile("cp.async.commit_group;\n" ::);
          }
        }
        const int32_t* stg = s_stg[wide_buf];
        if (nc > 32) wide_buf ^= 1;  // the prefetched row becomes current next time
        auto staged_of = [&](int j) -> int32_t {
          if (nc > 32) return stg[j];
          return j == lane ? own_v : A.staged[static_cast<int64_t>(first) * A.max_cand + j];
        };
        // full sched::route over the group's candidates (router.cpp:24-43): the
        // reference's strict lexicographic running max on (headroom, staged, -replica_id) in
        // input order == argmax of (h, s, -id, -pos); tiebreak <=> first position with
        // headroom H precedes the first with (H, S)
        // classes 0 / 1: headroom order is free-capacity order (tt is fixed per request),
        // so the winners are the bound-feasible nodes whose free capacity equals F0 / Fa
        // (the class maxima refresh() keeps); only that tie set is scanned for staged / id.
        // "Other" alphas need bound_loop per node: full scan.
        const bool by_max = cl < 2;
        const int64_t F = cl == 0 ? F0 : Fa;
        for (int j = lane; j < nc; j += 32) {
          const int64_t fr = s_free[j];
          if (by_max ? (fr != F || tt > fr) : tt > fr) continue;
          if (bound_of(j, cl, a) > A.eps) continue;
          RouteAcc x{fr - tt, staged_of(j), s_rid[j], j};
          if (acc_better(x, best)) best = x;
        }
        const int64_t H = redux_max_i64(best.pos >= 0 ? best.h : INT64_MIN);
        if (H != INT64_MIN) {
          const bool onH = best.pos >= 0 && best.h == H;
          const int64_t S = redux_max_i64(onH ? best.s : INT64_MIN);
          const bool onS = onH && best.s == S;
          const int32_t ID = __reduce_min_sync(kFull, onS ? best.id : INT32_MAX);
          const int32_t POS = __reduce_min_sync(kFull, onS && best.id == ID ? best.pos : INT32_MAX);
          best = RouteAcc{H, S, ID, POS};
        } else {
          best.pos = -1;
        }
        if (best.pos >= 0) {
          int32_t p1 = 0x7fffffff, p2 = 0x7fffffff;
          for (int j = lane; j < nc; j += 32) {
            const int64_t fr = s_free[j];
            if (tt > fr || fr - tt != best.h) continue;
            if (bound_of(j, cl, a) > A.eps) continue;
            p1 = min(p1, j);
            if (staged_of(j) == best.s) p2 = min(p2, j);
          }
          p1 = __reduce_min_sync(kFull, p1);
          p2 = __reduce_min_sync(kFull, p2);
          tb = p1 < p2 ? 1 : 0;
        }
      }
      if (best.pos >= 0) {
        const int w = best.pos;
        if (lane == 0) {
          A.out[first] = pyg_decision{best.id, tb, best.h, bound_of(w, cl, a)};
          const int n = s_node[w];
          A.t_idx[first] = n;
          A.glist[lbase + nplaced] = first;
          s_cnt[w] += 1;
          // commit: the placement joins the node's pool (engine.cpp:686); oom_bound appends
          // its alpha last (router.cpp:15)
          s_free[w] -= tt;
          s_b0[w] += a;
          if (have_star) s_ba[w] += a;
          if (st.n_other) {  // "other" alphas need the full ordered list
            A.ns.app_alpha[first] = a;
            A.ns.app_next[first] = -1;
            if (A.ns.tail[n] >= 0)
              A.ns.app_next[A.ns.tail[n]] = first;
            else
              A.ns.head[n] = first;
            A.ns.tail[n] = first;
          }
        }
        ++nplaced;
        __syncwarp();
        __threadfence_block();
        refresh();
      }
      done = first;
    }
    __syncwarp();
  }
  __syncwarp();
  for (int j = lane; j < nc; j += 32) A.rcount[s_node[j]] = s_cnt[j];
  if (lane == 0) A.gs[g].nplaced = nplaced;
}

// placed_off = exclusive scan of per-replica placement counts (one CTA)
__global__ void k_rep_off(const int32_t* rcount, int n, int32_t* off) {
  __shared__ int64_t sm[64];
  int64_t carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int64_t v = i < n ? rcount[i] : 0;
    int64_t tot;
    const int64_t ex = block_exscan(v, sm, &tot);
    if (i < n) off[i] = static_cast<int32_t>(carry + ex);
    carry += tot;
  }
  if (threadIdx.x == 0) off[n] = static_cast<int32_t>(carry);
}

// per-replica lists in placement (= request) order, from each group's list; one warp per group
__global__ void k_rep_fill(const GroupStat* gs, const int32_t* goff, const int32_t* glist,
                           const int32_t* t_idx, const int32_t* off, int32_t* rcur,
                           int32_t* placed) {
  const int g = blockIdx.x, lane = threadIdx.x;
  const int np = gs[g].nplaced;
  for (int b = 0; b < np; b += 32) {
    const int k = b + lane;
    const bool ok = k < np;
    const int r = ok ? glist[goff[g] + k] : 0;
    const int n = ok ? t_idx[r] : -1;
    const unsigned act = __ballot_sync(kFull, ok);
    const unsigned grp = __match_any_sync(kFull, n) & act;
    const int rank = __popc(grp & lanemask_lt());
    int pos = 0;
    if (ok) pos = off[n] + rcur[n] + rank;
    __syncwarp();
    if (ok) {
      placed[pos] = r;
      if (rank == 0) rcur[n] += __popc(grp);
    }
    __syncwarp();
  }
}

__global__ void k_iota_key(const int32_t* key_src, int R, int add, uint32_t* key, int32_t* val) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  key[r] = static_cast<uint32_t>(key_src[r] + add);
  val[r] = r;
}

// placed_off[n] = first sorted position with key >= n+1 (key = t_idx + 1), minus the waiting
__global__ void k_placed_off(const uint32_t* keys, int R, int n_rep, int32_t* off) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n > n_rep) return;
  auto lb = [&](uint32_t x) {
    int lo = 0, hi = R;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (keys[mid] < x)
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  };
  off[n] = lb(static_cast<uint32_t>(n + 1)) - lb(1u);
}

// placed[i] = v_out[n_wait + i]: the requests with a target, grouped by replica, in order
__global__ void k_placed_copy(const uint32_t* keys, const int32_t* vals, int R, int32_t* placed) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R) return;
  int lo = 0, hi = R;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (keys[mid] < 1u)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo + i < R) placed[i] = vals[lo + i];
}

int bits_for(int x) {
  int b = 1;
  while ((1 << b) <= x) ++b;
  return b;
}

}  // namespace

extern "C" int pyg_route_batch_dev(pyg_ctx* c, int32_t mode, const pyg_nodes_dev* nodes,
                                   const pyg_reservation* d_req, int32_t R,
                                   const int32_t* d_group, int32_t G, const int32_t* d_cand_off,
                                   const int32_t* d_cand, int32_t max_cand,
                                   const int32_t* d_staged, double eps, pyg_decision* d_out,
                                   int32_t* d_placed_off, int32_t* d_placed) {
  PYG_ON_DEVICE(c);
  if (!c || !nodes || R < 0 || G < 0) return PYG_EINVAL;
  if (mode != PYG_ROUTE_SNAPSHOT && mode != PYG_ROUTE_SEQ_COMMIT) {
    set_error("unknown route mode");
    return PYG_EINVAL;
  }
  if (mode == PYG_ROUTE_SEQ_COMMIT && max_cand > kMaxSeqCand) {
    set_error("SEQ_COMMIT supports at most 1024 candidates per group");
    return PYG_ENOTSUP;
  }
  if (mode == PYG_ROUTE_SEQ_COMMIT && G > 1024) {
    set_error("SEQ_COMMIT supports at most 1024 candidate groups");
    return PYG_ENOTSUP;
  }
  const int nchunk = (std::max(R, 1) + kScan - 1) / kScan;
  const int nsup = (nchunk + 31) / 32;
  const int n = c->sharded ? c->n_global : c->n_rep;  // the node table is the whole cluster
  size_t tmp2 = 0;
  const int rbits = bits_for(n + 1);
  PYG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, static_cast<uint32_t*>(nullptr),
                                           static_cast<uint32_t*>(nullptr),
                                           static_cast<int32_t*>(nullptr),
                                           static_cast<int32_t*>(nullptr), R, 0, rbits,
                                           c->stream));
  auto al = [](size_t x) { return (x + 255) & ~size_t{255}; };
  const size_t Rn = static_cast<size_t>(std::max(R, 1));
  const size_t Nn = static_cast<size_t>(std::max(n, 1));
  const size_t bytes = 2 * al(Nn * 8) + al(Rn * 8) + al(Rn * 4) + 4 * al(Nn * 4) + al(Rn * 4) +
                       4 * al(Rn * 4) + al((G + 1) * sizeof(GroupStat)) + al((G + 1) * 4) +
                       al(Rn * 4) + al(tmp2) + 2 * al(static_cast<size_t>(nchunk) * G * 8) +
                       al(static_cast<size_t>(nchunk) * G * 4) +
                       2 * al(static_cast<size_t>(nsup) * G * 8) + al(static_cast<size_t>(nsup) * G * 4) +
                       al(Rn * 8) + al(Rn * 4) + 1024;
  void* sp;
  int rc = scratch(c, bytes, &sp);
  if (rc) return rc;
  char* p = static_cast<char*>(sp);
  auto take = [&](size_t b) {
    char* q = p;
    p += al(b);
    return q;
  };
  NodeScratch ns;
  ns.free_ = reinterpret_cast<int64_t*>(take(Nn * 8));
  ns.b0 = reinterpret_cast<double*>(take(Nn * 8));
  ns.app_alpha = reinterpret_cast<double*>(take(Rn * 8));
  ns.app_next = reinterpret_cast<int32_t*>(take(Rn * 4));
  ns.head = reinterpret_cast<int32_t*>(take(Nn * 4));
  ns.tail = reinterpret_cast<int32_t*>(take(Nn * 4));
  auto* rcount = reinterpret_cast<int32_t*>(take(Nn * 4));
  auto* rcur = reinterpret_cast<int32_t*>(take(Nn * 4));
  auto* t_idx = reinterpret_cast<int32_t*>(take(Rn * 4));
  auto* k_in = reinterpret_cast<uint32_t*>(take(Rn * 4));
  auto* k_out = reinterpret_cast<uint32_t*>(take(Rn * 4));
  auto* v_in = reinterpret_cast<int32_t*>(take(Rn * 4));
  auto* v_out = reinterpret_cast<int32_t*>(take(Rn * 4));
  auto* gs = reinterpret_cast<GroupStat*>(take((G + 1) * sizeof(GroupStat)));
  auto* goff = reinterpret_cast<int32_t*>(take((G + 1) * 4));
  auto* glist = reinterpret_cast<int32_t*>(take(Rn * 4));
  void* d_tmp = take(tmp2);
  auto* cmin0 = reinterpret_cast<int64_t*>(take(static_cast<size_t>(nchunk) * G * 8));
  auto* cmin1 = reinterpret_cast<int64_t*>(take(static_cast<size_t>(nchunk) * G * 8));
  auto* cother = reinterpret_cast<int32_t*>(take(static_cast<size_t>(nchunk) * G * 4));
  auto* smin0 = reinterpret_cast<int64_t*>(take(static_cast<size_t>(nsup) * G * 8));
  auto* smin1 = reinterpret_cast<int64_t*>(take(static_cast<size_t>(nsup) * G * 8));
  auto* sother = reinterpret_cast<int32_t*>(take(static_cast<size_t>(nsup) * G * 4));
  auto* rt = reinterpret_cast<int64_t*>(take(Rn * 8));
  auto* rcls = reinterpret_cast<int32_t*>(take(Rn * 4));
  if (n) {
    k_node_prep<<<(n + 127) / 128, 128, 0, c->stream>>>(n, *nodes, ns);
    PYG_LAUNCHED(c);
  }
  if (mode == PYG_ROUTE_SNAPSHOT) {
    if (R) {
      k_route_snapshot<<<(R + 7) / 8, 256, 0, c->stream>>>(*nodes, ns, d_cand_off, d_cand,
                                                           max_cand, d_staged, eps, d_req,
                                                           d_group, R, d_out, t_idx);
      PYG_LAUNCHED(c);
    }
    if (d_placed_off && d_placed && n) {
      // stable per-replica lists: radix sort of (t_idx + 1) with values = request index
      if (R) {
        k_iota_key<<<(R + 255) / 256, 256, 0, c->stream>>>(t_idx, R, 1, k_in, v_in);
        PYG_LAUNCHED(c);
        PYG_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp2, k_in, k_out, v_in, v_out, R, 0,
                                                 rbits, c->stream));
        PYG_LAUNCHED(c);
      }
      k_placed_off<<<(n + 1 + 127) / 128, 128, 0, c->stream>>>(k_out, R, n, d_placed_off);
      PYG_LAUNCHED(c);
      if (R) {
        k_placed_copy<<<(R + 255) / 256, 256, 0, c->stream>>>(k_out, v_out, R, d_placed);
        PYG_LAUNCHED(c);
      }
    }
    return PYG_OK;
  }
  // SEQ_COMMIT
  const int ginit = std::max(G, n);
  k_gs_init<<<(ginit + 127) / 128 + 1, 128, 0, c->stream>>>(gs, G, rcount, rcur, n);
  PYG_LAUNCHED(c);
  if (R) {
    k_seq_stats1<<<(R + 255) / 256, 256, 2 * G * sizeof(int32_t), c->stream>>>(
        d_req, d_group, R, G, gs, d_out, t_idx);
    PYG_LAUNCHED(c);
    k_super_init<<<(nsup * G + 255) / 256, 256, 0, c->stream>>>(smin0, smin1, sother, nsup * G);
    PYG_LAUNCHED(c);
    k_chunk_stats<<<nchunk, kScan, 2 * G * sizeof(int64_t) + G * sizeof(int32_t), c->stream>>>(
        d_req, d_group, R, G, gs, cmin0, cmin1, cother, smin0, smin1, sother, rt, rcls);
    PYG_LAUNCHED(c);
    k_group_off<<<1, 1, 0, c->stream>>>(gs, G, goff);
    PYG_LAUNCHED(c);
    SeqArgs a{*nodes, ns,  d_cand_off, d_cand, max_cand, d_staged, eps,   d_req,  d_group, R,
              gs,     goff, glist,     rcount, cmin0,    cmin1,    cother, smin0, smin1, sother,
              rt,     rcls, G,         d_out,  t_idx};
    k_route_seq<<<G, 32, 0, c->stream>>>(a);
    PYG_LAUNCHED(c);
  }
  if (d_placed_off && d_placed && n) {
    k_rep_off<<<1, 1024, 0, c->stream>>>(rcount, n, d_placed_off);
    PYG_LAUNCHED(c);
    if (R && G) {
      k_rep_fill<<<G, 32, 0, c->stream>>>(gs, goff, glist, t_idx, d_placed_off, rcur, d_placed);
      PYG_LAUNCHED(c);
    }
  }
  return PYG_OK;
}
