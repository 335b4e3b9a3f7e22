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
struct SeqIn {
  int64_t t;     // reservation tokens()
  double alpha;
};

// Parallel prep over the group-sorted order: tokens(), alpha; every decision
// starts as "wait" (target nullopt, headroom 0, bound 0.0, no tiebreak); group
// ranges; first non-zero-alpha position per group (defines a*).
struct GroupStat {
  int32_t start, end;
  int32_t first_nz;   // position of the first alpha != +0.0 (INT32_MAX: none)
  int32_t n_other;    // requests whose alpha is neither +0.0 nor a*
  int64_t min_t0;     // smallest tokens() among alpha == +0.0 requests
  int64_t min_t1;     // smallest tokens() among alpha == a* requests
};

__device__ __forceinline__ bool seg_head(uint32_t g, int lane) {
  const uint32_t up = __shfl_up_sync(kFull, g, 1);
  return lane == 0 || up != g;
}

template <class T, class Op>
__device__ __forceinline__ T seg_reduce(T v, uint32_t g, int lane, Op op) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_down_sync(kFull, v, o);
    const uint32_t gy = __shfl_down_sync(kFull, g, o);
    if (lane + o < 32 && gy == g) v = op(v, y);
  }
  return v;
}

__global__ void k_seq_prep(const pyg_reservation* req, const int32_t* order,
                           const uint32_t* gkey, int R, SeqIn* in, GroupStat* gs,
                           pyg_decision* out, int32_t* t_idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool ok = i < R;
  const uint32_t g = ok ? gkey[i] : 0xffffffffu;
  int32_t nz = INT32_MAX;
  if (ok) {
    const int r = order[i];
    const pyg_reservation q = req[r];
    in[i] = SeqIn{res_tokens(q.prompt_len, q.upper, q.tokens_generated), q.alpha};
    out[r] = pyg_decision{-1, 0, 0, 0.0};
    t_idx[r] = -1;
    if (i == 0 || gkey[i - 1] != g) gs[g].start = i;
    if (i == R - 1 || gkey[i + 1] != g) gs[g].end = i + 1;
    if (!same_bits(q.alpha, 0.0)) nz = i;
  }
  nz = seg_reduce(nz, g, lane, [](int32_t a, int32_t b) { return a < b ? a : b; });
  if (ok && seg_head(g, lane) && nz != INT32_MAX) atomicMin(&gs[g].first_nz, nz);
}

__global__ void k_seq_classes(const SeqIn* in, const uint32_t* gkey, int R, GroupStat* gs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool ok = i < R;
  const uint32_t g = ok ? gkey[i] : 0xffffffffu;
  int64_t m0 = INT64_MAX, m1 = INT64_MAX;
  int32_t other = 0;
  if (ok) {
    const SeqIn v = in[i];
    const int32_t f = gs[g].first_nz;
    if (same_bits(v.alpha, 0.0))
      m0 = v.t;
    else if (same_bits(v.alpha, in[f].alpha))
      m1 = v.t;
    else
      other = 1;
  }
  auto mn = [](int64_t a, int64_t b) { return a < b ? a : b; };
  m0 = seg_reduce(m0, g, lane, mn);
  m1 = seg_reduce(m1, g, lane, mn);
  other = seg_reduce(other, g, lane, [](int32_t a, int32_t b) { return a + b; });
  if (ok && seg_head(g, lane)) {
    if (m0 != INT64_MAX) atomicMin(reinterpret_cast<long long*>(&gs[g].min_t0), m0);
    if (m1 != INT64_MAX) atomicMin(reinterpret_cast<long long*>(&gs[g].min_t1), m1);
    if (other) atomicAdd(&gs[g].n_other, other);
  }
}

__global__ void k_gs_init(GroupStat* gs, int G) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < G) gs[g] = GroupStat{0, 0, INT32_MAX, 0, INT64_MAX, INT64_MAX};
}

struct SeqArgs {
  pyg_nodes_dev nodes;
  NodeScratch ns;
  const int32_t* cand_off;
  const int32_t* cand;
  int max_cand;
  const int32_t* staged;
  double eps;
  const int32_t* order;
  const SeqIn* in;
  const GroupStat* gs;
  pyg_decision* out;
  int32_t* t_idx;
};

__global__ void __launch_bounds__(32) k_route_seq(SeqArgs A) {
  __shared__ int64_t s_free[kMaxSeqCand];
  __shared__ double s_b0[kMaxSeqCand];
  __shared__ double s_ba[kMaxSeqCand];
  __shared__ int32_t s_rid[kMaxSeqCand];
  __shared__ int32_t s_node[kMaxSeqCand];
  const int g = blockIdx.x;
  const int lane = threadIdx.x;
  const int c0 = A.cand_off[g], nc = min(A.cand_off[g + 1] - c0, kMaxSeqCand);
  const GroupStat st = A.gs[g];
  const int i0 = st.start, i1 = st.end;
  if (i1 <= i0) return;
  for (int j = lane; j < nc; j += 32) {
    const int n = A.cand[c0 + j];
    s_node[j] = n;
    s_free[j] = A.ns.free_[n];
    s_b0[j] = A.ns.b0[n];
    s_rid[j] = A.nodes.replica_id[n];
  }
  __syncwarp();
  const bool have_star = st.first_nz != INT32_MAX;
  const double astar = have_star ? A.in[st.first_nz].alpha : 0.0;
  if (have_star) {
    for (int j = lane; j < nc; j += 32) s_ba[j] = bound_loop(A.nodes, A.ns, s_node[j], astar);
    __syncwarp();
  }
  int64_t F0 = INT64_MIN, Fa = INT64_MIN;
  auto refresh = [&]() {
    int64_t f0 = INT64_MIN, fa = INT64_MIN;
    for (int j = lane; j < nc; j += 32) {
      if (!(s_b0[j] > A.eps)) f0 = max(f0, s_free[j]);
      if (have_star && !(s_ba[j] > A.eps)) fa = max(fa, s_free[j]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      f0 = max(f0, __shfl_xor_sync(kFull, f0, o));
      fa = max(fa, __shfl_xor_sync(kFull, fa, o));
    }
    F0 = f0;
    Fa = fa;
  };
  refresh();
  // bound of node slot j for request alpha al (class 0: +0.0, 1: a*, 2: other)
  auto bound_of = [&](int j, int cls, double al) -> double {
    if (cls == 0) return s_b0[j];
    if (cls == 1) return s_ba[j];
    return bound_loop(A.nodes, A.ns, s_node[j], al);
  };
  // once no remaining request of any class can fit anywhere, the rest wait
  auto saturated = [&]() {
    return st.n_other == 0 && F0 < st.min_t0 && (!have_star || Fa < st.min_t1);
  };
  constexpr int kPer = 4;
  for (int base = i0; base < i1 && !saturated(); base += 32 * kPer) {
    SeqIn v[kPer];
    int cls[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int i = base + lane * kPer + u;
      v[u] = i < i1 ? A.in[i] : SeqIn{INT64_MAX, 0.0};
    }
    int done = base - 1;  // positions <= done are decided
    for (;;) {
      // first position > done whose request could be placed under the current state
      int first = INT32_MAX;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int i = base + lane * kPer + u;
        if (i <= done || i >= i1) continue;
        const bool nz = !same_bits(v[u].alpha, 0.0);
        cls[u] = !nz ? 0 : (same_bits(v[u].alpha, astar) ? 1 : 2);
        const bool could = cls[u] == 0 ? v[u].t <= F0 : (cls[u] == 1 ? v[u].t <= Fa : true);
        if (could) first = min(first, i);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(kFull, first, o));
      if (first == INT32_MAX) break;
      // fetch the request at `first`
      const int owner = (first - base) / kPer, uu = (first - base) % kPer;
      int64_t t = 0;
      double al = 0.0;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        if (u == uu) {
          t = __shfl_sync(kFull, v[u].t, owner);
          al = __shfl_sync(kFull, v[u].alpha, owner);
        }
      }
      const int cl = same_bits(al, 0.0) ? 0 : (same_bits(al, astar) ? 1 : 2);
      const int r = A.order[first];
      // full sched::route over the group's candidates (router.cpp:24-43)
      RouteAcc best{0, 0, 0, -1};
      for (int j = lane; j < nc; j += 32) {
        const int64_t fr = s_free[j];
        if (t > fr) continue;
        if (bound_of(j, cl, al) > A.eps) continue;
        RouteAcc a{fr - t, A.staged[static_cast<int64_t>(r) * A.max_cand + j], s_rid[j], j};
        if (acc_better(a, best)) best = a;
      }
      best = warp_best(best);
      if (best.pos >= 0) {
        int32_t p1 = 0x7fffffff, p2 = 0x7fffffff;
        for (int j = lane; j < nc; j += 32) {
          const int64_t fr = s_free[j];
          if (t > fr || fr - t != best.h) continue;
          if (bound_of(j, cl, al) > A.eps) continue;
          p1 = min(p1, j);
          if (A.staged[static_cast<int64_t>(r) * A.max_cand + j] == best.s) p2 = min(p2, j);
        }
        p1 = warp_min_i32(p1);
        p2 = warp_min_i32(p2);
        const int w = best.pos;
        if (lane == 0) {
          A.out[r] = pyg_decision{best.id, p1 < p2 ? 1 : 0, best.h, bound_of(w, cl, al)};
          const int n = s_node[w];
          A.t_idx[r] = n;
          // commit: the placement joins the node's pool (engine.cpp:686); oom_bound appends its
          // alpha last (router.cpp:15)
          s_free[w] -= t;
          s_b0[w] += al;
          if (have_star) s_ba[w] += al;
          A.ns.app_alpha[first] = al;
          A.ns.app_next[first] = -1;
          if (A.ns.tail[n] >= 0)
            A.ns.app_next[A.ns.tail[n]] = first;
          else
            A.ns.head[n] = first;
          A.ns.tail[n] = first;
        }
        __syncwarp();
        __threadfence_block();
        refresh();
      }
      done = first;
    }
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
  if (!c || !nodes || R < 0 || G < 0) return PYG_EINVAL;
  if (mode != PYG_ROUTE_SNAPSHOT && mode != PYG_ROUTE_SEQ_COMMIT) {
    set_error("unknown route mode");
    return PYG_EINVAL;
  }
  if (mode == PYG_ROUTE_SEQ_COMMIT && max_cand > kMaxSeqCand) {
    set_error("SEQ_COMMIT supports at most 1024 candidates per group");
    return PYG_ENOTSUP;
  }
  const int n = c->n_rep;
  size_t tmp1 = 0, tmp2 = 0;
  const int gbits = bits_for(G), rbits = bits_for(n + 1);
  PYG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp1, static_cast<uint32_t*>(nullptr),
                                           static_cast<uint32_t*>(nullptr),
                                           static_cast<int32_t*>(nullptr),
                                           static_cast<int32_t*>(nullptr), R, 0, gbits,
                                           c->stream));
  PYG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, static_cast<uint32_t*>(nullptr),
                                           static_cast<uint32_t*>(nullptr),
                                           static_cast<int32_t*>(nullptr),
                                           static_cast<int32_t*>(nullptr), R, 0, rbits,
                                           c->stream));
  auto al = [](size_t x) { return (x + 255) & ~size_t{255}; };
  const size_t Rn = static_cast<size_t>(std::max(R, 1));
  const size_t bytes = al(n * 8) + al(n * 8) + al(Rn * 8) + al(Rn * 4) + 2 * al(n * 4) +
                       al(Rn * 4) + 4 * al(Rn * 4) + al(Rn * sizeof(SeqIn)) + al((G + 1) * sizeof(GroupStat)) +
                       al(std::max(tmp1, tmp2)) + 256;
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
  ns.free_ = reinterpret_cast<int64_t*>(take(n * 8));
  ns.b0 = reinterpret_cast<double*>(take(n * 8));
  ns.app_alpha = reinterpret_cast<double*>(take(Rn * 8));
  ns.app_next = reinterpret_cast<int32_t*>(take(Rn * 4));
  ns.head = reinterpret_cast<int32_t*>(take(n * 4));
  ns.tail = reinterpret_cast<int32_t*>(take(n * 4));
  auto* t_idx = reinterpret_cast<int32_t*>(take(Rn * 4));
  auto* k_in = reinterpret_cast<uint32_t*>(take(Rn * 4));
  auto* k_out = reinterpret_cast<uint32_t*>(take(Rn * 4));
  auto* v_in = reinterpret_cast<int32_t*>(take(Rn * 4));
  auto* v_out = reinterpret_cast<int32_t*>(take(Rn * 4));
  auto* sin = reinterpret_cast<SeqIn*>(take(Rn * sizeof(SeqIn)));
  auto* gs = reinterpret_cast<GroupStat*>(take((G + 1) * sizeof(GroupStat)));
  void* d_tmp = take(std::max(tmp1, tmp2));
  if (n) {
    k_node_prep<<<(n + 127) / 128, 128, 0, c->stream>>>(n, *nodes, ns);
    PYG_LAUNCHED(c);
  }
  if (R) {
    if (mode == PYG_ROUTE_SNAPSHOT) {
      k_route_snapshot<<<(R + 7) / 8, 256, 0, c->stream>>>(*nodes, ns, d_cand_off, d_cand,
                                                           max_cand, d_staged, eps, d_req,
                                                           d_group, R, d_out, t_idx);
      PYG_LAUNCHED(c);
    } else {
      // stable partition by group
      k_iota_key<<<(R + 255) / 256, 256, 0, c->stream>>>(d_group, R, 0, k_in, v_in);
      PYG_LAUNCHED(c);
      PYG_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp1, k_in, k_out, v_in, v_out, R, 0, gbits,
                                               c->stream));
      PYG_LAUNCHED(c);
      k_gs_init<<<(G + 127) / 128, 128, 0, c->stream>>>(gs, G);
      PYG_LAUNCHED(c);
      k_seq_prep<<<(R + 255) / 256, 256, 0, c->stream>>>(d_req, v_out, k_out, R, sin, gs, d_out,
                                                         t_idx);
      PYG_LAUNCHED(c);
      k_seq_classes<<<(R + 255) / 256, 256, 0, c->stream>>>(sin, k_out, R, gs);
      PYG_LAUNCHED(c);
      SeqArgs a{*nodes, ns, d_cand_off, d_cand, max_cand, d_staged, eps, v_out, sin, gs, d_out,
                t_idx};
      k_route_seq<<<G, 32, 0, c->stream>>>(a);
      PYG_LAUNCHED(c);
    }
  }
  if (d_placed_off && d_placed && n) {
    // stable per-replica lists: sort (t_idx + 1) with values = request index
    if (R) {
      k_iota_key<<<(R + 255) / 256, 256, 0, c->stream>>>(t_idx, R, 1, k_in, v_in);
      PYG_LAUNCHED(c);
      PYG_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, tmp2, k_in, k_out, v_in, v_out, R, 0, rbits,
                                               c->stream));
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
