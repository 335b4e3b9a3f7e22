// k_nextuse.cu -- K6: workflow-aware next-use prediction from the agent workflow DAG.
//
//   expected_distance_to(cursor, role)   path_analysis.cpp:553-557
//     = first_occurrence(remaining_expr(cursor), role).e_first if p_some > 0
//   future_roles(cursor)                 path_analysis.cpp:547-551 (collect_reachable :338-360)
//
// A path expression is a flattened preorder node table (children after their
// parent), so one bottom-up sweep per role (node ids descending) yields the
// FirstOcc summary of EVERY node (k_fo_table; path_analysis.cpp:408-444) and
// the reachable-role mask of every node (k_reach).  A cursor's remaining
// expression is the sequence of pieces its frames leave behind
// (remaining_expr, path_analysis.cpp:257-290): later children of Seq frames
// and Repeat frames with shifted bounds.  k_next_use folds those pieces with
// seq_compose in the reference's order, one thread per (cursor, role).
//
// FP64 throughout with explicitly rounded __dadd_rn/__dmul_rn/__ddiv_rn: no FMA
// contraction, so each value is the reference's bit for bit (the parity bar
// BASELINE.json states is 1e-6 relative).
#include <cuda_runtime.h>

#include <cmath>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

namespace {

enum : int32_t { kAtom = 0, kSeq = 1, kRepeat = 2, kFanout = 3, kOptional = 4, kTerminal = 5 };

struct FO {  // FirstOcc (path_analysis.cpp:364-369)
  double pn, eln, ps, ef;
};

__device__ __forceinline__ FO fo_default() { return FO{1.0, 0.0, 0.0, 0.0}; }
__device__ __forceinline__ double ad(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mu(double a, double b) { return __dmul_rn(a, b); }

// seq_compose (path_analysis.cpp:374-386)
__device__ __forceinline__ FO seq_compose(const FO& a, const FO& b) {
  FO r = fo_default();
  r.ps = ad(a.ps, mu(a.pn, b.ps));
  if (r.ps > 0.0)
    r.ef = __ddiv_rn(ad(mu(a.ps, a.ef), mu(mu(a.pn, b.ps), ad(a.eln, b.ef))), r.ps);
  r.pn = mu(a.pn, b.pn);
  r.eln = r.pn > 0.0 ? ad(a.eln, b.eln) : 0.0;
  return r;
}

// mix (path_analysis.cpp:388-404), accumulated branch by branch
struct Mix {
  double ps = 0.0, pn = 0.0, first = 0.0, nlen = 0.0;
  __device__ __forceinline__ void add(double w, const FO& o) {
    ps = ad(ps, mu(w, o.ps));
    first = ad(first, mu(mu(w, o.ps), o.ef));
    pn = ad(pn, mu(w, o.pn));
    nlen = ad(nlen, mu(mu(w, o.pn), o.eln));
  }
  __device__ __forceinline__ FO done() const {
    FO r{pn, 0.0, ps, 0.0};
    if (r.ps > 0.0) r.ef = __ddiv_rn(first, r.ps);
    if (r.pn > 0.0) r.eln = __ddiv_rn(nlen, r.pn);
    return r;
  }
};

// repeat_continue_prob / fanout_continue_prob (path_analysis.cpp:14-24)
__device__ __forceinline__ double cont_prob(bool rep, int a, int b, double q, int done) {
  if (done < a) return 1.0;
  if (done >= b) return 0.0;
  if (rep) return q;
  return __ddiv_rn(static_cast<double>(b - done), static_cast<double>(b - done + 1));
}

// Repeat / ParallelFanout branch of first_occurrence (path_analysis.cpp:425-441)
__device__ FO loop_occ(bool rep, int mn, int mx, double q, const FO& child) {
  Mix m;
  FO prefix = fo_default();
  double reach = 1.0;
  for (int done = 0; done <= mx; ++done) {
    const double c = cont_prob(rep, mn, mx, q, done);
    const double stop = mu(reach, ad(1.0, -c));
    if (stop > 0.0) m.add(stop, prefix);
    reach = mu(reach, c);
    if (reach <= 0.0) break;
    prefix = seq_compose(prefix, child);
  }
  return m.done();
}

__device__ FO node_occ(const pyg_path_node& n, const int32_t* ch, const FO* fo, int n_roles,
                       int role) {
  switch (n.kind) {
    case kAtom:
      return n.role == role ? FO{0.0, 0.0, 1.0, 1.0} : FO{1.0, 1.0, 0.0, 0.0};
    case kSeq: {
      FO acc = fo_default();
      for (int k = n.ch_begin; k < n.ch_end; ++k)
        acc = seq_compose(acc, fo[static_cast<int64_t>(ch[k]) * n_roles + role]);
      return acc;
    }
    case kOptional: {
      Mix m;
      m.add(ad(1.0, -n.p), fo_default());
      m.add(n.p, fo[static_cast<int64_t>(n.child) * n_roles + role]);
      return m.done();
    }
    case kRepeat:
    case kFanout:
      return loop_occ(n.kind == kRepeat, n.min, n.max, n.p_continue,
                      fo[static_cast<int64_t>(n.child) * n_roles + role]);
    default:
      return fo_default();
  }
}

// FirstOcc of every node for one role: ids descending (children after parents)
__global__ void k_fo_table(const pyg_path_node* nodes, int n_nodes, const int32_t* ch,
                           int n_roles, FO* fo) {
  const int role = blockIdx.x * blockDim.x + threadIdx.x;
  if (role >= n_roles) return;
  for (int i = n_nodes - 1; i >= 0; --i)
    fo[static_cast<int64_t>(i) * n_roles + role] = node_occ(nodes[i], ch, fo, n_roles, role);
}

// collect_reachable (path_analysis.cpp:338-360) of every node as a role bitmask
__global__ void k_reach(const pyg_path_node* nodes, int n_nodes, const int32_t* ch,
                        uint64_t* reach) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int i = n_nodes - 1; i >= 0; --i) {
    const pyg_path_node& n = nodes[i];
    uint64_t m = 0;
    switch (n.kind) {
      case kAtom: m = (n.role >= 0 && n.role < 64) ? 1ULL << n.role : 0; break;
      case kSeq:
        for (int k = n.ch_begin; k < n.ch_end; ++k) m |= reach[ch[k]];
        break;
      case kOptional: m = n.p > 0.0 ? reach[n.child] : 0; break;
      case kRepeat:
        m = (n.max >= 1 && (n.min >= 1 || n.p_continue > 0.0)) ? reach[n.child] : 0;
        break;
      case kFanout: m = n.max >= 1 ? reach[n.child] : 0; break;
      default: m = 0;
    }
    reach[i] = m;
  }
}

// one thread per (cursor, role): fold the pieces of remaining_expr(cursor)
__global__ void k_next_use(const pyg_path_node* nodes, const int32_t* ch, const FO* fo,
                           const uint64_t* reach, int n_cursors, const int32_t* f_off,
                           const int32_t* f_node, const int32_t* f_prog, int n_roles,
                           double* dist, uint64_t* future) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= static_cast<int64_t>(n_cursors) * n_roles) return;
  const int c = static_cast<int>(x / n_roles), role = static_cast<int>(x % n_roles);
  const int a = f_off[c], b = f_off[c + 1];
  FO acc = fo_default();
  uint64_t m = 0;
  for (int idx = b - 2; idx >= a; --idx) {  // skip the atom frame; inner structures first
    const pyg_path_node& n = nodes[f_node[idx]];
    const int prog = f_prog[idx];
    if (n.kind == kSeq) {
      for (int k = n.ch_begin + prog + 1; k < n.ch_end; ++k) {
        acc = seq_compose(acc, fo[static_cast<int64_t>(ch[k]) * n_roles + role]);
        m |= reach[ch[k]];
      }
    } else if (n.kind == kRepeat) {
      const int done = prog + 1;
      const int rem_max = n.max - done;
      if (rem_max > 0) {
        const int rem_min = n.min - done > 0 ? n.min - done : 0;
        acc = seq_compose(acc, loop_occ(true, rem_min, rem_max, n.p_continue,
                                        fo[static_cast<int64_t>(n.child) * n_roles + role]));
        if (rem_min >= 1 || n.p_continue > 0.0) m |= reach[n.child];
      }
    }
  }
  dist[x] = acc.ps > 0.0 ? acc.ef : __longlong_as_double(0x7ff8000000000000LL);
  if (role == 0) future[c] = m;
}

// predicted next use of every block of a tier, in id order: distance of the block's role
// from its workflow's cursor; NaN when the workflow has no cursor or the role is dead
__global__ void k_block_next_use(const TierDev* tp, const int32_t* wf_cursor, int n_wf,
                                 const double* dist, int n_roles, double* out, int64_t cap,
                                 int64_t* count) {
  __shared__ int64_t sm[64];
  const TierDev& t = *tp;
  int64_t base = 0;
  for (int64_t i0 = 0; i0 < t.log_len; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool alive = i < t.log_len && (t.log[i].flags & kAlive);
    int64_t tot;
    const int64_t pos = base + block_exscan(alive ? 1 : 0, sm, &tot);
    if (alive && pos < cap) {
      const Block& bl = t.log[i];
      double v = __longlong_as_double(0x7ff8000000000000LL);
      if (bl.wf >= 0 && bl.wf < n_wf) {
        const int c = wf_cursor[bl.wf];
        if (c >= 0 && bl.role >= 0 && bl.role < n_roles)
          v = dist[static_cast<int64_t>(c) * n_roles + bl.role];
      }
      out[pos] = v;
    }
    base += tot;
  }
  if (threadIdx.x == 0) *count = base;
}

// FutureRegistry::update from cursors: at issue the engine registers future_roles(cursor)
// plus the current role (engine.cpp:605-609), at completion future_roles only (:1064-1065)
__global__ void k_registry_from_cursors(CtxDev c, int n, const int32_t* wf, const int32_t* cur,
                                        const uint64_t* future, const int32_t* current_role) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int w = wf[i];
  if (w < 0 || w >= c.reg_cap) return;
  uint64_t m = cur[i] >= 0 ? future[cur[i]] : 0;
  if (current_role && current_role[i] >= 0 && current_role[i] < 64) m |= 1ULL << current_role[i];
  c.reg_present[w] = 1;
  c.reg_mask[w] = m;
}

}  // namespace

namespace pyg_host {
int reg_ensure(pyg_ctx* c, int32_t max_wf);  // ops_single.cu
}

extern "C" {

int pyg_next_use_dev(pyg_ctx* c, const pyg_path_node* d_nodes, int32_t n_nodes,
                     const int32_t* d_ch_list, int32_t n_cursors, const int32_t* d_frame_off,
                     const int32_t* d_frame_node, const int32_t* d_frame_prog, int32_t n_roles,
                     double* d_dist, uint64_t* d_future) {
  PYG_ON_DEVICE(c);
  if (!c || n_nodes < 0 || n_cursors < 0 || n_roles < 1 || n_roles > 64) return PYG_EINVAL;
  if (!n_cursors) return PYG_OK;
  auto al = [](size_t x) { return (x + 255) & ~size_t{255}; };
  const size_t b_fo = al(static_cast<size_t>(std::max(n_nodes, 1)) * n_roles * sizeof(FO));
  const size_t b_re = al(static_cast<size_t>(std::max(n_nodes, 1)) * 8);
  void* sp;
  int rc = scratch(c, b_fo + b_re, &sp);
  if (rc) return rc;
  auto* fo = static_cast<FO*>(sp);
  auto* reach = reinterpret_cast<uint64_t*>(static_cast<char*>(sp) + b_fo);
  k_fo_table<<<1, 64, 0, c->stream>>>(d_nodes, n_nodes, d_ch_list, n_roles, fo);
  PYG_LAUNCHED(c);
  k_reach<<<1, 1, 0, c->stream>>>(d_nodes, n_nodes, d_ch_list, reach);
  PYG_LAUNCHED(c);
  const int64_t nq = static_cast<int64_t>(n_cursors) * n_roles;
  k_next_use<<<static_cast<unsigned>((nq + 127) / 128), 128, 0, c->stream>>>(
      d_nodes, d_ch_list, fo, reach, n_cursors, d_frame_off, d_frame_node, d_frame_prog, n_roles,
      d_dist, d_future);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_block_next_use_dev(pyg_ctx* c, int32_t replica, int32_t tier, const int32_t* d_wf_cursor,
                           int32_t n_wf, const double* d_dist, int32_t n_roles, double* d_out,
                           int64_t cap, int64_t* d_count) {
  PYG_ON_DEVICE(c);
  int ti;
  int rc = tier_index(c, replica, tier, false, &ti);
  if (rc) return rc;
  k_block_next_use<<<1, 1024, 0, c->stream>>>(c->d_tiers + ti, d_wf_cursor, n_wf, d_dist,
                                              n_roles, d_out, cap, d_count);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_registry_from_cursors_dev(pyg_ctx* c, int32_t n, int32_t max_wf, const int32_t* d_wf,
                                  const int32_t* d_cursor, const uint64_t* d_future,
                                  const int32_t* d_current_role) {
  PYG_ON_DEVICE(c);
  if (!c || n < 0 || max_wf < 0) return PYG_EINVAL;
  int rc = reg_ensure(c, max_wf);
  if (rc) return rc;
  if (!n) return PYG_OK;
  k_registry_from_cursors<<<(n + 255) / 256, 256, 0, c->stream>>>(c->hd, n, d_wf, d_cursor,
                                                                  d_future, d_current_role);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

}  // extern "C"
