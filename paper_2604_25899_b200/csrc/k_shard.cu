// k_shard.cu -- the multi-GPU step's data movement over NVLink peer memory.
//
// After every GPU has routed the whole burst (identical decisions everywhere),
// the owner of each target replica PULLS the placed requests' tokens and boundary
// hashes straight out of the origin GPU's HBM (CUDA IPC mappings of the peer's
// buffers, NVLink P2P loads), admits them, and the other GPUs read the owner's
// exported L2/L3 erase lists and admission results the same way.  No host
// round trip sits inside the step: every size the kernels need is bounded by
// capacity_holds (router.cpp:7-11) -- the prompt tokens placed on a replica
// never exceed its kv_capacity -- and the actual counts stay on the device.
//
//   k_recv_flag / CUB select   global requests placed on my replicas, ascending
//   k_recv_lens + CUB scan     their token / hash offsets in my receive buffers
//   k_pull                     peer -> local copy of tokens and hashes
//   k_local_placed             global per-replica placed lists -> local indices
//   k_apply_lists              every shard's L3 erasures + others' L2 clears
//   k_results                  origin reads admitted / match3 from the owner
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <cstring>
#include <map>
#include <string>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

namespace {

__device__ __forceinline__ int owner_of(const int64_t* rep_off, int world, int rep) {
  int lo = 0, hi = world;  // rep_off[k] <= rep < rep_off[k+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (rep_off[mid] <= rep) lo = mid;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int src_of(const int64_t* req_off, int world, int64_t r) {
  int lo = 0, hi = world;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (req_off[mid] <= r) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct IsMine {
  const pyg_decision* dec;
  int32_t lo, hi;
  __device__ __forceinline__ bool operator()(const int32_t& r) const {
    const int t = dec[r].target;
    return t >= lo && t < hi;
  }
};

__global__ void k_clamp(int64_t* count, int64_t cap, int32_t* err) {
  if (*count > cap) {
    *count = cap;
    atomicExch(err, 5);
  }
}

__global__ void k_iota(int32_t* x, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = static_cast<int32_t>(i);
}

// k-th received request (0 beyond the count): global index, lineage and token / hash counts,
// read from the origin shard's HBM (peer loads)
__global__ void k_recv_lens(const int32_t* sel, const int64_t* count, const pyg_peer* peers,
                            int world, const int64_t* req_off, int64_t cap, int B, int32_t* gidx,
                            int32_t* wf, int32_t* role, int64_t* tl, int64_t* hl) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k > cap) return;
  const bool in = k < *count;
  const int32_t g = in ? sel[k] : 0;
  int64_t L = 0;
  int32_t w = 0, ro = 0;
  if (in) {
    const int s = src_of(req_off, world, g);
    const pyg_peer& p = peers[s];
    const int64_t li = g - req_off[s];
    L = p.tok_off[li + 1] - p.tok_off[li];
    w = p.workflow[li];
    ro = p.role[li];
  }
  tl[k] = L;
  hl[k] = (L + B - 1) / B;
  if (k < cap) {
    gidx[k] = g;
    wf[k] = w;
    role[k] = ro;
  }
}

__global__ void k_pack(const pyg_reservation* req, const int32_t* group, const int32_t* staged,
                       int R, int mc, int s16, int32_t* rows, int32_t* err) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int wd = 5 + (s16 ? (mc + 1) / 2 : mc);
  int32_t* o = rows + static_cast<int64_t>(r) * wd;
  const pyg_reservation q = req[r];
  const int64_t t = res_tokens(q.prompt_len, q.upper, q.tokens_generated);
  const int64_t ab = __double_as_longlong(q.alpha);
  o[0] = static_cast<int32_t>(t);
  o[1] = static_cast<int32_t>(t >> 32);
  o[2] = static_cast<int32_t>(ab);
  o[3] = static_cast<int32_t>(ab >> 32);
  o[4] = group[r];
  const int32_t* st = staged + static_cast<int64_t>(r) * mc;
  if (s16) {
    // 16-bit staged values: a prompt of >= 65536 tokens (staged value > 0xffff) would be
    // truncated -- flag it (error 7) so the caller switches to 32-bit rows
    for (int j = 0; j < mc; ++j)
      if (static_cast<uint32_t>(st[j]) > 0xffffu) atomicExch(err, 7);
    for (int j = 0; j < mc; j += 2) {
      const uint32_t lo = static_cast<uint32_t>(st[j]) & 0xffffu;
      const uint32_t hi = j + 1 < mc ? (static_cast<uint32_t>(st[j + 1]) & 0xffffu) : 0u;
      o[5 + j / 2] = static_cast<int32_t>(lo | (hi << 16));
    }
  } else {
    for (int j = 0; j < mc; ++j) o[5 + j] = st[j];
  }
}

__global__ void k_unpack(const int32_t* rows, int R, int mc, int s16, pyg_reservation* req,
                         int32_t* group, int32_t* staged) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int wd = 5 + (s16 ? (mc + 1) / 2 : mc);
  const int32_t* o = rows + static_cast<int64_t>(r) * wd;
  const int64_t t = (static_cast<int64_t>(o[1]) << 32) | static_cast<uint32_t>(o[0]);
  const int64_t ab = (static_cast<int64_t>(o[3]) << 32) | static_cast<uint32_t>(o[2]);
  req[r] = pyg_reservation{t, 0, __longlong_as_double(ab), 0};
  group[r] = o[4];
  int32_t* st = staged + static_cast<int64_t>(r) * mc;
  if (s16) {
    for (int j = 0; j < mc; ++j)
      st[j] = static_cast<int32_t>((static_cast<uint32_t>(o[5 + j / 2]) >> (16 * (j & 1))) & 0xffffu);
  } else {
    for (int j = 0; j < mc; ++j) st[j] = o[5 + j];
  }
}

// Unpack the whole burst's route rows straight from every shard's row buffer over NVLink
// (rows_of[k] = shard k's rows, mapped in this process): the NCCL all-gather's replacement.
// One warp per 32 rows: lane l unpacks row r0+l's reservation and group, then the warp
// copies each row's staged values one candidate per lane (coalesced 128-byte stores).
// own_mask (groups < 64; 0 = all): the staged row is only read for the requests of groups
// this shard routes -- the others are never evaluated here.
__global__ void k_unpack_peer(const int64_t* rows_of, int world, const int64_t* req_off, int R,
                              int mc, int s16, uint64_t own_mask, pyg_reservation* req,
                              int32_t* group, int32_t* staged) {
  const int lane = threadIdx.x & 31;
  const int r0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32;
  if (r0 >= R) return;
  const int wd = 5 + (s16 ? (mc + 1) / 2 : mc);
  const int r = r0 + lane;
  const int32_t* o = nullptr;
  bool own = false;
  if (r < R) {
    const int k = src_of(req_off, world, r);
    o = reinterpret_cast<const int32_t*>(rows_of[k]) + static_cast<int64_t>(r - req_off[k]) * wd;
    const int64_t t = (static_cast<int64_t>(o[1]) << 32) | static_cast<uint32_t>(o[0]);
    const int64_t ab = (static_cast<int64_t>(o[3]) << 32) | static_cast<uint32_t>(o[2]);
    req[r] = pyg_reservation{t, 0, __longlong_as_double(ab), 0};
    const int g = o[4];
    group[r] = g;
    own = own_mask == 0 || g < 0 || g >= 64 || ((own_mask >> g) & 1ULL);
  }
  unsigned todo = __ballot_sync(kFull, own);
  while (todo) {
    const int l = __ffs(todo) - 1;
    todo &= todo - 1;
    const int32_t* src = reinterpret_cast<const int32_t*>(
        __shfl_sync(kFull, reinterpret_cast<unsigned long long>(o), l));
    int32_t* st = staged + static_cast<int64_t>(r0 + l) * mc;
    for (int j = lane; j < mc; j += 32) {
      st[j] = s16 ? static_cast<int32_t>((static_cast<uint32_t>(src[5 + j / 2]) >> (16 * (j & 1))) &
                                         0xffffu)
                  : src[5 + j];
    }
  }
}

// Cross-GPU stream barrier over peer memory.  signal: after a system-scope fence (this
// stream's earlier writes -- rows, lists -- are visible to the peers first), store seq into
// slot [me] of every shard's flag array with release semantics.  wait: spin (acquire) until
// all `world` slots of this shard's own flag array reach seq; a peer that never arrives
// (timeout ~10 s) raises the device error instead of hanging the GPU.
__global__ void k_signal(const int64_t* flag_of, int world, int me, int64_t seq) {
  const int k = threadIdx.x;
  __threadfence_system();
  if (k < world) {
    int64_t* f = reinterpret_cast<int64_t*>(flag_of[k]) + me;
    asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(f), "l"(seq) : "memory");
  }
}

__global__ void k_wait(const int64_t* flags, int world, int64_t seq, int32_t* err,
                       const unsigned long long* cond) {
  if (cond && *cond == 0) return;  // nothing depends on the peers' data this time
  const int k = threadIdx.x;
  if (k < world) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      int64_t v;
      asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(flags + k) : "memory");
      if (v >= seq) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10000000000ull) {
        atomicExch(err, 5);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
}

__global__ void k_pull(const pyg_peer* peers, int world, const int64_t* req_off,
                       const int32_t* gidx, const int64_t* count, const int64_t* toff,
                       const int64_t* hoff, uint64_t* tok_out, uint64_t* hash_out,
                       int64_t tok_cap, int64_t hash_cap, int32_t* err) {
  const int64_t n = *count;
  for (int64_t k = blockIdx.x; k < n; k += gridDim.x) {
    const int64_t r = gidx[k];
    const int s = src_of(req_off, world, r);
    const pyg_peer& p = peers[s];
    const int64_t li = r - req_off[s];
    const int64_t a = p.tok_off[li], len = p.tok_off[li + 1] - a;
    const int64_t ha = p.hash_off[li], hn = p.hash_off[li + 1] - ha;
    if (toff[k] + len > tok_cap || hoff[k] + hn > hash_cap) {  // broken capacity invariant
      if (threadIdx.x == 0) atomicExch(err, 6);
      continue;
    }
    const uint64_t* st = p.tokens + a;
    uint64_t* dt = tok_out + toff[k];
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) dt[i] = st[i];
    const uint64_t* sh = p.hashes + ha;
    uint64_t* dh = hash_out + hoff[k];
    for (int64_t i = threadIdx.x; i < hn; i += blockDim.x) dh[i] = sh[i];
  }
}

// placed_off/placed: global CSR over every replica (global request indices in placement
// order).  Output: CSR over my replicas of positions in my receive list.
__global__ void k_local_placed(const int32_t* placed_off, const int32_t* placed, int rep_lo,
                               int n_local, const int32_t* gidx, const int64_t* count,
                               int32_t* p_off, int32_t* p_loc) {
  const int32_t a = placed_off[rep_lo];
  const int32_t e = placed_off[rep_lo + n_local];
  for (int i = threadIdx.x; i <= n_local; i += blockDim.x) p_off[i] = placed_off[rep_lo + i] - a;
  const int64_t n = *count;
  for (int32_t q = a + static_cast<int32_t>(blockIdx.x * blockDim.x + threadIdx.x); q < e;
       q += gridDim.x * blockDim.x) {
    const int32_t g = placed[q];
    int64_t lo = 0, hi = n;  // lower_bound
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (gidx[mid] < g) lo = mid + 1;
      else hi = mid;
    }
    p_loc[q - a] = static_cast<int32_t>(lo);
  }
}

__global__ void k_apply_lists(CtxDev c, const pyg_peer* peers, int world, int me, int l3_lo,
                              int l3_hi, int with_l2, const unsigned long long* cond) {
  if (cond && *cond == 0) return;
  TierDev* tp = c.tiers + 2 * c.n_rep;
  for (int k = 0; k < world; ++k) {
    const pyg_peer& p = peers[k];
    const int64_t n3 = k >= l3_lo && k < l3_hi ? p.list_counts[1] : 0;
    int64_t freed = 0, cnt = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n3;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t sl = idx_find_slot(*tp, p.l3_list[i]);
      if (sl < 0) continue;
      unsigned long long* pv = reinterpret_cast<unsigned long long*>(&tp->idx[sl].val);
      const unsigned long long v = *reinterpret_cast<volatile unsigned long long*>(pv);
      if (v == 0 || v == kTomb) continue;
      Block& b = tp->log[v - 1];
      if (b.pin > 0) continue;
      if (atomicCAS(pv, v, static_cast<unsigned long long>(kTomb)) != v) continue;
      b.flags &= ~kAlive;
      freed += b.e - b.s;
      cnt += 1;
    }
    if (cnt) {
      atomicAdd(reinterpret_cast<unsigned long long*>(&tp->occupancy),
                static_cast<unsigned long long>(-freed));
      atomicAdd(reinterpret_cast<unsigned long long*>(&tp->n_alive),
                static_cast<unsigned long long>(-cnt));
    }
    if (k == me || !with_l2 || !c.dir_main) continue;
    const int64_t n2 = p.list_counts[0];
    const DirRecord* rec = static_cast<const DirRecord*>(p.l2_list);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n2;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const DirRecord r = rec[i];
      dir_clear_bit(c.dir_main, c.dir_main_mask, c.dir_stride, dir_key(r.hash), r.replica);
      if (r.s % c.B == 0 && r.e % c.B != 0 && r.e > r.s)
        dir_clear_bit(c.dir_rver, c.dir_rver_mask, c.dir_stride, rver_key(r.hash, r.s, r.e),
                      r.replica);
    }
  }
}

__global__ void k_results(const pyg_peer* peers, int world, const int64_t* rep_off,
                          const pyg_decision* dec, int64_t req_base, int64_t R,
                          int32_t* adm, int64_t* m3) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int t = dec[req_base + r].target;
  adm[r] = 0;
  m3[3 * r] = m3[3 * r + 1] = m3[3 * r + 2] = 0;
  if (t < 0) return;
  const pyg_peer& p = peers[owner_of(rep_off, world, t)];
  const int64_t n = *p.recv_count;
  const int32_t g = static_cast<int32_t>(req_base + r);
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (p.recv_gidx[mid] < g) lo = mid + 1;
    else hi = mid;
  }
  if (lo >= n || p.recv_gidx[lo] != g) return;
  adm[r] = p.admitted[lo];
  m3[3 * r] = p.match3[3 * lo];
  m3[3 * r + 1] = p.match3[3 * lo + 1];
  m3[3 * r + 2] = p.match3[3 * lo + 2];
}

using GetAddrRange = int (*)(uint64_t*, size_t*, uint64_t);  // cuMemGetAddressRange_v2

GetAddrRange get_addr_range() {
  static GetAddrRange fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<GetAddrRange>(p);
  }
  return fn;
}

std::map<std::string, void*>& ipc_cache() {
  static std::map<std::string, void*> m;
  return m;
}

}  // namespace

extern "C" {

int pyg_ipc_export(const void* d_ptr, void* handle_out, int64_t* offset_out) {
  if (!d_ptr || !handle_out || !offset_out) return PYG_EINVAL;
  GetAddrRange fn = get_addr_range();
  if (!fn) {
    set_error("cuMemGetAddressRange unavailable");
    return PYG_ECUDA;
  }
  uint64_t base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<uint64_t>(d_ptr)) != 0) {
    set_error("cuMemGetAddressRange failed (not a device allocation?)");
    return PYG_ECUDA;
  }
  cudaIpcMemHandle_t h;
  PYG_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = static_cast<int64_t>(reinterpret_cast<uint64_t>(d_ptr) - base);
  return PYG_OK;
}

int pyg_ipc_import(pyg_ctx* c, const void* handle, int64_t offset, void** d_ptr_out) {
  PYG_ON_DEVICE(c);
  if (!c || !handle || !d_ptr_out) return PYG_EINVAL;
  const std::string key(static_cast<const char*>(handle), sizeof(cudaIpcMemHandle_t));
  auto& m = ipc_cache();
  auto it = m.find(key);
  void* base = nullptr;
  if (it != m.end()) {
    base = it->second;
  } else {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    PYG_CUDA(cudaSetDevice(c->device));
    PYG_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    m[key] = base;
  }
  *d_ptr_out = static_cast<char*>(base) + offset;
  return PYG_OK;
}

int pyg_shard_recv_plan_dev(pyg_ctx* c, int32_t R_total, const pyg_decision* d_dec,
                            const pyg_peer* d_peers, int32_t world, const int64_t* d_req_off,
                            int64_t cap, int32_t* d_recv_gidx, int64_t* d_recv_count,
                            int64_t* d_recv_toff, int64_t* d_recv_hoff, int32_t* d_recv_wf,
                            int32_t* d_recv_role) {
  PYG_ON_DEVICE(c);
  if (!c || R_total < 0 || cap < 0 || !c->sharded) return PYG_EINVAL;
  const int32_t lo = c->rep_base, hi = c->rep_base + c->n_rep;
  size_t t1 = 0, t2 = 0;
  IsMine pred{d_dec, lo, hi};
  PYG_CUDA(cub::DeviceSelect::If(nullptr, t1, static_cast<int32_t*>(nullptr),
                                 static_cast<int32_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                 R_total, pred, c->stream));
  PYG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, static_cast<int64_t*>(nullptr),
                                         static_cast<int64_t*>(nullptr), cap + 1, c->stream));
  auto al = [](size_t x) { return (x + 255) & ~size_t{255}; };
  const size_t bytes = al(static_cast<size_t>(R_total) * 4 + 4) + al(t1) + al(t2) +
                       2 * al(static_cast<size_t>(cap + 1) * 8) + al(static_cast<size_t>(R_total) * 4 + 4);
  void* sp;
  int rc = scratch(c, bytes, &sp);
  if (rc) return rc;
  char* p = static_cast<char*>(sp);
  auto take = [&](size_t b) {
    char* q = p;
    p += al(b);
    return q;
  };
  auto* iota = reinterpret_cast<int32_t*>(take(static_cast<size_t>(R_total) * 4 + 4));
  void* tmp1 = take(t1);
  void* tmp2 = take(t2);
  auto* tl = reinterpret_cast<int64_t*>(take(static_cast<size_t>(cap + 1) * 8));
  auto* hl = reinterpret_cast<int64_t*>(take(static_cast<size_t>(cap + 1) * 8));
  auto* sel = reinterpret_cast<int32_t*>(take(static_cast<size_t>(R_total) * 4 + 4));
  if (R_total) {
    k_iota<<<(R_total + 255) / 256, 256, 0, c->stream>>>(iota, R_total);
    PYG_LAUNCHED(c);
  }
  PYG_CUDA(cub::DeviceSelect::If(tmp1, t1, iota, sel, d_recv_count, R_total, pred, c->stream));
  PYG_LAUNCHED(c);
  // more placed requests than the capacity bound would be a broken invariant: clamp + flag
  k_clamp<<<1, 1, 0, c->stream>>>(d_recv_count, cap, c->hd.error);
  PYG_LAUNCHED(c);
  k_recv_lens<<<static_cast<unsigned>((cap + 1 + 255) / 256), 256, 0, c->stream>>>(
      sel, d_recv_count, d_peers, world, d_req_off, cap, c->B, d_recv_gidx, d_recv_wf,
      d_recv_role, tl, hl);
  PYG_LAUNCHED(c);
  PYG_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, t2, tl, d_recv_toff, cap + 1, c->stream));
  PYG_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, t2, hl, d_recv_hoff, cap + 1, c->stream));
  count_launch(c, 3);
  return PYG_OK;
}

int pyg_shard_pack_dev(pyg_ctx* c, const pyg_reservation* d_req, const int32_t* d_group,
                       const int32_t* d_staged, int32_t R, int32_t mc, int32_t s16,
                       int32_t* d_rows) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0 || mc < 0) return PYG_EINVAL;
  if (!R) return PYG_OK;
  k_pack<<<(R + 255) / 256, 256, 0, c->stream>>>(d_req, d_group, d_staged, R, mc, s16, d_rows,
                                                 c->hd.error);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_unpack_dev(pyg_ctx* c, const int32_t* d_rows, int32_t R, int32_t mc, int32_t s16,
                         pyg_reservation* d_req, int32_t* d_group, int32_t* d_staged) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0 || mc < 0) return PYG_EINVAL;
  if (!R) return PYG_OK;
  k_unpack<<<(R + 255) / 256, 256, 0, c->stream>>>(d_rows, R, mc, s16, d_req, d_group, d_staged);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_unpack_peer_dev(pyg_ctx* c, const int64_t* d_rows_of, int32_t world,
                              const int64_t* d_req_off, int32_t R, int32_t mc, int32_t s16,
                              pyg_reservation* d_req, int32_t* d_group, int32_t* d_staged) {
  return pyg_shard_unpack_peer_own_dev(c, d_rows_of, world, d_req_off, R, mc, s16, 0, d_req,
                                       d_group, d_staged);
}

int pyg_shard_unpack_peer_own_dev(pyg_ctx* c, const int64_t* d_rows_of, int32_t world,
                                  const int64_t* d_req_off, int32_t R, int32_t mc, int32_t s16,
                                  uint64_t own_mask, pyg_reservation* d_req, int32_t* d_group,
                                  int32_t* d_staged) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0 || mc < 0 || world < 1) return PYG_EINVAL;
  if (!R) return PYG_OK;
  const int warps = (R + 31) / 32;
  k_unpack_peer<<<(warps + 7) / 8, 256, 0, c->stream>>>(d_rows_of, world, d_req_off, R, mc, s16,
                                                        own_mask, d_req, d_group, d_staged);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_signal_dev(pyg_ctx* c, const int64_t* d_flag_of, int32_t world, int32_t me,
                         int64_t seq) {
  PYG_ON_DEVICE(c);
  if (!c || world < 1 || world > 1024 || me < 0 || me >= world) return PYG_EINVAL;
  k_signal<<<1, 32 * ((world + 31) / 32), 0, c->stream>>>(d_flag_of, world, me, seq);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_wait_dev(pyg_ctx* c, const int64_t* d_flags, int32_t world, int64_t seq) {
  PYG_ON_DEVICE(c);
  if (!c || world < 1 || world > 1024) return PYG_EINVAL;
  k_wait<<<1, 32 * ((world + 31) / 32), 0, c->stream>>>(d_flags, world, seq, c->hd.error,
                                                         nullptr);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_pull_dev(pyg_ctx* c, const pyg_peer* d_peers, int32_t world,
                       const int64_t* d_req_off, const int32_t* d_recv_gidx,
                       const int64_t* d_recv_count, const int64_t* d_recv_toff,
                       const int64_t* d_recv_hoff, uint64_t* d_tok_out, int64_t tok_cap,
                       uint64_t* d_hash_out, int64_t hash_cap) {
  PYG_ON_DEVICE(c);
  if (!c || world < 1) return PYG_EINVAL;
  k_pull<<<592, 256, 0, c->stream>>>(d_peers, world, d_req_off, d_recv_gidx, d_recv_count,
                                     d_recv_toff, d_recv_hoff, d_tok_out, d_hash_out, tok_cap,
                                     hash_cap, c->hd.error);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_local_placed_dev(pyg_ctx* c, const int32_t* d_placed_off, const int32_t* d_placed,
                               const int32_t* d_recv_gidx, const int64_t* d_recv_count,
                               int32_t* d_p_off, int32_t* d_p_loc) {
  PYG_ON_DEVICE(c);
  if (!c || !c->sharded) return PYG_EINVAL;
  k_local_placed<<<148, 256, 0, c->stream>>>(d_placed_off, d_placed, c->rep_base, c->n_rep,
                                             d_recv_gidx, d_recv_count, d_p_off, d_p_loc);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_apply_lists_dev(pyg_ctx* c, const pyg_peer* d_peers, int32_t world, int32_t me) {
  PYG_ON_DEVICE(c);
  if (!c || world < 1) return PYG_EINVAL;
  k_apply_lists<<<148, 256, 0, c->stream>>>(c->hd, d_peers, world, me, 0, world, 1, nullptr);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_apply_lists_range_dev(pyg_ctx* c, const pyg_peer* d_peers, int32_t world,
                                    int32_t me, int32_t l3_lo, int32_t l3_hi, int32_t with_l2) {
  PYG_ON_DEVICE(c);
  if (!c || world < 1 || l3_lo < 0 || l3_hi > world) return PYG_EINVAL;
  if (l3_lo >= l3_hi && !with_l2) return PYG_OK;
  k_apply_lists<<<148, 256, 0, c->stream>>>(c->hd, d_peers, world, me, l3_lo, l3_hi, with_l2,
                                            nullptr);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_l3_prepare_dev(pyg_ctx* c, const pyg_peer* d_peers, const int64_t* d_flags,
                             int32_t world, int32_t me, int64_t seq) {
  PYG_ON_DEVICE(c);
  if (!c || world < 1 || me < 0 || me >= world) return PYG_EINVAL;
  if (me == 0) return PYG_OK;
  const unsigned long long* cond = c->hd.stats + 7;  // k_admit: an admission matched in L3
  k_wait<<<1, 32 * ((me + 31) / 32), 0, c->stream>>>(d_flags, me, seq, c->hd.error, cond);
  PYG_LAUNCHED(c);
  k_apply_lists<<<148, 256, 0, c->stream>>>(c->hd, d_peers, world, me, 0, me, 0, cond);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_shard_results_dev(pyg_ctx* c, const pyg_peer* d_peers, int32_t world,
                          const int64_t* d_rep_off, const pyg_decision* d_dec, int64_t req_base,
                          int32_t R_local, int32_t* d_admitted, int64_t* d_match3) {
  PYG_ON_DEVICE(c);
  if (!c || world < 1 || R_local < 0) return PYG_EINVAL;
  if (!R_local) return PYG_OK;
  k_results<<<(R_local + 255) / 256, 256, 0, c->stream>>>(d_peers, world, d_rep_off, d_dec,
                                                          req_base, R_local, d_admitted, d_match3);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

}  // extern "C"
