// capi.cu -- C-ABI: context lifecycle, tier management and the single-call
// drop-in API (one call == one reference call).  Every call launches CUDA
// kernels on the ctx stream; there is no host-side fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;

namespace {
thread_local std::string g_err;
}

namespace pyg_host {

void set_error(const std::string& msg) { g_err = msg; }

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PYG_OK;
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? PYG_ENOMEM : PYG_ECUDA;
}

int tier_index(pyg_ctx* c, int32_t replica, int32_t tier, bool hierarchy_level, int* out) {
  if (tier < 0 || tier > 2) {
    g_err = "tier must be 0 (L1), 1 (L2) or 2 (L3)";
    return PYG_EINVAL;
  }
  if (tier == 2 && !hierarchy_level) {
    *out = 2 * c->n_rep;
    return PYG_OK;
  }
  if (replica < 0 || replica >= c->n_rep) {
    g_err = "replica out of range";
    return PYG_EINVAL;
  }
  // CacheHierarchy::tier(t): every non-L1 tier is l2_ (hierarchy.cpp:106-107)
  *out = 2 * replica + (tier == 0 ? 0 : 1);
  return PYG_OK;
}

int read_tier(pyg_ctx* c, int ti, TierDev* out) {
  PYG_CUDA(cudaMemcpyAsync(out, c->d_tiers + ti, sizeof(TierDev), cudaMemcpyDeviceToHost,
                           c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int scratch(pyg_ctx* c, size_t bytes, void** out) {
  if (bytes > c->d_scratch_size) {
    if (c->d_scratch) {
      PYG_CUDA(cudaStreamSynchronize(c->stream));
      PYG_CUDA(cudaFree(c->d_scratch));
      c->d_scratch = nullptr;
    }
    size_t sz = std::max<size_t>(bytes, 1 << 20);
    PYG_CUDA(cudaMalloc(&c->d_scratch, sz));
    c->d_scratch_size = sz;
  }
  *out = c->d_scratch;
  return PYG_OK;
}

int aux(pyg_ctx* c, size_t bytes, void** out) {
  if (bytes > c->d_aux_size) {
    if (c->d_aux) {
      PYG_CUDA(cudaStreamSynchronize(c->stream));
      PYG_CUDA(cudaFree(c->d_aux));
      c->d_aux = nullptr;
    }
    size_t sz = std::max<size_t>(bytes + bytes / 8, 1 << 20);
    PYG_CUDA(cudaMalloc(&c->d_aux, sz));
    c->d_aux_size = sz;
  }
  *out = c->d_aux;
  return PYG_OK;
}

}  // namespace pyg_host

using namespace pyg_host;

// ------------------------------------------------------------------ kernels
namespace {

__global__ void k_compact(CtxDev c, int ti) {
  __shared__ int64_t sm[64];
  block_compact(c, c.tiers + ti, sm);
}

static size_t tier_bytes(int64_t log_cap) {
  // log 64 B + idx 2x16 B + ridx 2x16 B + scratch 3x8 B per block
  return static_cast<size_t>(log_cap) * (64 + 32 + 32 + 24);
}

static int alloc_tier(pyg_ctx* c, int ti, int64_t log_cap, int64_t capacity, int32_t counter,
                      int32_t replica) {
  TierHost& th = c->tiers[ti];
  void* mem = nullptr;
  PYG_CUDA(cudaMalloc(&mem, tier_bytes(log_cap)));
  PYG_CUDA(cudaMemsetAsync(mem, 0, tier_bytes(log_cap), c->stream));
  char* p = static_cast<char*>(mem);
  TierDev d{};
  d.log = reinterpret_cast<Block*>(p);
  p += log_cap * 64;
  d.idx = reinterpret_cast<Slot*>(p);
  p += log_cap * 32;
  d.ridx = reinterpret_cast<RSlot*>(p);
  p += log_cap * 32;
  d.scratch = reinterpret_cast<uint64_t*>(p);
  d.log_cap = log_cap;
  d.idx_mask = static_cast<uint64_t>(2 * log_cap - 1);
  d.capacity = capacity;
  d.counter = counter;
  d.replica = replica;
  th.d = d;
  th.bound = 0;
  th.mem = mem;
  PYG_CUDA(cudaMemcpyAsync(c->d_tiers + ti, &d, sizeof(TierDev), cudaMemcpyHostToDevice,
                           c->stream));
  return PYG_OK;
}

}  // namespace

namespace pyg_host {

// Guarantees room for k_new appended records in tier ti (compacting or
// growing; both keep id order and rebuild the indexes).
int ensure_capacity(pyg_ctx* c, int ti, int64_t k_new) {
  TierHost& th = c->tiers[ti];
  if (th.bound + k_new <= th.d.log_cap) {
    th.bound += k_new;
    return PYG_OK;
  }
  TierDev cur;
  int rc = read_tier(c, ti, &cur);
  if (rc) return rc;
  if (cur.log_len + k_new <= cur.log_cap) {
    th.bound = cur.log_len + k_new;
    return PYG_OK;
  }
  const int64_t need = cur.n_alive + k_new;
  if (need <= cur.log_cap / 2) {
    k_compact<<<1, 1024, 0, c->stream>>>(c->hd, ti);
    PYG_LAUNCHED(c);
    th.bound = cur.n_alive + k_new;
    return PYG_OK;
  }
  int64_t cap = cur.log_cap;
  while (cap < 2 * need) cap *= 2;
  void* old = th.mem;
  const int64_t old_len = cur.log_len;
  rc = alloc_tier(c, ti, cap, cur.capacity, cur.counter, cur.replica);
  if (rc) return rc;
  PYG_CUDA(cudaMemcpyAsync(th.d.log, cur.log, old_len * sizeof(Block), cudaMemcpyDeviceToDevice,
                           c->stream));
  TierDev nd = th.d;
  nd.log_len = old_len;
  nd.n_alive = cur.n_alive;
  nd.occupancy = cur.occupancy;
  nd.idx_used = cur.idx_used;
  nd.n_long_orphans = cur.n_long_orphans;
  PYG_CUDA(cudaMemcpyAsync(c->d_tiers + ti, &nd, sizeof(TierDev), cudaMemcpyHostToDevice,
                           c->stream));
  k_compact<<<1, 1024, 0, c->stream>>>(c->hd, ti);
  PYG_LAUNCHED(c);
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  PYG_CUDA(cudaFree(old));
  th.bound = cur.n_alive + k_new;
  return PYG_OK;
}

}  // namespace pyg_host

// ------------------------------------------------------------------ context
extern "C" {

const char* pyg_last_error(void) { return g_err.c_str(); }

int pyg_create(const pyg_config* cfg, pyg_ctx** out) {
  if (!cfg || !out || cfg->n_replicas < 0 || cfg->block_tokens < 1 || cfg->block_tokens > 64 ||
      (cfg->n_replicas > 0 && (!cfg->l1_capacity || !cfg->l2_capacity))) {
    g_err = "invalid pyg_config (block_tokens must be 1..64)";
    return PYG_EINVAL;
  }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    g_err = "no CUDA device (the B200 path has no CPU fallback)";
    return PYG_ECUDA;
  }
  auto* c = new pyg_ctx();
  c->device = cfg->device;
  c->B = cfg->block_tokens;
  c->n_rep = cfg->n_replicas;
  int rc = cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
  if (rc) {
    delete c;
    return rc;
  }
  rc = cuda_check(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking),
                  "cudaStreamCreate");
  if (rc) {
    delete c;
    return rc;
  }
  c->stream = c->own_stream;
  const int nt = 2 * c->n_rep + 1;
  c->tiers.resize(nt);
  CtxDev& hd = c->hd;
  hd.n_rep = c->n_rep;
  hd.B = c->B;
  auto fail = [&](int code) {
    pyg_destroy(c);
    return code;
  };
  if ((rc = cuda_check(cudaMalloc(&c->d_tiers, nt * sizeof(TierDev)), "cudaMalloc"))) return fail(rc);
  hd.tiers = c->d_tiers;
  if ((rc = cuda_check(cudaMalloc(&hd.counters, (c->n_rep + 1) * sizeof(uint64_t)), "cudaMalloc")))
    return fail(rc);
  if ((rc = cuda_check(cudaMalloc(&hd.decode, std::max(1, c->n_rep) * sizeof(int64_t)), "cudaMalloc")))
    return fail(rc);
  if ((rc = cuda_check(cudaMalloc(&hd.off, std::max(1, c->n_rep) * sizeof(int32_t)), "cudaMalloc")))
    return fail(rc);
  if ((rc = cuda_check(cudaMalloc(&hd.error, sizeof(int32_t)), "cudaMalloc"))) return fail(rc);
  if ((rc = cuda_check(cudaMalloc(&hd.stats, 8 * sizeof(unsigned long long)), "cudaMalloc")))
    return fail(rc);
  hd.reg_cap = 1024;
  if ((rc = cuda_check(cudaMalloc(&hd.reg_present, hd.reg_cap), "cudaMalloc"))) return fail(rc);
  if ((rc = cuda_check(cudaMalloc(&hd.reg_mask, hd.reg_cap * sizeof(uint64_t)), "cudaMalloc")))
    return fail(rc);
  cudaMemsetAsync(hd.decode, 0, std::max(1, c->n_rep) * sizeof(int64_t), c->stream);
  cudaMemsetAsync(hd.off, 0, std::max(1, c->n_rep) * sizeof(int32_t), c->stream);
  cudaMemsetAsync(hd.error, 0, sizeof(int32_t), c->stream);
  cudaMemsetAsync(hd.stats, 0, 8 * sizeof(unsigned long long), c->stream);
  cudaMemsetAsync(hd.reg_present, 0, hd.reg_cap, c->stream);
  cudaMemsetAsync(hd.reg_mask, 0, hd.reg_cap * sizeof(uint64_t), c->stream);
  std::vector<uint64_t> ones(c->n_rep + 1, 1);  // next_id_ = 1 (hierarchy.hpp:82,122)
  if ((rc = cuda_check(cudaMemcpy(hd.counters, ones.data(), ones.size() * 8, cudaMemcpyHostToDevice),
                       "cudaMemcpy")))
    return fail(rc);
  const int64_t minb = std::max<int64_t>(cfg->min_blocks, 256);
  for (int r = 0; r < c->n_rep; ++r) {
    int64_t cap1 = 256, cap2 = 256;
    const int64_t want1 = std::max(minb, 2 * (cfg->l1_capacity[r] / c->B + 1));
    const int64_t want2 = std::max(minb, 2 * (cfg->l2_capacity[r] / c->B + 1));
    while (cap1 < want1 && cap1 < (1LL << 22)) cap1 *= 2;
    while (cap2 < want2 && cap2 < (1LL << 22)) cap2 *= 2;
    if ((rc = alloc_tier(c, 2 * r, cap1, cfg->l1_capacity[r], r, r))) return fail(rc);
    if ((rc = alloc_tier(c, 2 * r + 1, cap2, cfg->l2_capacity[r], r, r))) return fail(rc);
  }
  int64_t cap3 = 256;
  while (cap3 < minb) cap3 *= 2;
  if ((rc = alloc_tier(c, 2 * c->n_rep, cap3, INT64_MAX, c->n_rep, -1))) return fail(rc);
  if ((rc = cuda_check(cudaStreamSynchronize(c->stream), "init"))) return fail(rc);
  *out = c;
  return PYG_OK;
}

void pyg_destroy(pyg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaSetDevice(c->device);
  if (c->own_stream) cudaStreamSynchronize(c->own_stream);
  if (c->stream && c->stream != c->own_stream) cudaStreamSynchronize(c->stream);
  for (auto& t : c->tiers)
    if (t.mem) cudaFree(t.mem);
  cudaFree(c->d_tiers);
  cudaFree(c->hd.counters);
  cudaFree(c->hd.decode);
  cudaFree(c->hd.off);
  cudaFree(c->hd.error);
  cudaFree(c->hd.stats);
  cudaFree(c->hd.reg_present);
  cudaFree(c->hd.reg_mask);
  cudaFree(c->d_scratch);
  cudaFree(c->d_aux);
  cudaFree(c->d_claim);
  cudaFree(c->d_gate);
  cudaFree(c->memo);
  cudaFree(c->d_list);
  cudaFree(c->dir_mem);
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
}

int pyg_set_stream(pyg_ctx* c, void* s) {
  PYG_ON_DEVICE(c);
  if (!c) return PYG_EINVAL;
  c->stream = static_cast<cudaStream_t>(s);  // NULL = the default (legacy) stream
  return PYG_OK;
}

int pyg_synchronize(pyg_ctx* c) {
  PYG_ON_DEVICE(c);
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

int64_t pyg_kernel_launches(pyg_ctx* c) { return c ? c->launches : 0; }

int pyg_set_capacity(pyg_ctx* c, int32_t replica, int64_t l1_capacity, int64_t l2_capacity) {
  PYG_ON_DEVICE(c);
  if (!c || replica < 0 || replica >= c->n_rep || l1_capacity < 0 || l2_capacity < 0)
    return PYG_EINVAL;
  const int64_t caps[2] = {l1_capacity, l2_capacity};
  for (int k = 0; k < 2; ++k) {
    const int ti = 2 * replica + k;
    c->tiers[ti].d.capacity = caps[k];
    PYG_CUDA(cudaMemcpyAsync(&c->d_tiers[ti].capacity, &caps[k], sizeof(int64_t),
                             cudaMemcpyHostToDevice, c->stream));
  }
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  return PYG_OK;
}

}  // extern "C"
