// k_worker.cu -- worker batch formation and preemption, one CTA per
// replica queue:
//
//   form_batch (worker.cpp:16-37): order the pool by effective priority
//     base + aging*(now - enqueue) descending, then enqueue time ascending, then
//     request id ascending; admit the longest prefix whose reservations fit
//     capacity - active_reservation.  Keys are sorted in shared memory (bitonic over
//     a 3-word key: order(-eff), order(enqueue), id rank); the prefix is one scan.
//   select_preemption_victim (worker.cpp:39-58): the item with the LOWEST effective
//     priority, latest enqueue time, largest id -- a CTA argmin.
//
// The effective priority is computed with explicitly rounded FP64 (__dsub_rn,
// __dmul_rn, __dadd_rn) so every comparison sees the reference's bits.
#include <cuda_runtime.h>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

namespace {

constexpr int kMaxQueue = 4096;

__device__ __forceinline__ double eff_prio(const pyg_queue_item& q, double now, double aging) {
  return __dadd_rn(q.base_priority, __dmul_rn(aging, __dsub_rn(now, q.enqueue_time)));
}

struct QKey {
  uint64_t a, b;  // order(-eff), order(enqueue)
  int64_t c;      // id rank
  int32_t i;      // item index
};

__device__ __forceinline__ bool qless(const QKey& x, const QKey& y) {
  if (x.a != y.a) return x.a < y.a;
  if (x.b != y.b) return x.b < y.b;
  if (x.c != y.c) return x.c < y.c;
  return x.i < y.i;
}

__global__ void __launch_bounds__(512) k_form_batch(const int64_t* off, const pyg_queue_item* items,
                                                   const int64_t* active_res, const int64_t* cap,
                                                   double now, double aging, int32_t* order,
                                                   int32_t* n_admitted, int32_t* err) {
  extern __shared__ __align__(16) unsigned char qsmem[];
  QKey* key = reinterpret_cast<QKey*>(qsmem);
  __shared__ int64_t sm[64];
  const int s = blockIdx.x;
  const int64_t a = off[s], n = off[s + 1] - a;
  if (n > kMaxQueue) {
    if (threadIdx.x == 0) {
      atomicExch(err, 7);
      n_admitted[s] = 0;
    }
    return;
  }
  int64_t np2 = 1;
  while (np2 < n) np2 <<= 1;
  for (int64_t i = threadIdx.x; i < np2; i += blockDim.x) {
    if (i < n) {
      const pyg_queue_item q = items[a + i];
      key[i] = QKey{order_double(-eff_prio(q, now, aging)), order_double(q.enqueue_time), q.id_rank,
                    static_cast<int32_t>(i)};
    } else {
      key[i] = QKey{~0ULL, ~0ULL, INT64_MAX, INT32_MAX};
    }
  }
  __syncthreads();
  for (int64_t k = 2; k <= np2; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < np2; i += blockDim.x) {
        const int64_t ixj = i ^ j;
        if (ixj > i) {
          const bool asc = (i & k) == 0;
          const QKey x = key[i], y = key[ixj];
          if (qless(y, x) == asc) {
            key[i] = y;
            key[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  // strict priority prefix: admitted while active + sum(reservations) <= capacity
  const int64_t budget = cap[s] - active_res[s];
  int64_t base = 0;
  int64_t cut = n;
  for (int64_t i0 = 0; i0 < n; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const int64_t r = i < n ? items[a + key[i].i].reservation : 0;
    int64_t tot;
    const int64_t incl = base + block_exscan(r, sm, &tot) + r;
    const bool over = i < n && incl > budget;
    // first index whose inclusive prefix exceeds the budget (reservations are >= 0)
    const unsigned m = __ballot_sync(kFull, over);
    if ((threadIdx.x & 31) == 0) sm[40 + (threadIdx.x >> 5)] = m ? i0 + (threadIdx.x & ~31) + __ffs(m) - 1 : INT64_MAX;
    __syncthreads();
    int64_t first = INT64_MAX;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) first = min(first, sm[40 + w]);
    __syncthreads();
    if (first != INT64_MAX) {
      cut = first;
      break;
    }
    base += tot;
  }
  for (int64_t i = threadIdx.x; i < cut; i += blockDim.x) order[a + i] = key[i].i;
  if (threadIdx.x == 0) n_admitted[s] = static_cast<int32_t>(cut);
}

// victim = argmin over (eff asc, enqueue desc, id desc, index asc)
__global__ void k_victim(const int64_t* off, const pyg_queue_item* items, double now, double aging,
                         int32_t* victim) {
  const int s = blockIdx.x;
  const int64_t a = off[s], n = off[s + 1] - a;
  __shared__ QKey best[32];
  QKey mine{~0ULL, ~0ULL, INT64_MAX, INT32_MAX};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const pyg_queue_item q = items[a + i];
    const QKey k{order_double(eff_prio(q, now, aging)), ~order_double(q.enqueue_time), ~q.id_rank,
                 static_cast<int32_t>(i)};
    if (qless(k, mine)) mine = k;
  }
  for (int o = 16; o > 0; o >>= 1) {
    QKey y;
    y.a = __shfl_xor_sync(kFull, mine.a, o);
    y.b = __shfl_xor_sync(kFull, mine.b, o);
    y.c = __shfl_xor_sync(kFull, mine.c, o);
    y.i = __shfl_xor_sync(kFull, mine.i, o);
    if (qless(y, mine)) mine = y;
  }
  if ((threadIdx.x & 31) == 0) best[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    QKey b = best[0];
    for (int w = 1; w < static_cast<int>((blockDim.x + 31) / 32); ++w)
      if (qless(best[w], b)) b = best[w];
    victim[s] = n > 0 ? b.i : -1;
  }
}

}  // namespace

extern "C" {

int pyg_form_batch_dev(pyg_ctx* c, int32_t n_sets, const int64_t* d_off,
                       const pyg_queue_item* d_items, const int64_t* d_active_reservation,
                       const int64_t* d_capacity, double now, double aging_rate, int32_t* d_order,
                       int32_t* d_n_admitted) {
  PYG_ON_DEVICE(c);
  if (!c || n_sets < 0) return PYG_EINVAL;
  if (!n_sets) return PYG_OK;
  const int smem = kMaxQueue * static_cast<int>(sizeof(QKey));
  // the attribute is per device: set on every call (cheap) rather than cached per process
  PYG_CUDA(cudaFuncSetAttribute(k_form_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_form_batch<<<n_sets, 512, smem, c->stream>>>(d_off, d_items, d_active_reservation, d_capacity, now,
                                              aging_rate, d_order, d_n_admitted, c->hd.error);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

int pyg_preemption_victim_dev(pyg_ctx* c, int32_t n_sets, const int64_t* d_off,
                              const pyg_queue_item* d_items, double now, double aging_rate,
                              int32_t* d_victim) {
  PYG_ON_DEVICE(c);
  if (!c || n_sets < 0) return PYG_EINVAL;
  if (!n_sets) return PYG_OK;
  k_victim<<<n_sets, 256, 0, c->stream>>>(d_off, d_items, now, aging_rate, d_victim);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

}  // extern "C"
