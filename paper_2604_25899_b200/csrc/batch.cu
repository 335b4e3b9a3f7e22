// batch.cu -- batched (device-resident) hot path: K1 hashing, K2 staged
// matrix / lookups, K3 routing, K4/K5 admission and release.
#include <cuda_runtime.h>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

extern "C" {

int pyg_check_device_error(pyg_ctx* c) {
  int32_t e = 0;
  PYG_CUDA(cudaMemcpyAsync(&e, c->hd.error, 4, cudaMemcpyDeviceToHost, c->stream));
  PYG_CUDA(cudaMemsetAsync(c->hd.error, 0, 4, c->stream));
  PYG_CUDA(cudaStreamSynchronize(c->stream));
  if (e) {
    set_error("device-side capacity overflow in a batched kernel");
    return PYG_ECAPACITY;
  }
  return PYG_OK;
}

int pyg_hash_offsets_dev(pyg_ctx*, const int64_t*, int32_t, int64_t*, int64_t*) { return PYG_ENOTSUP; }
int pyg_hash_batch_dev(pyg_ctx*, const uint64_t*, const int64_t*, int32_t, const int64_t*, uint64_t*) { return PYG_ENOTSUP; }
int pyg_staged_matrix_dev(pyg_ctx*, const uint64_t*, const int64_t*, const int64_t*, const uint64_t*, int32_t, const int32_t*, const int32_t*, const int32_t*, int32_t, int32_t*) { return PYG_ENOTSUP; }
int pyg_lookup_batch_dev(pyg_ctx*, const uint64_t*, const int64_t*, const int64_t*, const uint64_t*, int32_t, const int32_t*, int32_t, int64_t*) { return PYG_ENOTSUP; }
int pyg_route_batch_dev(pyg_ctx*, int32_t, const pyg_nodes_dev*, const pyg_reservation*, int32_t, const int32_t*, int32_t, const int32_t*, const int32_t*, int32_t, const int32_t*, double, pyg_decision*, int32_t*, int32_t*) { return PYG_ENOTSUP; }
int pyg_admit_batch_dev(pyg_ctx*, const uint64_t*, const int64_t*, const int64_t*, const uint64_t*, const int32_t*, const int32_t*, int32_t, const int32_t*, const int32_t*, double, int32_t, int32_t*, int64_t*) { return PYG_ENOTSUP; }
int pyg_release_batch_dev(pyg_ctx*, const int64_t*, const int64_t*, const uint64_t*, int32_t, const int32_t*, const int32_t*, const int32_t*) { return PYG_ENOTSUP; }

}  // extern "C"
