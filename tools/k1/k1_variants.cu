// K1 variant harness (experiments only; the product kernel is csrc/k_hash.cu).
// Builds a ragged batch with config-2-like lengths, runs each variant, checks its
// hashes against V0 and prints device time and GB/s (algorithmic bytes).
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cmath>
#include "../../paper_2604_25899_b200/csrc/common.cuh"
using namespace pyg;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// ---------------- V0: the product kernel (1 chain per lane, 16-token chunks)
namespace v0 {
constexpr int kChunk = 16, kRowBytes = kChunk * 8 + 16, kStageBytes = 32 * kRowBytes;
template <int kWarps, int kMinB, int kStages = 2>
__global__ void __launch_bounds__(kWarps * 32, kMinB)
k(const uint64_t* __restrict__ tokens, const int64_t* __restrict__ tok_off, int R,
  const int32_t* __restrict__ order, const int64_t* __restrict__ hash_off,
  uint64_t* __restrict__ hashes, int B, int* __restrict__ next_task) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbuf = smem + warp * kStages * kStageBytes;
  const int ntasks = (R + 31) / 32;
  for (;;) {
    int task = 0;
    if (lane == 0) task = atomicAdd(next_task, 1);
    task = __shfl_sync(kFull, task, 0);
    if (task >= ntasks) break;
    const int idx = task * 32 + lane;
    const bool valid = idx < R;
    const int r = valid ? order[idx] : 0;
    const int64_t s = valid ? tok_off[r] : 0;
    const int64_t n = valid ? tok_off[r + 1] - s : 0;
    const int nch = static_cast<int>((n + kChunk - 1) / kChunk);
    const int maxch = __reduce_max_sync(kFull, nch);
    if (maxch == 0) continue;
    uint64_t* out = hashes + (valid ? hash_off[r] : 0);
    const int cpb = B / kChunk;
    int cc = cpb;
    const int sub = lane >> 4, q = lane & 15;
    auto issue = [&](int c) {
      unsigned char* st = wbuf + (c % kStages) * kStageBytes;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const int jj = j + sub;
        const int64_t sj = __shfl_sync(kFull, s, jj);
        const int64_t nj = __shfl_sync(kFull, n, jj);
        const int64_t pos = static_cast<int64_t>(c) * kChunk + q;
        if (pos < nj) cp_async8(st + jj * kRowBytes + q * 8, tokens + sj + pos, 8);
      }
      cp_commit();
    };
    uint64_t h = kFnvOffset;
    int64_t kk = 0;
#pragma unroll
    for (int c0 = 0; c0 < kStages - 1; ++c0) {
      if (c0 < maxch) issue(c0); else cp_commit();
    }
    for (int c = 0; c < maxch; ++c) {
      if (c + kStages - 1 < maxch) issue(c + kStages - 1); else cp_commit();
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kStages - 1));
      __syncwarp();
      if (c < nch) {
        const unsigned char* row = wbuf + (c % kStages) * kStageBytes + lane * kRowBytes;
        const int64_t rem = n - static_cast<int64_t>(c) * kChunk;
        if (rem >= kChunk) {
#pragma unroll
          for (int x = 0; x < kChunk / 2; ++x) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(row + 16 * x);
            h = fnv_token(h, v.x);
            h = fnv_token(h, v.y);
          }
          if (--cc == 0 || rem == kChunk) { out[kk++] = h; cc = cpb; }
        } else {
          const int p1 = static_cast<int>(rem);
          for (int p = 0; p < p1; ++p) {
            h = fnv_token(h, *reinterpret_cast<const uint64_t*>(row + 8 * p));
            const int64_t j = static_cast<int64_t>(c) * kChunk + p;
            if ((j + 1) % B == 0 || j + 1 == n) out[kk++] = h;
          }
        }
      }
      __syncwarp();
    }
  }
}
}  // namespace v0

// ---------------- V2: two chains per lane (64 requests per warp task), 8-token chunks
namespace v2 {
constexpr int kChunk = 8, kRowBytes = kChunk * 8 + 16, kStageBytes = 64 * kRowBytes;
template <int kWarps, int kMinB>
__global__ void __launch_bounds__(kWarps * 32, kMinB)
k(const uint64_t* __restrict__ tokens, const int64_t* __restrict__ tok_off, int R,
  const int32_t* __restrict__ order, const int64_t* __restrict__ hash_off,
  uint64_t* __restrict__ hashes, int B, int* __restrict__ next_task) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbuf = smem + warp * 2 * kStageBytes;
  const int ntasks = (R + 63) / 64;
  for (;;) {
    int task = 0;
    if (lane == 0) task = atomicAdd(next_task, 1);
    task = __shfl_sync(kFull, task, 0);
    if (task >= ntasks) break;
    int64_t s[2], n[2];
    uint64_t* out[2];
    int nch[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int idx = task * 64 + u * 32 + lane;
      const bool valid = idx < R;
      const int r = valid ? order[idx] : 0;
      s[u] = valid ? tok_off[r] : 0;
      n[u] = valid ? tok_off[r + 1] - s[u] : 0;
      nch[u] = static_cast<int>((n[u] + kChunk - 1) / kChunk);
      out[u] = hashes + (valid ? hash_off[r] : 0);
    }
    const int maxch = __reduce_max_sync(kFull, max(nch[0], nch[1]));
    if (maxch == 0) continue;
    const int cpb = B / kChunk;
    int cc[2] = {cpb, cpb};
    const int sub = lane >> 3, q = lane & 7;  // 4 requests per instruction, 8 lanes x 8 B
    auto issue = [&](int c) {
      unsigned char* st = wbuf + (c & 1) * kStageBytes;
#pragma unroll
      for (int j = 0; j < 64; j += 4) {
        const int jj = j + sub;              // request slot 0..63
        const int src = jj & 31;
        const int64_t sj = __shfl_sync(kFull, jj < 32 ? s[0] : s[1], src);
        const int64_t nj = __shfl_sync(kFull, jj < 32 ? n[0] : n[1], src);
        const int64_t pos = static_cast<int64_t>(c) * kChunk + q;
        if (pos < nj) cp_async8(st + jj * kRowBytes + q * 8, tokens + sj + pos, 8);
      }
      cp_commit();
    };
    uint64_t h[2] = {kFnvOffset, kFnvOffset};
    int64_t kk[2] = {0, 0};
    issue(0);
    for (int c = 0; c < maxch; ++c) {
      if (c + 1 < maxch) issue(c + 1); else cp_commit();
      cp_wait1();
      __syncwarp();
      const unsigned char* row0 = wbuf + (c & 1) * kStageBytes + lane * kRowBytes;
      const unsigned char* row1 = row0 + 32 * kRowBytes;
      const int64_t rem0 = n[0] - static_cast<int64_t>(c) * kChunk;
      const int64_t rem1 = n[1] - static_cast<int64_t>(c) * kChunk;
      if (rem0 >= kChunk && rem1 >= kChunk) {
#pragma unroll
        for (int x = 0; x < kChunk / 2; ++x) {
          const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(row0 + 16 * x);
          const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(row1 + 16 * x);
          h[0] = fnv_token(h[0], a.x);
          h[1] = fnv_token(h[1], b.x);
          h[0] = fnv_token(h[0], a.y);
          h[1] = fnv_token(h[1], b.y);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t rem = u ? rem1 : rem0;
          if (--cc[u] == 0 || rem == kChunk) { out[u][kk[u]++] = h[u]; cc[u] = cpb; }
        }
      } else {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t rem = u ? rem1 : rem0;
          if (rem <= 0) continue;
          const unsigned char* row = u ? row1 : row0;
          if (rem >= kChunk) {
#pragma unroll
            for (int x = 0; x < kChunk; ++x) h[u] = fnv_token(h[u], *reinterpret_cast<const uint64_t*>(row + 8 * x));
            if (--cc[u] == 0 || rem == kChunk) { out[u][kk[u]++] = h[u]; cc[u] = cpb; }
          } else {
            for (int p = 0; p < rem; ++p) {
              h[u] = fnv_token(h[u], *reinterpret_cast<const uint64_t*>(row + 8 * p));
              const int64_t j = static_cast<int64_t>(c) * kChunk + p;
              if ((j + 1) % B == 0 || j + 1 == n[u]) out[u][kk[u]++] = h[u];
            }
          }
        }
      }
      __syncwarp();
    }
  }
}
}  // namespace v2


// ---------------- V3: v0 + per-lane direct loads (no staging) for tasks longer than kLong tokens
namespace v3 {
using v0::kChunk; using v0::kRowBytes; using v0::kStageBytes;
__device__ __forceinline__ void hash_direct(const uint64_t* __restrict__ p, int64_t n, int B,
                                            uint64_t* __restrict__ out) {
  uint64_t h = kFnvOffset;
  int64_t k = 0;
  int cnt = 0;
  int64_t i = 0;
  if (n > 0 && (reinterpret_cast<uintptr_t>(p) & 8)) {
    h = fnv_token(h, __ldg(p));
    i = 1;
    if (++cnt == B) { out[k++] = h; cnt = 0; }
  }
  const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p + i);
  const int64_t npair = (n - i) / 2;
  constexpr int U = 8;  // pairs per group (16 tokens)
  ulonglong2 cur[U], nxt[U];
#pragma unroll
  for (int u = 0; u < U; ++u) cur[u] = u < npair ? __ldg(q + u) : make_ulonglong2(0, 0);
  for (int64_t g = 0; g < npair; g += U) {
#pragma unroll
    for (int u = 0; u < U; ++u) nxt[u] = g + U + u < npair ? __ldg(q + g + U + u) : make_ulonglong2(0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (g + u < npair) {
        h = fnv_token(h, cur[u].x);
        if (++cnt == B) { out[k++] = h; cnt = 0; }
        h = fnv_token(h, cur[u].y);
        if (++cnt == B) { out[k++] = h; cnt = 0; }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
  }
  for (int64_t j = i + 2 * npair; j < n; ++j) {
    h = fnv_token(h, __ldg(p + j));
    if (++cnt == B) { out[k++] = h; cnt = 0; }
  }
  if (cnt > 0) out[k++] = h;
}

template <int kWarps, int kMinB, int kLong>
__global__ void __launch_bounds__(kWarps * 32, kMinB)
k(const uint64_t* __restrict__ tokens, const int64_t* __restrict__ tok_off, int R,
  const int32_t* __restrict__ order, const int64_t* __restrict__ hash_off,
  uint64_t* __restrict__ hashes, int B, int* __restrict__ next_task) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbuf = smem + warp * 2 * kStageBytes;
  const int ntasks = (R + 31) / 32;
  for (;;) {
    int task = 0;
    if (lane == 0) task = atomicAdd(next_task, 1);
    task = __shfl_sync(kFull, task, 0);
    if (task >= ntasks) break;
    const int idx = task * 32 + lane;
    const bool valid = idx < R;
    const int r = valid ? order[idx] : 0;
    const int64_t s = valid ? tok_off[r] : 0;
    const int64_t n = valid ? tok_off[r + 1] - s : 0;
    const int nch = static_cast<int>((n + kChunk - 1) / kChunk);
    const int maxch = __reduce_max_sync(kFull, nch);
    if (maxch == 0) continue;
    uint64_t* out = hashes + (valid ? hash_off[r] : 0);
    if (maxch * kChunk >= kLong) {
      if (valid) hash_direct(tokens + s, n, B, out);
      __syncwarp();
      continue;
    }
    const int cpb = B / kChunk;
    int cc = cpb;
    const int sub = lane >> 4, q = lane & 15;
    auto issue = [&](int c) {
      unsigned char* st = wbuf + (c & 1) * kStageBytes;
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const int jj = j + sub;
        const int64_t sj = __shfl_sync(kFull, s, jj);
        const int64_t nj = __shfl_sync(kFull, n, jj);
        const int64_t pos = static_cast<int64_t>(c) * kChunk + q;
        if (pos < nj) cp_async8(st + jj * kRowBytes + q * 8, tokens + sj + pos, 8);
      }
      cp_commit();
    };
    uint64_t h = kFnvOffset;
    int64_t kk = 0;
    issue(0);
    for (int c = 0; c < maxch; ++c) {
      if (c + 1 < maxch) issue(c + 1); else cp_commit();
      cp_wait1();
      __syncwarp();
      if (c < nch) {
        const unsigned char* row = wbuf + (c & 1) * kStageBytes + lane * kRowBytes;
        const int64_t rem = n - static_cast<int64_t>(c) * kChunk;
        if (rem >= kChunk) {
#pragma unroll
          for (int x = 0; x < kChunk / 2; ++x) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(row + 16 * x);
            h = fnv_token(h, v.x);
            h = fnv_token(h, v.y);
          }
          if (--cc == 0 || rem == kChunk) { out[kk++] = h; cc = cpb; }
        } else {
          const int p1 = static_cast<int>(rem);
          for (int p = 0; p < p1; ++p) {
            h = fnv_token(h, *reinterpret_cast<const uint64_t*>(row + 8 * p));
            const int64_t j = static_cast<int64_t>(c) * kChunk + p;
            if ((j + 1) % B == 0 || j + 1 == n) out[kk++] = h;
          }
        }
      }
      __syncwarp();
    }
  }
}
}  // namespace v3

__global__ void k_len_keys(const int64_t* tok_off, int R, uint16_t* key, int32_t* val) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int64_t L = (tok_off[r + 1] - tok_off[r] + 3) >> 2;
  key[r] = static_cast<uint16_t>(L > 65535 ? 65535 : L);
  val[r] = r;
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 145000, B = 16;
  const double mean = argc > 2 ? atof(argv[2]) : 1100, cv = argc > 3 ? atof(argv[3]) : 0.6;
  const int64_t lmax = argc > 4 ? atol(argv[4]) : 4096;
  std::mt19937_64 rng(1);
  std::lognormal_distribution<double> ln(std::log(mean) - 0.5 * std::log(1 + cv * cv), std::sqrt(std::log(1 + cv * cv)));
  std::vector<int64_t> off(R + 1, 0), hoff(R + 1, 0);
  for (int r = 0; r < R; ++r) {
    int64_t L = std::max<int64_t>(1, std::min<int64_t>(lmax, (int64_t)ln(rng)));
    off[r + 1] = off[r] + L;
    hoff[r + 1] = hoff[r] + (L + B - 1) / B;
  }
  const int64_t T = off[R], H = hoff[R];
  std::vector<uint64_t> tok(T);
  for (auto& t : tok) t = rng();
  uint64_t *d_tok, *d_h0, *d_h1; int64_t *d_off, *d_hoff; int32_t *d_ord; int* d_ctr;
  CK(cudaMalloc(&d_tok, T * 8)); CK(cudaMalloc(&d_h0, H * 8)); CK(cudaMalloc(&d_h1, H * 8));
  CK(cudaMalloc(&d_off, (R + 1) * 8)); CK(cudaMalloc(&d_hoff, (R + 1) * 8));
  CK(cudaMalloc(&d_ord, R * 4)); CK(cudaMalloc(&d_ctr, 4));
  CK(cudaMemcpy(d_tok, tok.data(), T * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_off, off.data(), (R + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_hoff, hoff.data(), (R + 1) * 8, cudaMemcpyHostToDevice));
  // length-descending order
  uint16_t *k_in, *k_out; int32_t* v_in; void* tmp = nullptr; size_t tb = 0;
  CK(cudaMalloc(&k_in, R * 2)); CK(cudaMalloc(&k_out, R * 2)); CK(cudaMalloc(&v_in, R * 4));
  k_len_keys<<<(R + 255) / 256, 256>>>(d_off, R, k_in, v_in);
  cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, k_in, k_out, v_in, d_ord, R, 0, 16);
  CK(cudaMalloc(&tmp, tb));
  cub::DeviceRadixSort::SortPairsDescending(tmp, tb, k_in, k_out, v_in, d_ord, R, 0, 16);
  CK(cudaDeviceSynchronize());
  const double bytes = 8.0 * T + 8.0 * H + 16.0 * (R + 1);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, auto kern, int warps, int ctas_per_sm, int smem, int per_task, uint64_t* dh) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int tasks = (R + per_task - 1) / per_task;
    const int grid = std::min((tasks + warps - 1) / warps, ctas_per_sm * nsm);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9, sum = 0; int reps = 10;
    for (int i = 0; i < reps + 2; ++i) {
      CK(cudaMemset(d_ctr, 0, 4));
      cudaEventRecord(a);
      kern<<<grid, warps * 32, smem>>>(d_tok, d_off, R, d_ord, d_hoff, dh, B, d_ctr);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (i >= 2) { best = std::min(best, ms); sum += ms; }
    }
    CK(cudaGetLastError());
    printf("%-34s grid %5d  best %.4f ms  avg %.4f ms  %.0f GB/s\n", name, grid, best, sum / reps, bytes / (sum / reps * 1e-3) / 1e9);
  };
  run("v0 8w x2 (product)", v0::k<8, 2>, 8, 2, 8 * 2 * v0::kStageBytes, 32, d_h0);
  std::vector<uint64_t> ref(H), got(H);
  CK(cudaMemcpy(ref.data(), d_h0, H * 8, cudaMemcpyDeviceToHost));
  auto check = [&](const char* name) {
    CK(cudaMemcpy(got.data(), d_h1, H * 8, cudaMemcpyDeviceToHost));
    if (got != ref) printf("  !! %s MISMATCH\n", name);
    CK(cudaMemset(d_h1, 0, H * 8));
  };
  run("v0 8w x1", v0::k<8, 1>, 8, 1, 8 * 2 * v0::kStageBytes, 32, d_h1); check("v0 8x1");
  run("v3 8w x1 long>=4096", v3::k<8, 1, 4096>, 8, 1, 8 * 2 * v0::kStageBytes, 32, d_h1); check("v3 4096");
  run("v3 8w x1 long>=2048", v3::k<8, 1, 2048>, 8, 1, 8 * 2 * v0::kStageBytes, 32, d_h1); check("v3 2048");
  run("v3 8w x1 long>=512", v3::k<8, 1, 512>, 8, 1, 8 * 2 * v0::kStageBytes, 32, d_h1); check("v3 512");
  run("v3 8w x1 all direct", v3::k<8, 1, 16>, 8, 1, 8 * 2 * v0::kStageBytes, 32, d_h1); check("v3 all");
  run("v3 8w x2 all direct", v3::k<8, 2, 16>, 8, 2, 8 * 2 * v0::kStageBytes, 32, d_h1); check("v3 all x2");
  return 0;
}
