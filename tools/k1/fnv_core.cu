// FNV-1a core throughput microbenchmark (experiments only): tokens/clk/SM of several
// formulations of fnv1a(uint64 v, h) (tokens.hpp:30-36) with register-resident inputs.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2604_25899_b200/csrc/common.cuh"
using namespace pyg;

__device__ __forceinline__ uint64_t f_plain(uint64_t h, uint64_t v) {
#pragma unroll
  for (int i = 0; i < 8; ++i) { h ^= (v >> (8 * i)) & 0xff; h *= 1099511628211ULL; }
  return h;
}
// lo chain IMAD (lo only), carry IMAD.HI, hi' = hi*435 + carry + (x << 8) with PRMT+IADD3
__device__ __forceinline__ uint64_t f_split(uint64_t h, uint64_t v) {
  uint32_t lo = (uint32_t)h, hi = (uint32_t)(h >> 32);
  const uint32_t vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w = i < 4 ? vl : vh;
    const uint32_t x = lo ^ ((w >> (8 * (i & 3))) & 0xffu);
    uint32_t c, sh, u;
    asm("mul.hi.u32 %0, %1, 435;" : "=r"(c) : "r"(x));
    asm("prmt.b32 %0, %1, 0, 0x2104;" : "=r"(sh) : "r"(x));  // x << 8
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(u) : "r"(hi), "r"(c));
    asm("add.u32 %0, %1, %2;" : "=r"(hi) : "r"(u), "r"(sh));
    asm("mul.lo.u32 %0, %1, 435;" : "=r"(lo) : "r"(x));
  }
  return ((uint64_t)hi << 32) | lo;
}
// byte extract via PRMT
__device__ __forceinline__ uint64_t f_prmt(uint64_t h, uint64_t v) {
  uint32_t lo = (uint32_t)h, hi = (uint32_t)(h >> 32);
  const uint32_t vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w = i < 4 ? vl : vh;
    uint32_t b;
    const uint32_t sel = 0x4440u | (i & 3);
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(b) : "r"(w), "r"(sel));
    const uint32_t x = lo ^ b;
    uint64_t p;
    asm("mul.wide.u32 %0, %1, 435;" : "=l"(p) : "r"(x));
    const uint32_t t = (x << 8) + (uint32_t)(p >> 32);
    hi = hi * 435u + t;
    lo = (uint32_t)p;
  }
  return ((uint64_t)hi << 32) | lo;
}

// u = hi*435 + carry (fma), hi' = u + (x << 8) (ALU LEA wanted)
__device__ __forceinline__ uint64_t f_lea(uint64_t h, uint64_t v) {
  uint32_t lo = (uint32_t)h, hi = (uint32_t)(h >> 32);
  const uint32_t vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w = i < 4 ? vl : vh;
    const uint32_t x = lo ^ ((w >> (8 * (i & 3))) & 0xffu);
    uint64_t p;
    asm("mul.wide.u32 %0, %1, 435;" : "=l"(p) : "r"(x));
    uint32_t u;
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(u) : "r"(hi), "r"((uint32_t)(p >> 32)));
    hi = u + (x << 8);
    lo = (uint32_t)p;
  }
  return ((uint64_t)hi << 32) | lo;
}
// same with the shift as a funnel shift in inline asm
__device__ __forceinline__ uint64_t f_lea2(uint64_t h, uint64_t v) {
  uint32_t lo = (uint32_t)h, hi = (uint32_t)(h >> 32);
  const uint32_t vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w = i < 4 ? vl : vh;
    const uint32_t x = lo ^ ((w >> (8 * (i & 3))) & 0xffu);
    uint64_t p;
    asm("mul.wide.u32 %0, %1, 435;" : "=l"(p) : "r"(x));
    uint32_t u, sh;
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(u) : "r"(hi), "r"((uint32_t)(p >> 32)));
    asm("shf.l.clamp.b32 %0, 0, %1, 8;" : "=r"(sh) : "r"(x));
    asm("add.u32 %0, %1, %2;" : "=r"(hi) : "r"(u), "r"(sh));
    lo = (uint32_t)p;
  }
  return ((uint64_t)hi << 32) | lo;
}

// h' = x*435 + {hi*435 + (x << 8), 0}: one IMAD.WIDE with the high half as its 64-bit addend
__device__ __forceinline__ uint64_t f_wacc(uint64_t h, uint64_t v) {
  uint32_t lo = (uint32_t)h, hi = (uint32_t)(h >> 32);
  const uint32_t vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w = i < 4 ? vl : vh;
    const uint32_t x = lo ^ ((w >> (8 * (i & 3))) & 0xffu);
    const uint32_t u = hi * 435u + (x << 8);
    uint64_t r;
    asm("mad.wide.u32 %0, %1, 435, %2;" : "=l"(r) : "r"(x), "l"((uint64_t)u << 32));
    lo = (uint32_t)r;
    hi = (uint32_t)(r >> 32);
  }
  return ((uint64_t)hi << 32) | lo;
}
// same, the low half computed separately (short lo chain) and the pair only for hi
__device__ __forceinline__ uint64_t f_wacc2(uint64_t h, uint64_t v) {
  uint32_t lo = (uint32_t)h, hi = (uint32_t)(h >> 32);
  const uint32_t vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t w = i < 4 ? vl : vh;
    const uint32_t x = lo ^ ((w >> (8 * (i & 3))) & 0xffu);
    uint32_t c;
    asm("mul.hi.u32 %0, %1, 435;" : "=r"(c) : "r"(x));
    hi = hi * 435u + (x << 8) + c;
    lo = x * 435u;
  }
  return ((uint64_t)hi << 32) | lo;
}

template <int V>
__global__ void __launch_bounds__(256) bench(uint64_t* out, int ntok, uint64_t seed) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t h = kFnvOffset ^ t;
  uint64_t v = seed * (t + 1);
  for (int i = 0; i < ntok; ++i) {
    v = v * 6364136223846793005ULL + 1442695040888963407ULL;  // 2 IMAD-ish per token (overhead)
    if (V == 0) h = fnv_token(h, v);
    if (V == 1) h = f_plain(h, v);
    if (V == 2) h = f_split(h, v);
    if (V == 3) h = f_prmt(h, v);
    if (V == 4) h = f_lea(h, v);
    if (V == 5) h = f_lea2(h, v);
    if (V == 6) h = f_wacc(h, v);
    if (V == 7) h = f_wacc2(h, v);
  }
  out[t] = h;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint64_t* d; cudaMalloc(&d, 8ull << 22);
  const int ntok = 4096;
  const char* names[] = {"fnv_token (product)", "plain u64 *= P", "split IMAD.HI + PRMT", "PRMT byte extract", "mad hi + LEA", "mad hi + shf + add", "wide with hi addend", "mul.hi + lo split"};
  for (int blocks_per_sm : {0, 2, 8}) {
    const int grid = blocks_per_sm ? nsm * blocks_per_sm : nsm;  // 0: one warp per SM (latency)
    const int threads = blocks_per_sm ? 256 : 32;
    uint64_t ref[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int V = 0; V < 8; ++V) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto launch = [&]() {
        if (V == 0) bench<0><<<grid, threads>>>(d, ntok, 7);
        if (V == 1) bench<1><<<grid, threads>>>(d, ntok, 7);
        if (V == 2) bench<2><<<grid, threads>>>(d, ntok, 7);
        if (V == 3) bench<3><<<grid, threads>>>(d, ntok, 7);
        if (V == 4) bench<4><<<grid, threads>>>(d, ntok, 7);
        if (V == 5) bench<5><<<grid, threads>>>(d, ntok, 7);
        if (V == 6) bench<6><<<grid, threads>>>(d, ntok, 7);
        if (V == 7) bench<7><<<grid, threads>>>(d, ntok, 7);
      };
      launch();
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      uint64_t x; cudaMemcpy(&x, d + 12345, 8, cudaMemcpyDeviceToHost);
      ref[V] = x;
      const double toks = (double)grid * threads * ntok;
      printf("blocks/SM %d  %-24s %.3f ms  %.1f Gtok/s  = %.2f TB/s  %.1f cycles/token/lane  %s\n", blocks_per_sm,
             names[V], ms, toks / ms / 1e6, toks * 8 / ms / 1e9, ms * 1e-3 * 1.965e9 / ntok,
             V && ref[V] != ref[0] ? "MISMATCH" : "");
    }
  }
  return 0;
}
