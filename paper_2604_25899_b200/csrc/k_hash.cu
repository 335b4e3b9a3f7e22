// k_hash.cu -- K1: batched chain_boundary_hashes (hierarchy.cpp:21-30).
//
// FNV-1a is a serial chain per request, so parallelism comes from requests:
// one lane owns one request.  To keep HBM reads coalesced, each warp stages
// its 32 requests' tokens through shared memory in 16-token chunks: every lane
// publishes its request's chunk source (pointer | valid tokens, 8 B) in a smem
// slot, each half-warp reads the 16 slots of its requests with 8 broadcast
// LDS.128 and copies one request's 128-byte chunk per instruction with 8-byte
// cp.async (16 lanes x 8 B, 2 requests per warp instruction), double-buffered;
// each lane then hashes its own row with conflict-free LDS.128 (row stride
// 144 B).  Requests are processed in descending length order (a 16-bit radix
// sort on ceil(len/4)) so lanes of a warp carry equal work and the longest
// chains start first.  The same loader serves prompt assembly fused with K1
// (kGather): chunk sources then come from a precomputed table over the pool.
//
// Occupancy: ONE 8-warp CTA per SM (2 warps per scheduler), registers capped at 128
// (no spills) so that while K1 hashes the NEXT burst on a second stream, the current
// step's admission / routing CTAs can still be resident on the same SMs.  The FNV chain is
// latency-bound per lane (~119 cycles/token measured, tools/k1/fnv_core.cu) and
// the INT pipes cap the SM at ~512 Gtok/s (4.1 TB/s of token bytes); two warps
// per scheduler already saturate issue, and more co-resident warps only slow
// each chain (the long-prompt tail) -- 4 warps/scheduler was 25% slower on the
// config-2 length mix (tools/k1/k1_variants.cu).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "ctx.cuh"
#include "device_ops.cuh"

using namespace pyg;
using namespace pyg_host;

namespace {

constexpr int kChunk = 16;                      // tokens per staged chunk
constexpr int kRowBytes = kChunk * 8 + 16;      // 144: padded row
constexpr int kStageBytes = 32 * kRowBytes;     // one warp, one stage
constexpr int kWarps = 8;                       // warps per CTA
// per warp (fused assembly): 2 staging buffers, the destination base of each of its 32
// requests and 4 rotating slots of their packed chunk sources (8 B each).  Slot entries of
// request l sit at position perm(l) = (l & 1) * 16 + (l >> 1), so the 16 requests a
// half-warp loads (l = 2t + sub) are 128 contiguous bytes: 8 broadcast LDS.128.
constexpr int kMetaBytes = 5 * 32 * 8;
constexpr int smem_bytes(int w) { return w * (2 * kStageBytes + kMetaBytes); }
// more than half of the SM's 228 KB: one K1 CTA per SM (grid mode 2)
constexpr int kSmemOneCta = 116 * 1024;
// packed chunk source: pointer | (valid tokens in the chunk, 0..16) << 59
constexpr int kVShift = 59;
constexpr unsigned long long kPtrMask = (1ull << kVShift) - 1;
__device__ __forceinline__ int perm_slot(int l) { return (l & 1) * 16 + (l >> 1); }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
// admission gate (pyg_set_hash_gate): K1 warps read it once per chunk and, when it is set,
// sleep until the step's admission has finished (the latency-bound admission then runs
// without K1 warps competing for its SMs' issue slots)
__device__ __forceinline__ int gate_load(const int32_t* g) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(g));
  return v;
}
__device__ __forceinline__ void gate_wait(const int32_t* g) {
  while (gate_load(g)) __nanosleep(1000);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// Prompt source of K1.  kGather = false: the token CSR (tokens + tok_off).  kGather =
// true: K1 fused with prompt assembly (pyg_assemble_hash_dev) -- request r's tokens are
// the concatenation of its segments of a device token pool.  k_chunk_src first resolves
// every 16-token chunk of every request to ONE source pointer: the pool position of the
// chunk's first token when the chunk lies inside one segment (the common case), else a
// private 16-token copy in a side buffer (chunks that straddle segment boundaries; at most
// one per segment).  The K1 loader then reads chunk c of request r at src[c] + q exactly
// like the CSR path, with the pointers prefetched two chunks ahead by the request's own
// lane, and the warp writes each staged chunk back to the token CSR (coalesced) while it
// hashes.  Chunk table index of (r, c) = tok_off[r] / 16 + r + c (no scan needed: request
// r owns ceil(len/16) <= tok_off[r+1]/16 - tok_off[r]/16 + 1 slots).
struct GatherSrc {
  const unsigned long long* chunk_src;  // packed (pointer | valid << 59)
  uint64_t* tokens_out;
};

__global__ void k_chunk_src(int R, const int64_t* __restrict__ seg_off,
                            const pyg_segment* __restrict__ segs, const uint64_t* __restrict__ pool,
                            const int64_t* __restrict__ tok_off, unsigned long long* tab,
                            int64_t tab_cap, uint64_t* side, int64_t side_cap,
                            unsigned long long* side_ctr, int32_t* error) {
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += warps) {
    const int64_t s = tok_off[r], n = tok_off[r + 1] - s;
    const int64_t nch = (n + kChunk - 1) / kChunk;
    const int64_t base = s / kChunk + r;
    if (base + nch > tab_cap) {
      if (lane == 0) atomicExch(error, 4);  // caller's n_tokens bound too small
      continue;
    }
    const int64_t k1 = seg_off[r + 1];
    int64_t k = seg_off[r], ps = 0;  // this lane's cursor: segment k covers [ps, ps + len)
    for (int64_t c0 = 0; c0 < nch; c0 += 32) {
      const int64_t c = c0 + lane;
      const bool act = c < nch;
      const int64_t p0 = c * kChunk, p1 = min(p0 + kChunk, n);
      pyg_segment sg{0, 0};
      bool straddle = false;
      if (act) {
        while (k < k1) {
          sg = segs[k];
          if (ps + sg.len > p0) break;
          ps += sg.len;
          ++k;
        }
        straddle = p1 > ps + sg.len;
      }
      const unsigned m = __ballot_sync(kFull, straddle);
      unsigned long long b0 = 0;
      if (m && lane == __ffs(m) - 1) b0 = atomicAdd(side_ctr, static_cast<unsigned long long>(__popc(m)));
      b0 = __shfl_sync(kFull, b0, __ffs(m ? m : 1) - 1);
      if (!act) continue;
      if (!straddle) {
        tab[base + c] = reinterpret_cast<unsigned long long>(pool + sg.src + (p0 - ps)) |
                        (static_cast<unsigned long long>(p1 - p0) << kVShift);
      } else {
        const int64_t idx = static_cast<int64_t>(b0) + __popc(m & ((1u << lane) - 1));
        if (idx >= side_cap) {
          atomicExch(error, 4);
          continue;
        }
        uint64_t* dst = side + idx * kChunk;
        int64_t kk = k, pp = ps;
        pyg_segment g = sg;
        for (int64_t p = p0; p < p1; ++p) {
          while (p >= pp + g.len) {
            pp += g.len;
            g = segs[++kk];
          }
          dst[p - p0] = pool[g.src + (p - pp)];
        }
        tab[base + c] = reinterpret_cast<unsigned long long>(dst) |
                        (static_cast<unsigned long long>(p1 - p0) << kVShift);
      }
    }
  }
}

// ------------------------------------------------------------ split tasks
// A long prompt's chain is serial per token, so one lane per request leaves the longest
// prompts of a batch as a tail (~119 cycles/token: 2 ms for 32k tokens).  A SPLIT task
// hashes one long request on a whole warp, 512 tokens (a "super-chunk") at a time, lane l
// owning the 16-token segment [16 l, 16 l + 16).  FNV-1a's xor touches only the low byte,
// so with l = h mod 256 and h = l + 256 u:
//   chain_m(h) = chain_m(l) + 256 u * P^m  (mod 2^64)            (P = FNV prime, m bytes)
// and the low byte evolves on its own, l' = ((l ^ b) * 0xB3) mod 256, a triangular map:
// bit j of l' is bit j of (l ^ b) xor a function of the lower bits.  Pass A finds every
// segment's start low byte 2 bits at a time: a lane runs its segment for both values of
// bit j (packed in the two 16-bit halves of one register; bit j+1 starts at 0), which
// gives the segment's map on (bit j, bit j+1) -- (a, d) -> (a ^ X, d ^ Y[a]) -- and a
// warp scan of those maps gives every lane its start bits from the super-chunk's.  Pass B
// runs the 64-bit chain of each segment from its start low byte alone, and a warp scan of
// the affine maps D' = D * P^(8 n) + (chain & ~0xff) restores the high part (D = h - l).
// Requests with len >= kSplitMin and B % 16 == 0 become split tasks; they run first.
constexpr int kSplitTok = 16;                 // tokens per lane segment
constexpr int kSuper = 32 * kSplitTok;        // tokens per super-chunk
__constant__ uint64_t c_pw8[kSplitTok + 1];   // P^(8 t), t = 0..16

__device__ __forceinline__ uint32_t map2_then(uint32_t f, uint32_t g) {
  // maps on 2 bits as (X | Y0 << 1 | Y1 << 2): (a, d) -> (a ^ X, d ^ Y[a]); f first
  const uint32_t xf = f & 1u;
  const uint32_t gy0 = (g >> 1) & 1u, gy1 = (g >> 2) & 1u;
  const uint32_t y0 = ((f >> 1) & 1u) ^ (xf ? gy1 : gy0);
  const uint32_t y1 = ((f >> 2) & 1u) ^ (xf ? gy0 : gy1);
  return (xf ^ (g & 1u)) | (y0 << 1) | (y1 << 2);
}

// one 8-bit-automaton step on both packed candidates
// (volatile: the byte extraction stays inside its round; hoisted out of the round loop,
// 128 extracted bytes per lane would not fit in registers)
__device__ __forceinline__ uint32_t lo8_step(uint32_t x, uint32_t w, int bi) {
  uint32_t bb;
  asm volatile("prmt.b32 %0, %1, 0, %2;" : "=r"(bb) : "r"(w),
               "r"(0x4040u | static_cast<uint32_t>(bi) | (static_cast<uint32_t>(bi) << 8)));
  return ((x ^ bb) & 0x00FF00FFu) * 0xB3u;
}

// One split task: request of n tokens at src, boundary hashes to out (B % 16 == 0).
// wbuf: this warp's 2 staging buffers (rows of kRowBytes, row l = segment l).
// h0: the chain state before src[0] (the offset basis, or a memo state at a block boundary)
__device__ __noinline__ void split_task(const uint64_t* __restrict__ src, int64_t n, int B,
                           uint64_t* __restrict__ out, unsigned char* wbuf,
                           const int32_t* gate = nullptr, uint64_t h0 = kFnvOffset) {
  const int lane = threadIdx.x & 31;
  const int nsc = static_cast<int>((n + kSuper - 1) / kSuper);
  auto issue = [&](int sc) {
    unsigned char* st = wbuf + (sc & 1) * kStageBytes;
    const int64_t t0 = static_cast<int64_t>(sc) * kSuper;
    const int64_t nv = min(static_cast<int64_t>(kSuper), n - t0);
#pragma unroll
    for (int i = 0; i < kSuper / 32; ++i) {
      const int t = i * 32 + lane;  // token of the super-chunk: row t / 16, column t % 16
      if (t < nv) cp_async8(st + (t >> 4) * kRowBytes + (t & 15) * 8, src + t0 + t, 8);
    }
    cp_commit();
  };
  uint64_t H0 = h0;  // hash at the super-chunk start (warp-uniform)
  issue(0);
  for (int sc = 0; sc < nsc; ++sc) {
    const int gz = gate ? gate_load(gate) : 0;
    if (sc + 1 < nsc)
      issue(sc + 1);
    else
      cp_commit();
    cp_wait1();
    __syncwarp();
    const unsigned char* row = wbuf + (sc & 1) * kStageBytes + lane * kRowBytes;
    const int64_t seg0 = static_cast<int64_t>(sc) * kSuper + lane * kSplitTok;
    const int nt = static_cast<int>(max(int64_t{0}, min(static_cast<int64_t>(kSplitTok), n - seg0)));
    uint32_t w[2 * kSplitTok];
#pragma unroll
    for (int x = 0; x < kSplitTok / 2; ++x) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + 16 * x);
      w[4 * x] = v.x;
      w[4 * x + 1] = v.y;
      w[4 * x + 2] = v.z;
      w[4 * x + 3] = v.w;
    }
    const uint32_t L0 = static_cast<uint32_t>(H0) & 0xffu;
    // pass A: the segment's start low byte, two bits per round
    uint32_t known = 0;
#pragma unroll 1
    for (int j = 0; j < 8; j += 2) {
      uint32_t x = known | ((known | (1u << j)) << 16);
      if (nt == kSplitTok) {
#pragma unroll
        for (int wi = 0; wi < 2 * kSplitTok; ++wi) {
#pragma unroll
          for (int bi = 0; bi < 4; ++bi) x = lo8_step(x, w[wi], bi);
        }
      } else {
        for (int t = 0; t < nt; ++t) {
          const uint2 v = *reinterpret_cast<const uint2*>(row + 8 * t);
#pragma unroll
          for (int bi = 0; bi < 4; ++bi) x = lo8_step(x, v.x, bi);
#pragma unroll
          for (int bi = 0; bi < 4; ++bi) x = lo8_step(x, v.y, bi);
        }
      }
      uint32_t m = 0;  // empty segments are the identity
      if (nt > 0)
        m = ((x >> j) & 1u) | (((x >> (j + 1)) & 1u) << 1) | (((x >> (16 + j + 1)) & 1u) << 2);
      uint32_t inc = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc = map2_then(y, inc);
      }
      uint32_t pre = __shfl_up_sync(kFull, inc, 1);
      if (lane == 0) pre = 0;
      const uint32_t a0 = (L0 >> j) & 1u, d0 = (L0 >> (j + 1)) & 1u;
      const uint32_t a = a0 ^ (pre & 1u);
      const uint32_t d = d0 ^ ((pre >> (1 + a0)) & 1u);
      known |= (a << j) | (d << (j + 1));
    }
    // pass B: the 64-bit chain of the segment from its start low byte
    uint64_t h = known;
    if (nt == kSplitTok) {
#pragma unroll
      for (int t = 0; t < kSplitTok; ++t)
        h = fnv_token(h, static_cast<uint64_t>(w[2 * t]) | (static_cast<uint64_t>(w[2 * t + 1]) << 32));
    } else {
      for (int t = 0; t < nt; ++t) h = fnv_token(h, *reinterpret_cast<const uint64_t*>(row + 8 * t));
    }
    // D_{l+1} = D_l * P^(8 nt_l) + (chain_l & ~0xff), D = hash - low byte at a segment start
    uint64_t A = nt > 0 ? c_pw8[nt] : 1ull, Bq = nt > 0 ? (h & ~0xffull) : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t ya = __shfl_up_sync(kFull, A, o), yb = __shfl_up_sync(kFull, Bq, o);
      if (lane >= o) {
        Bq = yb * A + Bq;
        A = ya * A;
      }
    }
    uint64_t ea = __shfl_up_sync(kFull, A, 1), eb = __shfl_up_sync(kFull, Bq, 1);
    if (lane == 0) {
      ea = 1;
      eb = 0;
    }
    const uint64_t D = (H0 - L0) * ea + eb;
    const uint64_t hend = h + D * (nt > 0 ? c_pw8[nt] : 1ull);
    const int64_t e = seg0 + nt;
    if (nt > 0 && (e % B == 0 || e == n)) out[(e - 1) / B] = hend;  // hierarchy.cpp:26
    const int64_t nv = min(static_cast<int64_t>(kSuper), n - static_cast<int64_t>(sc) * kSuper);
    H0 = __shfl_sync(kFull, hend, static_cast<int>((nv - 1) / kSplitTok));
    __syncwarp();
    if (gz) gate_wait(gate);
  }
}

// ------------------------------------------------------------- prefix memo
// Requests that start with the same tokens share their leading chain hashes (the state at a
// chunk end depends only on the tokens before it).  Per burst, one LEADER per first-16-token
// content -- the longest request sharing it -- is hashed over its first kMemoTok tokens into
// a memo row of chunk-end states (tasks of K1 itself, ahead of every other task).  Before
// K1, k_memo_match compares every request with its leader, a warp per request streaming 128
// tokens per step (coalesced, memory-bound), and records how many leading 16-token chunks
// match in full; K1 starts each request's chain after them, and k_memo_emit (after K1)
// copies their boundary hashes from the memo row.  Exact for any input: a memo state is
// used only when every token up to its chunk end compared equal.  Only first chunks shared
// by >= kMemoMin requests get a row.  The task order and the split threshold use the work
// left past the memoised chunks.
constexpr int kMemoTok = 2048;                  // tokens memoised per leader
constexpr int kMemoChunks = kMemoTok / 16;      // 128 chunk-end states (1 KB) per row
constexpr int kMemoMin = 3;
constexpr int kMemoRows = 4096;

struct MemoTab {
  uint32_t* key;              // [cap] first-chunk digest (0 = empty)
  unsigned long long* lead;   // [cap] (length << 32) | ~r: max = longest, then lowest r
  int32_t* cnt;               // [cap] requests with the digest
  int32_t* row;               // [cap] memo row of the slot or -1
  int32_t* slot_of;           // [R] digest slot of request r or -1
  int32_t* mlen;              // [R] leading chunks equal to the leader's (k_memo_match)
  int32_t* row_lead;          // [kMemoRows] leader request
  int32_t* row_chunks;        // [kMemoRows] memoised chunks
  int32_t* ready;             // [kMemoRows] row written (release / acquire)
  uint64_t* state;            // [kMemoRows][kMemoChunks]
  int32_t* n_rows;
  uint32_t mask;
};

__global__ void k_memo_elect(const uint64_t* __restrict__ tokens,
                             const int64_t* __restrict__ tok_off, int R, MemoTab m) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int64_t s = tok_off[r], n = tok_off[r + 1] - s;
  if (n < 16) {
    m.slot_of[r] = -1;
    return;
  }
  uint64_t d = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) d = (d ^ tokens[s + i]) * 0x9E3779B97F4A7C15ull + i;
  const uint32_t key = (static_cast<uint32_t>(d >> 32) ^ static_cast<uint32_t>(d)) | 1u;
  uint32_t slot = key & m.mask;
  for (;;) {
    const uint32_t k = atomicCAS(m.key + slot, 0u, key);
    if (k == 0u || k == key) break;
    slot = (slot + 1) & m.mask;
  }
  m.slot_of[r] = static_cast<int32_t>(slot);
  atomicAdd(m.cnt + slot, 1);
  atomicMax(m.lead + slot, (static_cast<unsigned long long>(n) << 32) |
                               (0xFFFFFFFFu - static_cast<uint32_t>(r)));
}

// a row per slot shared by >= kMemoMin requests (up to kMemoRows)
__global__ void k_memo_rows(MemoTab m) {
  const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot > m.mask) return;
  int row = -1;
  if (m.key[slot] != 0u && m.cnt[slot] >= kMemoMin) {
    row = atomicAdd(m.n_rows, 1);
    if (row < kMemoRows) {
      const unsigned long long L = m.lead[slot];
      m.row_lead[row] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(L));
      m.row_chunks[row] = static_cast<int32_t>(min(static_cast<int64_t>(L >> 32),
                                                   static_cast<int64_t>(kMemoTok)) / 16);
    } else {
      row = -1;
    }
  }
  m.row[slot] = row;
}
__global__ void k_memo_clamp(int32_t* n_rows) {
  if (*n_rows > kMemoRows) *n_rows = kMemoRows;
}
// matched chunks of every request against its leader: a warp per request, 128 tokens per step
__global__ void k_memo_match(const uint64_t* __restrict__ tokens,
                             const int64_t* __restrict__ tok_off, int R, MemoTab m) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += nw) {
    const int slot = m.slot_of[r];
    const int row = slot >= 0 ? m.row[slot] : -1;
    int mc = 0;
    if (row >= 0) {
      const int64_t s = tok_off[r];
      const int64_t n = tok_off[r + 1] - s;
      const int64_t lim = 16 * min(static_cast<int64_t>(m.row_chunks[row]), n / 16);
      const uint64_t* a = tokens + s;
      const uint64_t* b = tokens + tok_off[m.row_lead[row]];
      int64_t eq = lim;  // tokens equal from the start
      for (int64_t i = 0; i < lim; i += 128) {  // 4 loads per lane in flight
        bool df[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = i + 32 * u + lane;
          df[u] = j < lim && a[j] != b[j];
        }
        unsigned d = 0;
        int u0 = 0;
#pragma unroll
        for (int u = 3; u >= 0; --u) {
          const unsigned du = __ballot_sync(kFull, df[u]);
          if (du) {
            d = du;
            u0 = u;
          }
        }
        if (d) {
          eq = i + 32 * u0 + __ffs(d) - 1;
          break;
        }
      }
      mc = static_cast<int>(eq / 16);
    }
    if (lane == 0) m.mlen[r] = mc;
  }
}

// boundary hashes of the memoised chunks (after K1): a warp per request, coalesced copies
// from the memo row (hierarchy.cpp:26: every B tokens and at the last token)
__global__ void k_memo_emit(const int64_t* __restrict__ tok_off,
                            const int64_t* __restrict__ hash_off, uint64_t* __restrict__ hashes,
                            int R, int B, MemoTab m) {
  const int lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int cpb = B / 16;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += nw) {
    const int m0 = m.mlen[r];
    if (m0 <= 0) continue;
    const int64_t n = tok_off[r + 1] - tok_off[r];
    const uint64_t* ms = m.state + static_cast<int64_t>(m.row[m.slot_of[r]]) * kMemoChunks;
    uint64_t* out = hashes + hash_off[r];
    // block j ends at chunk (j + 1) cpb - 1; the request's last chunk (if memoised) too
    const int nb = m0 / cpb;
    for (int j = lane; j < nb; j += 32) out[j] = ms[(j + 1) * cpb - 1];
    if (lane == 0 && 16 * static_cast<int64_t>(m0) == n && m0 % cpb) out[nb] = ms[m0 - 1];
  }
}
__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Chunks are aligned to each request's own first token, so with B % 16 == 0 a
// block boundary always coincides with the end of a chunk: the emit decision
// is per chunk and warp-uniform (no per-token test).  The last, partial chunk
// and B % 16 != 0 take the generic per-token path.
//
// Long prompts (>= the split threshold) are split tasks (split_task above); the rest run
// one lane per request in 32-request tasks.
template <bool kGather, int W, bool kMemo>
__global__ void __launch_bounds__(W * 32, (W <= 8 ? 2 : 1))
k_hash_staged(const uint64_t* __restrict__ tokens, const int64_t* __restrict__ tok_off,
              int R, const int32_t* __restrict__ order, const int64_t* __restrict__ hash_off,
              uint64_t* __restrict__ hashes, int B, int* __restrict__ next_task, GatherSrc g,
              const int* __restrict__ n_split_p, const int32_t* gate, MemoTab mt, int n_sm) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbuf = smem + warp * 2 * kStageBytes;
  // fused assembly: wbase[32] destination bases, lsl[4][32] packed chunk sources
  unsigned long long* wbase = reinterpret_cast<unsigned long long*>(
      smem + W * 2 * kStageBytes + warp * kMetaBytes);
  unsigned long long* lsl = wbase + 32;
  // tasks: [0, n_memo) memo rows (kMemo), then [.., + n_split) one long request each
  // (split_task, the longest first), then 32-request tasks over the rest of the
  // length-sorted order
  const int n_memo = kMemo ? *mt.n_rows : 0;
  const int n_split = (!kGather && n_split_p) ? *n_split_p : 0;
  const int ntasks = n_memo + n_split + (R - n_split + 31) / 32;
  // persistent: each warp pulls tasks, longest first, until none are left
  // persistent (next_task != null): warps pull tasks from a counter until none are left;
  // otherwise one task per warp (a CTA per 8 tasks, in the longest-first order), so CTAs
  // retire continually and a higher-priority stream's kernels get SMs between them
  // fewer tasks than warps on the SMs (a burst of few, long one-lane chains, config 3):
  // spread them -- at most ceil(tasks / CTAs) warps of each CTA take tasks, so each chain
  // gets an SM scheduler (nearly) to itself instead of sharing one on a few SMs
  const int ctas = next_task ? static_cast<int>(gridDim.x) : min(static_cast<int>(gridDim.x), n_sm);
  const bool sparse = ntasks < ctas * W;
  if (sparse && (warp >= (ntasks + ctas - 1) / ctas || static_cast<int>(blockIdx.x) >= ctas))
    return;
  for (int it = 0;; ++it) {
  int task = 0;
  if (next_task) {
    if (lane == 0) task = atomicAdd(next_task, 1);
    task = __shfl_sync(kFull, task, 0);
  } else if (sparse) {
    task = it == 0 ? warp * ctas + static_cast<int>(blockIdx.x) : ntasks;
  } else {
    task = it == 0 ? static_cast<int>(blockIdx.x) * W + warp : ntasks;
  }
  if (task >= ntasks) break;
  if (kMemo && task < n_memo) {  // memo row `task`: the leader's first chunks on this warp
    split_task(tokens + tok_off[mt.row_lead[task]], 16 * static_cast<int64_t>(mt.row_chunks[task]),
               16, mt.state + static_cast<int64_t>(task) * kMemoChunks, wbuf, gate);
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(mt.ready + task, 1);
    continue;
  }
  task -= n_memo;
  if (task < n_split) {
    const int r = order[task];
    const int64_t s0 = tok_off[r];
    // kMemo: start after the memoised chunks, at a block boundary (k_memo_emit writes the
    // boundary hashes before it)
    int64_t m0 = 0;
    uint64_t h0 = kFnvOffset;
    if (kMemo) {
      const int cpb = B / kChunk;
      m0 = (mt.mlen[r] / cpb) * cpb;
      if (m0 > 0) {
        const int row = mt.row[mt.slot_of[r]];
        while (ld_acquire(mt.ready + row) == 0) __nanosleep(256);
        h0 = mt.state[static_cast<int64_t>(row) * kMemoChunks + m0 - 1];
      }
    }
    split_task(tokens + s0 + kChunk * m0, tok_off[r + 1] - s0 - kChunk * m0, B,
               hashes + hash_off[r] + m0 / (B / kChunk > 0 ? B / kChunk : 1), wbuf, gate, h0);
    continue;
  }
  const int idx = n_split + (task - n_split) * 32 + lane;
  const bool valid = idx < R;
  const int r = valid ? (order ? order[idx] : idx) : 0;
  const int64_t s = valid ? tok_off[r] : 0;
  const int64_t n = valid ? tok_off[r + 1] - s : 0;
  const int nch = static_cast<int>((n + kChunk - 1) / kChunk);
  const int maxch = __reduce_max_sync(kFull, nch);
  if (maxch == 0) continue;
  uint64_t* out = hashes + (valid ? hash_off[r] : 0);
  const bool fast = (B % kChunk) == 0;
  const int cpb = fast ? B / kChunk : 1;  // chunks per block (fast path)
  int cc = cpb;
  uint64_t h = kFnvOffset;
  int64_t k = 0;
  // kMemo: the request's leading chunks equal to its leader's (k_memo_match) come from the
  // memo row (k_memo_emit writes their boundary hashes): the chain starts after them, at
  // chunk m0; the warp's chunk loop starts at its lanes' smallest m0
  int m0 = 0;
  if (kMemo && valid) {
    m0 = mt.mlen[r];
    if (m0 > 0) {
      const int row = mt.row[mt.slot_of[r]];
      while (ld_acquire(mt.ready + row) == 0) __nanosleep(256);  // its memo task is running
      h = mt.state[static_cast<int64_t>(row) * kMemoChunks + m0 - 1];
      k = m0 / cpb;                 // boundary hashes already written by k_memo_emit
      cc = cpb - m0 % cpb;
    }
  }
  const int c_start = kMemo ? __reduce_min_sync(kFull, valid ? m0 : 0x7fffffff) : 0;

  // fused assembly: chunk c's packed source of every request of the warp sits in smem slot
  // lsl[c % 4][perm(request)]; each lane prefetches its own request's entry for chunk c + 2
  // with cp.async in chunk c's copy group (complete before issue(c + 2) runs), and the
  // slot of chunk c survives until write_out(c) has used its valid counts
  const unsigned long long* csrc = nullptr;
  const int sub = lane >> 4, q = lane & 15;  // 2 requests per instruction, 16 lanes x 8 B
  const int me = perm_slot(lane);
  if (kGather) {
    __syncwarp();  // the previous task's readers of the slots are done
    wbase[me] = reinterpret_cast<unsigned long long>(g.tokens_out + s);
    csrc = g.chunk_src + (valid ? s / kChunk + r : 0);
    lsl[me] = nch > 0 ? csrc[0] : 0ull;
    lsl[32 + me] = nch > 1 ? csrc[1] : 0ull;
    __syncwarp();
  }

  auto issue = [&](int c) {
    unsigned char* st = wbuf + (c & 1) * kStageBytes;
    if (!kGather) {
      // CSR path: each lane publishes its own request's packed chunk source; the loader
      // below is then shared with the fused path (8 broadcast LDS.128 per half-warp
      // instead of 64 shuffles per chunk)
      const int64_t left = n - static_cast<int64_t>(c) * kChunk;
      const unsigned long long v = (left <= 0 || c < m0) ? 0ull : left >= kChunk ? kChunk : left;
      __syncwarp();
      lsl[(c & 3) * 32 + me] =
          (reinterpret_cast<unsigned long long>(tokens + s + static_cast<int64_t>(c) * kChunk) &
           kPtrMask) | (v << kVShift);
      __syncwarp();
    }
    {
      const unsigned long long* slot = lsl + (c & 3) * 32 + sub * 16;
      unsigned long long e[16];
#pragma unroll
      for (int t = 0; t < 16; t += 2) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(slot + t);
        e[t] = v.x;
        e[t + 1] = v.y;
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        if (q < static_cast<int>(e[t] >> kVShift))
          cp_async8(st + (2 * t + sub) * kRowBytes + q * 8,
                    reinterpret_cast<const uint64_t*>(e[t] & kPtrMask) + q, 8);
      }
      if (kGather) {
        unsigned long long* nxt = lsl + ((c + 2) & 3) * 32 + me;
        if (c + 2 < nch)
          cp_async8(nxt, csrc + c + 2, 8);
        else
          *nxt = 0ull;
      }
    }
    cp_commit();
  };
  // fused assembly: write staged chunk c of the warp's 32 requests to the token CSR
  auto write_out = [&](int c) {
    const unsigned char* st = wbuf + (c & 1) * kStageBytes;
    const unsigned long long* slot = lsl + (c & 3) * 32 + sub * 16;
    const unsigned long long* wb = wbase + sub * 16;
#pragma unroll
    for (int h8 = 0; h8 < 16; h8 += 8) {
      unsigned long long e[8], d[8];
      uint64_t v[8];
#pragma unroll
      for (int t = 0; t < 8; t += 2) {
        const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(slot + h8 + t);
        const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(wb + h8 + t);
        e[t] = a.x;
        e[t + 1] = a.y;
        d[t] = b.x;
        d[t + 1] = b.y;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t)
        v[t] = *reinterpret_cast<const uint64_t*>(st + (2 * (h8 + t) + sub) * kRowBytes + q * 8);
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (q < static_cast<int>(e[t] >> kVShift))
          reinterpret_cast<uint64_t*>(d[t])[static_cast<int64_t>(c) * kChunk + q] = v[t];
    }
  };

  issue(c_start);
  for (int c = c_start; c < maxch; ++c) {
    const int gz = gate ? gate_load(gate) : 0;
    if (c + 1 < maxch)
      issue(c + 1);
    else
      cp_commit();
    cp_wait1();
    __syncwarp();
    if (kGather) write_out(c);
    if (c < nch && !(kMemo && c < m0)) {
      const unsigned char* row = wbuf + (c & 1) * kStageBytes + lane * kRowBytes;
      const int64_t rem = n - static_cast<int64_t>(c) * kChunk;
      if (fast && rem >= kChunk) {
#pragma unroll
        for (int x = 0; x < kChunk / 2; ++x) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(row + 16 * x);
          h = fnv_token(h, v.x);
          h = fnv_token(h, v.y);
        }
        if (--cc == 0 || rem == kChunk) {  // block boundary or the last token
          out[k++] = h;
          cc = cpb;
        }
      } else {
        const int p1 = rem < kChunk ? static_cast<int>(rem) : kChunk;
        if (fast) {
          // the request's last, partial chunk: block boundaries (multiples of B, a multiple
          // of 16, from the chunk-aligned request start) fall only on full chunks, so the
          // one emit is the last token's (hierarchy.cpp:26)
          for (int p = 0; p < p1; ++p)
            h = fnv_token(h, *reinterpret_cast<const uint64_t*>(row + 8 * p));
          out[k++] = h;
        } else {
          // B % 16 != 0: per token; `left` counts down to the next boundary
          int64_t j = static_cast<int64_t>(c) * kChunk;  // position in the request
          int left = B - static_cast<int>(j % B);
          for (int p = 0; p < p1; ++p, ++j) {
            h = fnv_token(h, *reinterpret_cast<const uint64_t*>(row + 8 * p));
            if (--left == 0 || j + 1 == n) out[k++] = h;  // hierarchy.cpp:26
            if (left == 0) left = B;
          }
        }
      }
    }
    __syncwarp();
    if (gz) gate_wait(gate);
  }
  }  // task loop
}

// chain_boundary_hashes of ONE sequence (the drop-in calls): a split task on one warp, or
// one thread when B % 16 != 0 or the sequence is short.
__global__ void __launch_bounds__(32) k_hash_seq(const uint64_t* __restrict__ tokens, int64_t n,
                                                 int B, uint64_t* __restrict__ out, int split) {
  __shared__ __align__(16) unsigned char wbuf[2 * kStageBytes];
  if (split) {
    split_task(tokens, n, B, out, wbuf);
    return;
  }
  if (threadIdx.x) return;
  uint64_t h = kFnvOffset;
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    h = fnv_token(h, tokens[i]);
    if ((i + 1) % B == 0 || i + 1 == n) out[k++] = h;  // hierarchy.cpp:26
  }
}

// ------------------------------------------------------------- K1 task order
// K1 hashes requests longest first (split tasks, then 32-request tasks of near-equal
// lengths so the lanes of a warp finish together).  The order is a counting sort, descending
// over ORDER BUCKETS of the length: 32 per octave from 512 tokens (2.2% wide), 32-token-wide
// below; with a fixed split threshold the split requests get buckets of their own above all
// others.  Three kernels, no library sort: histogram (k_len_hist), bucket cursors and the
// split threshold (k_order_plan, one CTA), scatter (k_order_fill).
//
// The adaptive split threshold uses a coarser histogram derived from the order buckets: 8
// bins per octave from 512 tokens (bin 0 = shorter), requests and (estimated) tokens per
// bin; split bin k covers order buckets 32 + 4 (k - 1) .. 32 + 4 k - 1, so "bin >= k" is a
// suffix of the order.
constexpr int kHistBins = 80;
constexpr int kOrdPerOct = 32;
constexpr int kOrd = 32 + kOrdPerOct * 15;  // lengths below 512 * 2^15 tokens; longer share the top
constexpr int kOrdAll = 2 * kOrd;           // + the split buckets of a fixed threshold
static_assert(kOrdAll <= 1024, "k_order_plan scans the buckets with one CTA");
__device__ __forceinline__ int ord_of(int64_t n) {
  if (n < 512) return static_cast<int>(n >> 4);
  const int o = static_cast<int>(kOrdPerOct * log2(static_cast<double>(n) / 512.0));
  return min(32 + o, kOrd - 1);
}
__device__ __forceinline__ int bin_of_ord(int ob) {
  return ob < 32 ? 0 : min(1 + ((ob - 32) >> 2), kHistBins - 1);
}
__device__ __forceinline__ double bin_lo(int k) { return k == 0 ? 0.0 : 512.0 * exp2((k - 1) / 8.0); }

constexpr int kFillThreads = 1024;  // requests per CTA of k_len_hist / k_order_fill

struct OrderPlan {
  unsigned long long max_len;
  unsigned int ord[kOrdAll];          // requests per order bucket, then the bucket cursors
};

__device__ __forceinline__ int bucket_of(int64_t n, int64_t split_min) {
  return ord_of(n) + (split_min > 0 && n >= split_min ? kOrd : 0);
}

// With the prefix memo (mlen != null) a request's work is its length past the chunks the
// memo covers: the order, the split threshold and the split set use that length.
__device__ __forceinline__ int64_t work_len(const int64_t* tok_off, const int32_t* mlen, int r) {
  const int64_t n = tok_off[r + 1] - tok_off[r];
  return mlen ? n - 16 * static_cast<int64_t>(mlen[r]) : n;
}

__global__ void __launch_bounds__(kFillThreads) k_len_hist(const int64_t* tok_off, int R,
                                                           int64_t split_min, int* n_split,
                                                           OrderPlan* plan, const int32_t* mlen) {
  __shared__ unsigned int s_ord[kOrdAll];
  __shared__ unsigned long long s_max;
  for (int k = threadIdx.x; k < kOrdAll; k += blockDim.x) s_ord[k] = 0;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = r < R ? work_len(tok_off, mlen, r) : 0;
  const bool sp = split_min > 0 && n >= split_min;
  if (r < R) atomicAdd(s_ord + ord_of(n) + (sp ? kOrd : 0), 1u);
  if (split_min > 0) {  // fixed threshold: count the split requests here
    const unsigned m = __ballot_sync(kFull, sp);
    if (m && (threadIdx.x & 31) == 0) atomicAdd(n_split, __popc(m));
  }
  // one global atomic per CTA and bucket (all requests on one address would serialise in L2)
  const unsigned wmax = __reduce_max_sync(kFull, static_cast<unsigned>(n));  // n < 2^32
  if ((threadIdx.x & 31) == 0 && wmax) atomicMax(&s_max, static_cast<unsigned long long>(wmax));
  __syncthreads();
  for (int k = threadIdx.x; k < kOrdAll; k += blockDim.x)
    if (s_ord[k]) atomicAdd(plan->ord + k, s_ord[k]);
  if (threadIdx.x == 0 && s_max) atomicMax(&plan->max_len, s_max);
}

// One CTA of 1024 threads: (adaptive) the split threshold -- a makespan model of K1 on one
// B200 over "no split" and every bin edge from 512 tokens up: the longest one-lane task, the
// longest split task, the work (constants below); many long prompts keep one lane each
// (their chains overlap, config 3), a few long ones in a large batch, or any in a small
// batch, are split -- then the bucket cursors: exclusive scan of the counts in descending
// bucket order.
__global__ void __launch_bounds__(1024) k_order_plan(OrderPlan* plan, int adaptive, int* n_split) {
  __shared__ int64_t sm[33];
  __shared__ double s_cost[32];
  __shared__ int s_k[32];
  __shared__ unsigned long long s_tok[kHistBins], s_cnt[kHistBins];
  const int t = threadIdx.x;
  if (adaptive) {
    // the split model's histogram from the order buckets: requests per bin exact, tokens
    // as count x the bucket's mid length (buckets are 2.2% wide: the model's inputs to ~1%)
    if (t < kHistBins) s_tok[t] = s_cnt[t] = 0;
    __syncthreads();
    if (t < kOrd && plan->ord[t]) {
      const double mid = t < 32 ? 16.0 * t + 8.0 : 512.0 * exp2((t - 32 + 0.5) / kOrdPerOct);
      const int k = bin_of_ord(t);
      atomicAdd(s_cnt + k, static_cast<unsigned long long>(plan->ord[t]));
      atomicAdd(s_tok + k, static_cast<unsigned long long>(mid * plan->ord[t]));
    }
    __syncthreads();
    // measured on B200 (tools/k1_sweep.py, config-4 burst of 125k requests at thresholds
    // 4k..16k): a one-lane chain in a loaded SM ~90 ns per token, a split task ~8 ns per
    // token, ~280 Gtok/s one lane per request, a split token costs 2.8 lane tokens
    const double c_lane = 90e-9, c_split = 8e-9, rate = 280e9, extra = 1.8;
    // tokens of bins >= k (k = t): inclusive scan of the bins in descending order
    const int kd = kHistBins - 1 - t;  // thread t holds bin kHistBins - 1 - t
    const int64_t tk = t < kHistBins ? static_cast<int64_t>(s_tok[kd]) : 0;
    int64_t tot;
    const int64_t above = block_exscan(tk, sm, &tot) + tk;  // tokens in bins >= kd
    const double total = static_cast<double>(tot);
    const double lmax = static_cast<double>(plan->max_len);
    double cost = 1e300;
    int kk = -1;
    if (t < kHistBins && kd >= 1 && (s_cnt[kd] || above)) {
      const double T = bin_lo(kd);
      cost = fmax(fmax(T * c_lane, lmax * c_split), (total + extra * above) / rate);
      kk = kd;
    }
    // minimum cost, ties to the larger threshold (the model's scan from the top)
    for (int o = 16; o > 0; o >>= 1) {
      const double oc = __shfl_xor_sync(kFull, cost, o);
      const int ok = __shfl_xor_sync(kFull, kk, o);
      if (oc < cost || (oc == cost && ok > kk)) {
        cost = oc;
        kk = ok;
      }
    }
    if ((t & 31) == 0) {
      s_cost[t >> 5] = cost;
      s_k[t >> 5] = kk;
    }
    __syncthreads();
    if (t == 0) {
      double best = fmax(lmax * c_lane, total / rate);  // no split
      int bk = -1;
      for (int w = 0; w < 32; ++w)
        if (s_k[w] >= 0 && (s_cost[w] < best || (s_cost[w] == best && bk >= 0 && s_k[w] > bk))) {
          best = s_cost[w];
          bk = s_k[w];
        }
      unsigned long long ns = 0;
      if (bk >= 1)
        for (int k = bk; k < kHistBins; ++k) ns += s_cnt[k];
      *n_split = static_cast<int>(ns);
    }
  }
  // cursors: bucket b starts after every request of the buckets above it
  const int b = kOrdAll - 1 - t;
  const int64_t v = b >= 0 ? plan->ord[b] : 0;
  int64_t all;
  const int64_t ex = block_exscan(v, sm, &all);
  if (b >= 0) plan->ord[b] = static_cast<unsigned int>(ex);
}

// order[pos] = r: each CTA ranks its requests per bucket in shared memory and reserves its
// range of every bucket it touches with ONE global atomic (the lengths crowd into a few
// dozen buckets: per-warp atomics serialise in L2)
__global__ void __launch_bounds__(kFillThreads) k_order_fill(const int64_t* tok_off, int R,
                                                             int64_t split_min, OrderPlan* plan,
                                                             int32_t* order, const int32_t* mlen) {
  __shared__ unsigned int s_cnt[kOrdAll];
  for (int k = threadIdx.x; k < kOrdAll; k += blockDim.x) s_cnt[k] = 0;
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  int bk = -1;
  unsigned rk = 0;
  if (r < R) {
    bk = bucket_of(work_len(tok_off, mlen, r), split_min);
    rk = atomicAdd(s_cnt + bk, 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kOrdAll; k += blockDim.x)
    if (s_cnt[k]) s_cnt[k] = atomicAdd(plan->ord + k, s_cnt[k]);
  __syncthreads();
  if (bk >= 0) order[s_cnt[bk] + rk] = r;
}

__global__ void k_nblocks(const int64_t* tok_off, int R, int B, int64_t* nb) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) nb[r] = (tok_off[r + 1] - tok_off[r] + B - 1) / B;
  if (r == R) nb[R] = 0;
}

}  // namespace

extern "C" {

int pyg_hash_offsets_dev(pyg_ctx* c, const int64_t* d_tok_off, int32_t R, int64_t* d_hash_off,
                         int64_t* total) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0) return PYG_EINVAL;
  size_t tmp = 0;
  PYG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, static_cast<int64_t*>(nullptr), d_hash_off,
                                         R + 1, c->stream));
  void* sp;
  int rc = scratch(c, (R + 2) * sizeof(int64_t) + tmp + 256, &sp);
  if (rc) return rc;
  auto* nb = static_cast<int64_t*>(sp);
  void* d_tmp = static_cast<char*>(sp) + (((R + 2) * sizeof(int64_t) + 255) & ~size_t{255});
  k_nblocks<<<(R + 256) / 256, 256, 0, c->stream>>>(d_tok_off, R, c->B, nb);
  PYG_LAUNCHED(c);
  PYG_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, nb, d_hash_off, R + 1, c->stream));
  PYG_LAUNCHED(c);
  if (total) {
    PYG_CUDA(cudaMemcpyAsync(total, d_hash_off + R, 8, cudaMemcpyDeviceToHost, c->stream));
    PYG_CUDA(cudaStreamSynchronize(c->stream));
  }
  return PYG_OK;
}

}  // extern "C"

namespace pyg_host {
// Per-device one-time setup of K1: its dynamic shared memory attribute and the P^(8t)
// table of split tasks (both are per device, so cached per device id).
cudaError_t device_setup(int dev) {
  static bool done[64] = {};
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (done[dev]) return cudaSuccess;
  cudaError_t e = cudaSetDevice(dev);
  if (e != cudaSuccess) return e;
  for (const void* f : {reinterpret_cast<const void*>(k_hash_staged<false, kWarps, false>),
                        reinterpret_cast<const void*>(k_hash_staged<true, kWarps, false>)}) {
    e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOneCta);
    if (e != cudaSuccess) return e;
  }
  e = cudaFuncSetAttribute(k_hash_staged<false, kWarps, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOneCta);
  if (e != cudaSuccess) return e;
  uint64_t pw[kSplitTok + 1];
  uint64_t q = 1;
  for (int t = 0; t <= kSplitTok; ++t) {
    pw[t] = q;
    for (int i = 0; i < 8; ++i) q *= kFnvPrime;
  }
  e = cudaMemcpyToSymbol(c_pw8, pw, sizeof(pw));
  if (e != cudaSuccess) return e;
  done[dev] = true;
  return cudaSuccess;
}

int sm_count(int dev) {
  static int n[64] = {};
  if (dev < 0 || dev >= 64) return 1;
  if (!n[dev]) cudaDeviceGetAttribute(&n[dev], cudaDevAttrMultiProcessorCount, dev);
  return n[dev] > 0 ? n[dev] : 1;
}
}  // namespace pyg_host

namespace pyg_host {
int hash_seq_launch(pyg_ctx* c, const uint64_t* d_tok, int64_t n, uint64_t* d_hash) {
  if (n <= 0) return PYG_OK;
  PYG_CUDA(device_setup(c->device));
  const int split = (c->B % kSplitTok == 0 && n >= 64) ? 1 : 0;
  k_hash_seq<<<1, 32, 0, c->stream>>>(d_tok, n, c->B, d_hash, split);
  PYG_LAUNCHED(c);
  return PYG_OK;
}
}  // namespace pyg_host

// task order (descending length, for warp balance) + the K1 launch
template <bool kGather>
static int hash_launch(pyg_ctx* c, const uint64_t* d_src, const int64_t* d_tok_off, int32_t R,
                       const int64_t* d_hash_off, uint64_t* d_hashes, GatherSrc g) {
  const size_t vb = (static_cast<size_t>(R) * 4 + 255) & ~size_t{255};
  // prefix memo: CSR path, whole-chunk blocks, persistent grid (a warp waiting for a memo
  // row relies on the row's task having been taken by a running warp), bursts large enough
  // to amortise the election
  const bool memo = !kGather && c->B % kChunk == 0 && c->hash_memo && c->hash_grid == 1 &&
                    R >= 1024;
  uint32_t mcap = 1024;
  while (memo && mcap < 2u * static_cast<uint32_t>(R)) mcap <<= 1;
  const size_t tab_b = memo ? static_cast<size_t>(mcap) * 20 : 0;
  const size_t rows_b = memo ? static_cast<size_t>(kMemoRows) * (kMemoChunks * 8 + 12) : 0;
  void* sp;
  int rc = scratch(c, vb + 256 + ((sizeof(OrderPlan) + 255) & ~size_t{255}) + tab_b + 2 * vb +
                          rows_b + 256, &sp);
  if (rc) return rc;
  char* p = static_cast<char*>(sp);
  auto* v_out = reinterpret_cast<int32_t*>(p);
  auto* ctr0 = reinterpret_cast<int*>(p + vb);
  auto* plan = reinterpret_cast<OrderPlan*>(p + vb + 256);
  // [0] task counter, [1] split requests, [2] memo rows; the order plan
  PYG_CUDA(cudaMemsetAsync(ctr0, 0, 256 + sizeof(OrderPlan), c->stream));
  MemoTab mt{};
  if (memo) {
    char* q = p + vb + 256 + ((sizeof(OrderPlan) + 255) & ~size_t{255});
    mt.lead = reinterpret_cast<unsigned long long*>(q);                      // 8 B / slot
    mt.key = reinterpret_cast<uint32_t*>(q + static_cast<size_t>(mcap) * 8);  // 4
    mt.cnt = reinterpret_cast<int32_t*>(q + static_cast<size_t>(mcap) * 12);  // 4
    mt.row = reinterpret_cast<int32_t*>(q + static_cast<size_t>(mcap) * 16);  // 4
    q += tab_b;
    mt.slot_of = reinterpret_cast<int32_t*>(q);
    q += vb;
    mt.mlen = reinterpret_cast<int32_t*>(q);
    q += vb;
    mt.state = reinterpret_cast<uint64_t*>(q);
    mt.ready = reinterpret_cast<int32_t*>(q + static_cast<size_t>(kMemoRows) * kMemoChunks * 8);
    mt.row_lead = mt.ready + kMemoRows;
    mt.row_chunks = mt.row_lead + kMemoRows;
    mt.n_rows = ctr0 + 2;
    mt.mask = mcap - 1;
    PYG_CUDA(cudaMemsetAsync(mt.lead, 0, static_cast<size_t>(mcap) * 16, c->stream));
    PYG_CUDA(cudaMemsetAsync(mt.ready, 0, static_cast<size_t>(kMemoRows) * 4, c->stream));
    k_memo_elect<<<(R + 255) / 256, 256, 0, c->stream>>>(d_src, d_tok_off, R, mt);
    PYG_LAUNCHED(c);
    k_memo_rows<<<(mcap + 255) / 256, 256, 0, c->stream>>>(mt);
    PYG_LAUNCHED(c);
    k_memo_clamp<<<1, 1, 0, c->stream>>>(mt.n_rows);
    PYG_LAUNCHED(c);
    k_memo_match<<<std::min((R + 7) / 8, 16 * pyg_host::sm_count(c->device)), 256, 0,
                   c->stream>>>(d_src, d_tok_off, R, mt);
    PYG_LAUNCHED(c);
  }
  // split tasks: the fused-assembly loader and B % 16 != 0 keep one lane per request
  const int64_t split_min0 = (!kGather && c->B % kSplitTok == 0) ? c->split_min : 0;
  const int nb = (R + kFillThreads - 1) / kFillThreads;
  k_len_hist<<<nb, kFillThreads, 0, c->stream>>>(d_tok_off, R, split_min0, ctr0 + 1, plan,
                                                 mt.mlen);
  PYG_LAUNCHED(c);
  k_order_plan<<<1, 1024, 0, c->stream>>>(plan, split_min0 < 0 ? 1 : 0, ctr0 + 1);
  PYG_LAUNCHED(c);
  k_order_fill<<<nb, kFillThreads, 0, c->stream>>>(d_tok_off, R, split_min0, plan, v_out,
                                                   mt.mlen);
  PYG_LAUNCHED(c);
  PYG_CUDA(pyg_host::device_setup(c->device));
  const int n_sm = pyg_host::sm_count(c->device);
  const int cap = c->hash_ctas > 0 ? std::min(c->hash_ctas, n_sm) : n_sm;
  const int tasks_max = (R + 31) / 32 + (split_min0 ? R : 0);
  const bool persistent = c->hash_grid == 1;
  const int per = (tasks_max + kWarps - 1) / kWarps;  // CTAs of one task per warp
  const int grid = persistent ? std::max(1, std::min(per, cap)) : std::max(1, per);  // 1/SM
  // grid mode 2: shared memory padded so that one K1 CTA fits per SM (the rest of the SM
  // stays free for the step's kernels; device_setup allows the padded size)
  const int pad = c->hash_grid == 2 ? kSmemOneCta : 0;
  int* next = persistent ? ctr0 : nullptr;
  // the admission gate needs room for admission CTAs beside the paused K1 CTAs: honoured
  // with the persistent grid (<= one CTA per SM of 148) and grid mode 2 (one per SM) only
  const int32_t* gate = c->hash_grid != 0 ? c->hash_gate : nullptr;
  if (memo) {
    k_hash_staged<false, kWarps, true><<<grid, kWarps * 32, smem_bytes(kWarps), c->stream>>>(
        d_src, d_tok_off, R, v_out, d_hash_off, d_hashes, c->B, next, g, ctr0 + 1, gate, mt, n_sm);
    PYG_LAUNCHED(c);
    k_memo_emit<<<std::min((R + 7) / 8, 16 * n_sm), 256, 0, c->stream>>>(d_tok_off, d_hash_off,
                                                                          d_hashes, R, c->B, mt);
  } else {
    // grid mode 2: the SM's shared memory at its 164 KB setting (carveout 72 %), which holds
    // the padded K1 CTA (117 KB) and a K3 CTA (46 KB) but not an admission CTA (104 KB):
    // measured 86 vs 84 M req/s against the driver's choice for K1 alone (132 KB), 71 with
    // the 196 / 228 KB settings (an admission CTA then slows the K1 beside it).  The
    // attribute is per function: set when the mode changes (the gate sets its own).
    static int carve_set[64] = {};  // per device: 0 unset, else carveout + 1
    const int want = c->hash_grid == 2 ? 72 : -1;  // -1: the driver's default
    const int dev = c->device >= 0 && c->device < 64 ? c->device : 0;
    if (!c->hash_gate && carve_set[dev] != want + 1) {
      PYG_CUDA(cudaFuncSetAttribute(k_hash_staged<kGather, kWarps, false>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, want));
      carve_set[dev] = want + 1;
    }
  }
  if (!memo)
    k_hash_staged<kGather, kWarps, false><<<grid, kWarps * 32,
                                            std::max(pad, smem_bytes(kWarps)), c->stream>>>(
        d_src, d_tok_off, R, v_out, d_hash_off, d_hashes, c->B, next, g, ctr0 + 1, gate, mt, n_sm);
  PYG_LAUNCHED(c);
  return PYG_OK;
}

extern "C" {

int pyg_hash_batch_dev(pyg_ctx* c, const uint64_t* d_tokens, const int64_t* d_tok_off, int32_t R,
                       const int64_t* d_hash_off, uint64_t* d_hashes) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0) return PYG_EINVAL;
  if (R == 0) return PYG_OK;
  return hash_launch<false>(c, d_tokens, d_tok_off, R, d_hash_off, d_hashes, GatherSrc{});
}

int pyg_assemble_hash_dev(pyg_ctx* c, int32_t R, const int64_t* d_seg_off,
                          const pyg_segment* d_segs, int64_t n_segs, const uint64_t* d_pool,
                          int64_t n_tokens, int64_t* d_tok_off, uint64_t* d_tokens,
                          int64_t* d_hash_off, uint64_t* d_hashes) {
  PYG_ON_DEVICE(c);
  if (!c || R < 0 || n_segs < 0 || n_tokens < 0) return PYG_EINVAL;
  int rc = pyg_host::assemble_offsets(c, R, d_seg_off, d_segs, d_tok_off);
  if (rc) return rc;
  rc = pyg_hash_offsets_dev(c, d_tok_off, R, d_hash_off, nullptr);
  if (rc || R == 0) return rc;
  // chunk source table + side buffer for boundary-straddling chunks
  const int64_t tab_cap = n_tokens / kChunk + R + 1;
  const int64_t side_cap = std::max<int64_t>(n_segs, 1);
  const size_t tb = (static_cast<size_t>(tab_cap) * 8 + 255) & ~size_t{255};
  void* ap;
  rc = aux(c, tb + static_cast<size_t>(side_cap) * kChunk * 8 + 256, &ap);
  if (rc) return rc;
  auto* tab = static_cast<unsigned long long*>(ap);
  auto* side = reinterpret_cast<uint64_t*>(static_cast<char*>(ap) + tb);
  auto* ctr = reinterpret_cast<unsigned long long*>(side + side_cap * kChunk);
  PYG_CUDA(cudaMemsetAsync(ctr, 0, 8, c->stream));
  const int n_sm = pyg_host::sm_count(c->device);
  k_chunk_src<<<std::min((R + 7) / 8, 16 * n_sm), 256, 0, c->stream>>>(
      R, d_seg_off, d_segs, d_pool, d_tok_off, tab, tab_cap, side, side_cap, ctr, c->hd.error);
  PYG_LAUNCHED(c);
  return hash_launch<true>(c, d_pool, d_tok_off, R, d_hash_off, d_hashes,
                           GatherSrc{tab, d_tokens});
}

int pyg_set_hash_memo(pyg_ctx* c, int32_t on) {
  PYG_ON_DEVICE(c);
  if (!c) return PYG_EINVAL;
  c->hash_memo = on ? 1 : 0;
  return PYG_OK;
}

int pyg_set_hash_gate(pyg_ctx* c, pyg_ctx* step) {
  PYG_ON_DEVICE(c);
  if (!c) return PYG_EINVAL;
  if (!step) {
    c->hash_gate = nullptr;
    return PYG_OK;
  }
  if (step->device != c->device) return PYG_EINVAL;
  if (!step->d_gate) {
    PYG_CUDA(cudaMalloc(&step->d_gate, sizeof(int32_t)));
    PYG_CUDA(cudaMemset(step->d_gate, 0, sizeof(int32_t)));
  }
  PYG_CUDA(pyg_host::device_setup(c->device));
  // the whole 228 KB as shared memory on the SMs K1 runs on: an SM's L1/shared split is
  // fixed while CTAs are resident, and with the split the driver picks for K1 alone (~100 KB)
  // the admission CTAs (~103 KB) could not start beside a paused K1 CTA (k_admit asks for
  // the same when its ctx has a gate)
  for (const void* f : {reinterpret_cast<const void*>(k_hash_staged<false, kWarps, false>),
                        reinterpret_cast<const void*>(k_hash_staged<false, kWarps, true>),
                        reinterpret_cast<const void*>(k_hash_staged<true, kWarps, false>)})
    PYG_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  cudaSharedmemCarveoutMaxShared));
  c->hash_gate = step->d_gate;
  return PYG_OK;
}

int pyg_set_hash_split(pyg_ctx* c, int64_t min_tokens) {
  PYG_ON_DEVICE(c);
  if (!c || min_tokens < -1) return PYG_EINVAL;
  c->split_min = min_tokens < 0 ? -1 : (min_tokens + 3) & ~int64_t{3};
  return PYG_OK;
}

int pyg_set_hash_grid(pyg_ctx* c, int32_t mode) {
  PYG_ON_DEVICE(c);
  if (!c || mode < 0 || mode > 2) return PYG_EINVAL;
  c->hash_grid = mode;
  return PYG_OK;
}

int pyg_set_hash_ctas(pyg_ctx* c, int32_t n_ctas) {
  PYG_ON_DEVICE(c);
  if (!c || n_ctas < 0) return PYG_EINVAL;
  c->hash_ctas = n_ctas;
  return PYG_OK;
}

}  // extern "C"
