// Per-token hop totals for every token (SPEC.md:336-344 token_hops, applied to the whole trace):
//   hops[q*N + i] = sum_l sum_k pe_q[l][planes[l][(t0+i)*K + k]]      (q < 4, uint32 out)
// Layer-major planes need a cross-layer sum per token, so this kernel is token-tiled: a CTA owns
// a tile of TPT*blockDim tokens and walks the L layers, keeping each token's four placement sums
// in registers as u16 lanes.  Each layer's W=1 table is staged in shared memory replicated per
// lane (row = expert, slot = lane*4: conflict-free LDS.32 via one PRMT); the replicated tables
// are expanded once into global memory (32 KB per layer, L2-resident) and streamed into a
// double buffer with cp.async, so layer l+1's table lands while layer l is being gathered and
// each layer costs one barrier.
#include "common.cuh"

namespace mp {

#ifndef MP_TOK_PF
#define MP_TOK_PF 1
#endif

// Tile shape (R1, 10M tokens): 512 threads x 8 tokens, 2 CTAs/SM = 1.18 ms; 512 x 16 (1 CTA/SM)
// 1.26, 256 x 16 (3 CTAs) 1.23, 256 x 8 (3 CTAs) 1.28, 512 x 4 1.46 ms.
#ifndef MP_TOK_THREADS
#define MP_TOK_THREADS 512
#endif
#ifndef MP_TOK_TPT
#define MP_TOK_TPT 8
#endif
#ifndef MP_TOK_MINB
#define MP_TOK_MINB 2
#endif
constexpr int kTokThreads = MP_TOK_THREADS;
constexpr int kTPT = MP_TOK_TPT;          // tokens per thread per tile (512 x 8 -> 4096-token tiles)
constexpr int kRowBytes = 128;            // 32 lanes x 4 B
constexpr int kTabBytes = 256 * kRowBytes;  // 32 KB per layer

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// replicated[l][e][r] = tables[l][e] for r < 32 (one-time expansion, 32 KB per layer)
__global__ void replicate_kernel(const uint32_t* __restrict__ tables, int L, uint32_t* __restrict__ rep) {
  const int64_t n = (int64_t)L * 256 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rep[i] = tables[i >> 5];
}

// One layer of the token-tiled gather: the thread's kTPT tokens (ta + j*blockDim + tid) add their K
// lookups in layer table `base` (replicated rows, PRMT-addressed) into u16 lanes {q0,q2}, {q1,q3}.
template <bool K8, int ACC>
__device__ __forceinline__ void gather_layer(const uint8_t* __restrict__ plane, uint32_t base, uint32_t slot,
                                             int64_t ta, int64_t n, int K, uint32_t (&acc)[kTPT][2]) {
  if constexpr (K8) {
    uint2 v[kTPT];
#pragma unroll
    for (int j = 0; j < kTPT; ++j) {
      const int64_t i = (int64_t)j * blockDim.x + threadIdx.x;
      v[j] = (ta + i < n) ? __ldg(reinterpret_cast<const uint2*>(plane + i * 8)) : make_uint2(0, 0);
    }
#pragma unroll
    for (int j = 0; j < kTPT; ++j) {
      const uint32_t wv[2] = {v[j].x, v[j].y};
      uint32_t w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) w[k] = lds32(base + prmt(wv[k >> 2], slot, sel_row(k & 3)));
      if constexpr (ACC == 8) {  // max_p <= 31: a token's 8 lookups fit u8 lanes
        const uint32_t s8 = (w[0] + w[1] + w[2]) + (w[3] + w[4] + w[5]) + (w[6] + w[7]);
        acc[j][0] += s8 & 0x00ff00ffu;
        acc[j][1] += (s8 >> 8) & 0x00ff00ffu;
      } else if constexpr (ACC == 4) {  // max_p <= 63: 4 lookups per u8 lane
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t s8 = (w[4 * h] + w[4 * h + 1] + w[4 * h + 2]) + w[4 * h + 3];
          acc[j][0] += s8 & 0x00ff00ffu;
          acc[j][1] += (s8 >> 8) & 0x00ff00ffu;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          acc[j][0] += w[k] & 0x00ff00ffu;
          acc[j][1] += (w[k] >> 8) & 0x00ff00ffu;
        }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kTPT; ++j) {
      const int64_t i = (int64_t)j * blockDim.x + threadIdx.x;
      if (ta + i >= n) continue;
      for (int k = 0; k < K; ++k) {
        const uint32_t e = plane[i * K + k];
        const uint32_t w = lds32(base + e * 256 + slot);
        acc[j][0] += w & 0x00ff00ffu;
        acc[j][1] += (w >> 8) & 0x00ff00ffu;
      }
    }
  }
}

template <bool K8, int ACC>
__global__ void __launch_bounds__(kTokThreads, MP_TOK_MINB) token_hops_kernel(const uint8_t* __restrict__ planes, int64_t stride,
                                                                 int64_t t0, int64_t n, int L, int K,
                                                                 const uint32_t* __restrict__ rep,
                                                                 uint32_t* __restrict__ hops) {
  // 256 rows x 256 B: row e holds expert e's replicated word of table buffer 0 at bytes [0, 128)
  // and of buffer 1 at [128, 256), so PRMT's (e << 8) | lane*4 is the address with no shift
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31;
  const uint32_t base0 = smem_addr(sm);
  const uint32_t slot = (uint32_t)(lane << 2);
  const int64_t tile = (int64_t)kTPT * blockDim.x;
  auto fetch = [&](int l, int buf) {  // async copy of layer l's replicated table into buffer buf
    const uint8_t* src = reinterpret_cast<const uint8_t*>(rep) + (int64_t)l * kTabBytes;
    for (int i = threadIdx.x; i < kTabBytes / 16; i += blockDim.x)  // 8 x 16 B per expert row
      cp_async16(base0 + (i >> 3) * 256 + buf * kRowBytes + (i & 7) * 16, src + i * 16);
    cp_async_commit();
  };
  for (int64_t ta = (int64_t)blockIdx.x * tile; ta < n; ta += (int64_t)gridDim.x * tile) {
    uint32_t acc[kTPT][2];  // per token: u16 lanes {q0, q2} and {q1, q3}
#pragma unroll
    for (int j = 0; j < kTPT; ++j) acc[j][0] = acc[j][1] = 0;
    __syncthreads();  // previous tile done with both buffers
    fetch(0, 0);
    for (int l = 0; l < L; ++l) {
      cp_async_wait_all();
      __syncthreads();  // layer l's table visible; buffer (l+1)&1 free
      if (l + 1 < L) {
        fetch(l + 1, (l + 1) & 1);
#if MP_TOK_PF
        // pull layer l+1's slice of this tile into L2 while layer l is gathered
        if (threadIdx.x == 0) {
          const uintptr_t a0 = reinterpret_cast<uintptr_t>(planes + (int64_t)(l + 1) * stride + (t0 + ta) * K);
          const uintptr_t a1 = reinterpret_cast<uintptr_t>(planes + (int64_t)(l + 1) * stride + (t0 + min(n, ta + tile)) * K);
          const uintptr_t lo = a0 & ~(uintptr_t)15, hi = (a1 + 15) & ~(uintptr_t)15;
          if (hi > lo) prefetch_l2(reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo));
        }
#endif
      }
      const uint32_t base = base0 + (l & 1) * kRowBytes;
      const uint8_t* plane = planes + (int64_t)l * stride + (t0 + ta) * K;
      gather_layer<K8, ACC>(plane, base, slot, ta, n, K, acc);
    }
#pragma unroll
    for (int j = 0; j < kTPT; ++j) {
      const int64_t i = (int64_t)j * blockDim.x + threadIdx.x;
      if (ta + i >= n) continue;
      const int64_t t = ta + i;
      hops[0 * n + t] = acc[j][0] & 0xffffu;
      hops[2 * n + t] = acc[j][0] >> 16;
      hops[1 * n + t] = acc[j][1] & 0xffffu;
      hops[3 * n + t] = acc[j][1] >> 16;
    }
  }
}

// ---- token-tiled scoring (MP_ALGO_TOKEN): per-chunk hop sums whose cost does not depend on C -----
// Same tile / layer walk as token_hops_kernel, with the layer tables staged by the CTA itself from
// the compact W-word tables (word w = placements 4w..4w+3; 4 x LDG + 4 x STS.128 per thread per
// layer, double-buffered through registers) and, instead of writing per-token totals, a segmented
// reduction per 32-token warp group: chunk ids are non-decreasing across the lanes, so a
// Hillis-Steele scan that adds only equal keys is exact, and each segment's last lane adds the
// segment's four sums to hop_sums[4w+q][c] (int64 atomics).  Streaming kernels pay per (layer,
// chunk) piece and collapse when chunks are short (10M R1 tokens in 150k chunks: 32-56 ms); this
// one stays at ~1.2 ms for any C.
__device__ __forceinline__ void sts128(uint32_t a, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(a), "r"(w) : "memory");
}

template <bool K8, int ACC>
__global__ void __launch_bounds__(kTokThreads, MP_TOK_MINB)
score_tok_kernel(const uint8_t* __restrict__ planes, int64_t stride, int64_t t0, int64_t n, int L, int K,
                 const int64_t* __restrict__ bounds, int C, const uint32_t* __restrict__ tables, int W, int w,
                 int64_t* __restrict__ hop_sums) {
  extern __shared__ __align__(128) uint8_t sm[];  // 256 rows x 256 B: two interleaved table buffers
  constexpr int kStage = 256 * 8 / kTokThreads;    // 16-byte replica stores per thread per layer
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base0 = smem_addr(sm);
  const uint32_t slot = (uint32_t)(lane << 2);
  const int64_t tile = (int64_t)kTPT * blockDim.x;
  uint32_t wd[kStage];
  auto load_words = [&](int l) {
#pragma unroll
    for (int k = 0; k < kStage; ++k) {
      const int e = (threadIdx.x + k * blockDim.x) >> 3;
      wd[k] = __ldg(tables + ((int64_t)l * 256 + e) * W + w);
    }
  };
  auto store_words = [&](int buf) {
#pragma unroll
    for (int k = 0; k < kStage; ++k) {
      const int i = threadIdx.x + k * blockDim.x;
      sts128(base0 + (i >> 3) * 256 + buf * kRowBytes + (i & 7) * 16, wd[k]);
    }
  };
  for (int64_t ta = (int64_t)blockIdx.x * tile; ta < n; ta += (int64_t)gridDim.x * tile) {
    uint32_t acc[kTPT][2];
#pragma unroll
    for (int j = 0; j < kTPT; ++j) acc[j][0] = acc[j][1] = 0;
    load_words(0);
    __syncthreads();  // previous tile done with both buffers
    store_words(0);
    for (int l = 0; l < L; ++l) {
      __syncthreads();  // layer l's table visible; buffer (l+1)&1 no longer read
      if (l + 1 < L) load_words(l + 1);  // in flight while layer l is gathered
      const uint8_t* plane = planes + (int64_t)l * stride + (t0 + ta) * K;
      gather_layer<K8, ACC>(plane, base0 + (l & 1) * kRowBytes, slot, ta, n, K, acc);
      if (l + 1 < L) store_words((l + 1) & 1);
    }
    // chunk of each group's first token: lane j binary-searches group j (in parallel)
    int cj = 0;
    if (lane < kTPT) {
      const int64_t tf = t0 + ta + (int64_t)lane * blockDim.x + warp * 32;
      int lo = 0, hi = C;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(bounds + mid) <= tf) lo = mid; else hi = mid;
      }
      cj = lo;
    }
#pragma unroll
    for (int j = 0; j < kTPT; ++j) {
      const int64_t i = (int64_t)j * blockDim.x + threadIdx.x;
      const bool valid = ta + i < n;
      int c = __shfl_sync(0xffffffffu, cj, j);
      if (valid) {
        const int64_t t = t0 + ta + i;
        while (c + 1 < C && __ldg(bounds + c + 1) <= t) ++c;  // boundaries inside the 32-token group
      } else {
        c = 0x7fffffff;  // sentinel: after every real chunk, keeps keys sorted
      }
      uint32_t v[4] = {valid ? acc[j][0] & 0xffffu : 0u, valid ? acc[j][1] & 0xffffu : 0u,
                       valid ? acc[j][0] >> 16 : 0u, valid ? acc[j][1] >> 16 : 0u};
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int co = __shfl_up_sync(0xffffffffu, c, off);
        const bool same = lane >= off && co == c;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t o = __shfl_up_sync(0xffffffffu, v[q], off);
          if (same) v[q] += o;
        }
      }
      const int cn = __shfl_down_sync(0xffffffffu, c, 1);
      if (valid && (lane == 31 || cn != c)) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (v[q]) atomic_add_i64(hop_sums + (int64_t)q * C + c, (int64_t)v[q]);
      }
    }
  }
}

template <bool K8, int ACC>
static cudaError_t run_score_tok(int nsm, const uint8_t* planes, int64_t stride, int64_t t0, int64_t n, int L, int K,
                                 const int64_t* bounds, int C, const uint32_t* tables, int W, int64_t* hop_sums,
                                 cudaStream_t s) {
  const int smem = 256 * 256;
  int per_sm = 0;
  const cudaError_t e = prepare_kernel((const void*)score_tok_kernel<K8, ACC>, kTokThreads, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (n + (int64_t)kTPT * kTokThreads - 1) / ((int64_t)kTPT * kTokThreads);
  const int64_t grid = max((int64_t)1, min(tiles, (int64_t)nsm * max(1, per_sm)));
  for (int w = 0; w < W; ++w)  // one pass per table word (4 placements each)
    score_tok_kernel<K8, ACC><<<(unsigned)grid, kTokThreads, smem, s>>>(planes, stride, t0, n, L, K, bounds, C,
                                                                        tables, W, w, hop_sums + (int64_t)4 * w * C);
  return cudaGetLastError();
}

cudaError_t launch_score_tok(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K,
                             const int64_t* bounds, int C, const uint32_t* tables, int W, int max_p, int64_t* hop_sums,
                             cudaStream_t s) {
  const int64_t n = t1 - t0;
  if (n <= 0) return cudaSuccess;
  const int nsm = device_sm_count();
  if (K == 8 && max_p <= 31) return run_score_tok<true, 8>(nsm, planes, stride, t0, n, L, K, bounds, C, tables, W, hop_sums, s);
  if (K == 8 && max_p <= 63) return run_score_tok<true, 4>(nsm, planes, stride, t0, n, L, K, bounds, C, tables, W, hop_sums, s);
  if (K == 8) return run_score_tok<true, 1>(nsm, planes, stride, t0, n, L, K, bounds, C, tables, W, hop_sums, s);
  return run_score_tok<false, 1>(nsm, planes, stride, t0, n, L, K, bounds, C, tables, W, hop_sums, s);
}

template <bool K8, int ACC>
static void run_token_hops(int64_t tiles, int nsm, const uint8_t* planes, int64_t stride, int64_t t0, int64_t n,
                           int L, int K, const uint32_t* rep, uint32_t* hops, cudaStream_t s) {
  const int smem = 256 * 256;  // two interleaved table buffers
  int per_sm = 0;
  prepare_kernel((const void*)token_hops_kernel<K8, ACC>, kTokThreads, smem, &per_sm);
  const int64_t grid = max((int64_t)1, min(tiles, (int64_t)nsm * max(1, per_sm)));
  token_hops_kernel<K8, ACC><<<(unsigned)grid, kTokThreads, smem, s>>>(planes, stride, t0, n, L, K, rep, hops);
}

cudaError_t launch_token_hops(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K,
                              const uint32_t* tables, int max_p, uint32_t* replicated, uint32_t* hops,
                              cudaStream_t s) {
  const int64_t n = t1 - t0;
  if (n <= 0) return cudaSuccess;
  const int nsm = device_sm_count();
  const int64_t nrep = (int64_t)L * 256 * 32;
  replicate_kernel<<<(unsigned)min((nrep + 255) / 256, (int64_t)4096), 256, 0, s>>>(tables, L, replicated);
  const int64_t tiles = (n + (int64_t)kTPT * kTokThreads - 1) / ((int64_t)kTPT * kTokThreads);
  if (K == 8 && max_p <= 31) run_token_hops<true, 8>(tiles, nsm, planes, stride, t0, n, L, K, replicated, hops, s);
  else if (K == 8 && max_p <= 63) run_token_hops<true, 4>(tiles, nsm, planes, stride, t0, n, L, K, replicated, hops, s);
  else if (K == 8) run_token_hops<true, 1>(tiles, nsm, planes, stride, t0, n, L, K, replicated, hops, s);
  else run_token_hops<false, 1>(tiles, nsm, planes, stride, t0, n, L, K, replicated, hops, s);
  return cudaGetLastError();
}

}  // namespace mp
