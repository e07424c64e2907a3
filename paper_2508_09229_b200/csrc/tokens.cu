// Per-token hop totals for every token (SPEC.md:336-344 token_hops, applied to the whole trace):
//   hops[q*N + i] = sum_l sum_k pe_q[l][planes[l][(t0+i)*K + k]]      (q < 4, uint32 out)
// Layer-major planes need a cross-layer sum per token, so this kernel is token-tiled: a CTA owns
// a tile of TPT*blockDim tokens, walks the L layers, stages each layer's replicated W=1 table in
// shared memory (row = expert, slot = lane*4: conflict-free LDS.32 via one PRMT), and keeps each
// token's four placement sums in registers as u16 lanes until the end of the tile.
#include "common.cuh"

namespace mp {

constexpr int kTokThreads = 256;
constexpr int kTPT = 8;  // tokens per thread per tile

template <bool K8, bool SMALLP>
__global__ void __launch_bounds__(kTokThreads) token_hops_kernel(const uint8_t* __restrict__ planes, int64_t stride,
                                                                 int64_t t0, int64_t n, int L, int K,
                                                                 const uint32_t* __restrict__ tables,
                                                                 uint32_t* __restrict__ hops) {
  extern __shared__ __align__(128) uint8_t sm[];  // 256 rows x 128 B
  uint32_t* smw = reinterpret_cast<uint32_t*>(sm);
  const int lane = threadIdx.x & 31;
  const uint32_t base = smem_addr(sm);
  const uint32_t slot8 = (uint32_t)(lane << 3);  // PRMT yields (e << 8) | (lane << 3); >> 1 -> row e*128 + lane*4
  const uint32_t slot = (uint32_t)(lane << 2);
  const int64_t tile = (int64_t)kTPT * blockDim.x;
  for (int64_t ta = (int64_t)blockIdx.x * tile; ta < n; ta += (int64_t)gridDim.x * tile) {
    uint32_t acc[kTPT][2];  // per token: u16 lanes {q0, q2} and {q1, q3}
#pragma unroll
    for (int j = 0; j < kTPT; ++j) acc[j][0] = acc[j][1] = 0;
    for (int l = 0; l < L; ++l) {
      __syncthreads();
      for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x)
        smw[(i >> 5) * 32 + (i & 31)] = __ldg(tables + (int64_t)l * 256 + (i >> 5));
      __syncthreads();
      const uint8_t* plane = planes + (int64_t)l * stride + (t0 + ta) * K;
#pragma unroll
      for (int j = 0; j < kTPT; ++j) {
        const int64_t i = (int64_t)j * blockDim.x + threadIdx.x;  // token within tile (coalesced per j)
        if (ta + i >= n) continue;
        uint32_t s8 = 0;
        if constexpr (K8) {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(plane + i * 8));
          const uint32_t wv[2] = {v.x, v.y};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const uint32_t w = lds32(base + (prmt(wv[h], slot8, sel_row(b)) >> 1));
              if constexpr (SMALLP) {
                s8 += w;  // 4 lookups x max_p <= 63 fit a u8 lane
              } else {
                acc[j][0] += w & 0x00ff00ffu;
                acc[j][1] += (w >> 8) & 0x00ff00ffu;
              }
            }
            if constexpr (SMALLP) {
              acc[j][0] += s8 & 0x00ff00ffu;
              acc[j][1] += (s8 >> 8) & 0x00ff00ffu;
              s8 = 0;
            }
          }
        } else {
          for (int k = 0; k < K; ++k) {
            const uint32_t e = plane[i * K + k];
            const uint32_t w = lds32(base + e * 128 + slot);
            acc[j][0] += w & 0x00ff00ffu;
            acc[j][1] += (w >> 8) & 0x00ff00ffu;
          }
        }
      }
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

template <bool K8, bool SMALLP>
static void run_token_hops(int64_t tiles, int nsm, const uint8_t* planes, int64_t stride, int64_t t0, int64_t n,
                           int L, int K, const uint32_t* tables, uint32_t* hops, cudaStream_t s) {
  const int smem = 256 * 128;
  int per_sm = 0;
  cudaFuncSetAttribute(token_hops_kernel<K8, SMALLP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, token_hops_kernel<K8, SMALLP>, kTokThreads, smem);
  const int64_t grid = max((int64_t)1, min(tiles, (int64_t)nsm * max(1, per_sm)));
  token_hops_kernel<K8, SMALLP><<<(unsigned)grid, kTokThreads, smem, s>>>(planes, stride, t0, n, L, K, tables, hops);
}

cudaError_t launch_token_hops(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K,
                              const uint32_t* tables, int max_p, uint32_t* hops, cudaStream_t s) {
  const int64_t n = t1 - t0;
  if (n <= 0) return cudaSuccess;
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (n + (int64_t)kTPT * kTokThreads - 1) / ((int64_t)kTPT * kTokThreads);
  if (K == 8 && max_p <= 63) run_token_hops<true, true>(tiles, nsm, planes, stride, t0, n, L, K, tables, hops, s);
  else if (K == 8) run_token_hops<true, false>(tiles, nsm, planes, stride, t0, n, L, K, tables, hops, s);
  else run_token_hops<false, false>(tiles, nsm, planes, stride, t0, n, L, K, tables, hops, s);
  return cudaGetLastError();
}

}  // namespace mp
