// Token-major -> layer-plane ingestion (an ActivationTrace is per token, L lists
// of K expert ids).  A caller holding token-major uint8 [n][L][K] selections (router output, a
// numpy array, a pinned host buffer streamed slice by slice) gets them into the engine's layer
// planes with one device transpose per slice, so the end-to-end path never transposes on the host.
//
// K = 8 (R1): a (token, layer) record is one u64, so the slice is a u64 matrix [n][L] and the
// kernel is a tiled transpose: a CTA stages 64 tokens x L records (64*L*8 B, coalesced u64 loads,
// row pitch L|1 words so the column reads of a half-warp hit distinct bank pairs), then writes
// 512 contiguous bytes per plane.  HBM-bound: 2 bytes moved per trace byte.  Other K: one thread
// per output byte (K*L-strided reads), used for the smaller 16B shape only.
#include <algorithm>
#include "common.cuh"

namespace mp {
namespace {

constexpr int kTT = 64;        // tokens per tile
constexpr int kIngestThreads = 256;

__global__ void __launch_bounds__(kIngestThreads) tok2planes_k8(const uint64_t* __restrict__ tok, int64_t n, int L,
                                                                 uint64_t* __restrict__ planes, int64_t stride_w,
                                                                 int64_t t_out) {
  extern __shared__ uint64_t tile[];  // [kTT][Lp]
  const int Lp = L | 1;
  const int64_t n_tiles = (n + kTT - 1) / kTT;
  for (int64_t tt = blockIdx.x; tt < n_tiles; tt += gridDim.x) {
    const int64_t i0 = tt * kTT;
    const int nt = (int)min((int64_t)kTT, n - i0);
    const uint64_t* src = tok + i0 * L;
    const int words = nt * L;
    for (int w = threadIdx.x; w < words; w += kIngestThreads) {
      const int i = w / L, l = w - i * L;
      tile[i * Lp + l] = __ldg(src + w);
    }
    __syncthreads();
    const int outs = L * kTT;
    for (int w = threadIdx.x; w < outs; w += kIngestThreads) {
      const int l = w / kTT, i = w - l * kTT;
      if (i < nt) planes[(int64_t)l * stride_w + t_out + i0 + i] = tile[i * Lp + l];
    }
    __syncthreads();
  }
}

__global__ void tok2planes_any(const uint8_t* __restrict__ tok, int64_t n, int L, int K, uint8_t* __restrict__ planes,
                               int64_t stride, int64_t t_out) {
  const int64_t per_plane = n * K;
  const int64_t total = per_plane * L;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)(j / per_plane);
    const int64_t b = j - (int64_t)l * per_plane;
    const int64_t i = b / K;
    const int k = (int)(b - i * K);
    planes[(int64_t)l * stride + t_out * K + b] = tok[(i * L + l) * K + k];
  }
}

}  // namespace

cudaError_t launch_tokens_to_planes(const uint8_t* tok, int64_t n, int L, int K, uint8_t* planes, int64_t stride,
                                    int64_t t_out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int sms = device_sm_count();
  if (K == 8 && ((uintptr_t)tok & 7) == 0) {
    const size_t smem = (size_t)kTT * (L | 1) * 8;
    int per_sm = 0;
    const cudaError_t e = prepare_kernel((const void*)tok2planes_k8, kIngestThreads, (int)smem, &per_sm);
    if (e != cudaSuccess) return e;
    const int64_t tiles = (n + kTT - 1) / kTT;
    const int grid = (int)std::min(tiles, (int64_t)sms * 6);
    tok2planes_k8<<<grid, kIngestThreads, smem, s>>>(reinterpret_cast<const uint64_t*>(tok), n, L,
                                                     reinterpret_cast<uint64_t*>(planes), stride / 8, t_out);
  } else {
    const int64_t total = n * K * (int64_t)L;
    const int grid = (int)std::min((total + 255) / 256, (int64_t)sms * 16);
    tok2planes_any<<<grid, 256, 0, s>>>(tok, n, L, K, planes, stride, t_out);
  }
  return cudaGetLastError();
}

}  // namespace mp
