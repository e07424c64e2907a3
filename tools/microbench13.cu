// Design microbenchmark #13 (not product code): TMA operand delivery of the config-4 contraction
// without any MMA.  128 CTAs, each streaming its share of the (pe tile, k-block) units of a
// 4096 x 14848 u8 "pe" operand in 128-row x 128-byte boxes (plus one 304-row digit box per unit
// from a small 304 x 14848 operand shared by all CTAs) through an S-stage ring of full barriers.
// Question: is the contraction's operand pipeline slowed by the row-major pe layout (each 16 KB box
// = 128 rows of 128 bytes, 14848 bytes apart) against a tiled layout in which every box is one
// contiguous 16 KB block?
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int P = 4096, LE = 14848, KB = LE / 128, TILES = P / 128, NDIG = 304;

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(bar),
               "r"(parity) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
               "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar) : "memory");
}

// one thread issues and waits (no consumer work): the ring depth S bounds the bytes in flight
__global__ void __launch_bounds__(32, 1) stream_kernel(const __grid_constant__ CUtensorMap tm_pe,
                                                       const __grid_constant__ CUtensorMap tm_dig, int S, int tiled,
                                                       int with_dig, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[16];
  const uint32_t base = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
  const uint32_t a_bytes = 128 * 128, b_bytes = with_dig ? 2 * 152 * 128 : 0, stage = a_bytes + b_bytes;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init((uint32_t)__cvta_generic_to_shared(&bars[s]), 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int units = TILES * KB;
  const int u0 = blockIdx.x * units / gridDim.x, u1 = (blockIdx.x + 1) * units / gridDim.x;
  int i = 0;
  for (int u = u0; u < u1; ++u, ++i) {
    const int s = i % S;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[s]);
    if (i >= S) mbar_wait(bar, ((i / S) - 1) & 1);
    const int tile = u / KB, kb = u % KB;
    mbar_expect_tx(bar, stage);
    const uint32_t dst = base + (uint32_t)s * stage;
    if (tiled) tma2d(dst, &tm_pe, 0, (tile * KB + kb) * 128, bar);  // contiguous 16 KB block
    else tma2d(dst, &tm_pe, kb * 128, tile * 128, bar);             // 128 rows, 14848 B apart
    if (with_dig) {
      tma2d(dst + a_bytes, &tm_dig, kb * 128, 0, bar);
      tma2d(dst + a_bytes + 152 * 128, &tm_dig, kb * 128, 152, bar);
    }
  }
  for (int j = i - S > 0 ? i - S : 0; j < i; ++j) mbar_wait((uint32_t)__cvta_generic_to_shared(&bars[j % S]), (j / S) & 1);
  sink[blockIdx.x] = i;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_map(EncodeFn fn, CUtensorMap* m, void* ptr, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_rows) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld};
  cuuint32_t box[2] = {128, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  EncodeFn fn = reinterpret_cast<EncodeFn>(p);
  uint8_t *pe, *dig;
  unsigned long long* sink;
  CK(cudaMalloc(&pe, (size_t)P * LE));
  CK(cudaMalloc(&dig, (size_t)NDIG * LE));
  CK(cudaMalloc(&sink, 4096 * 8));
  CK(cudaMemset(pe, 1, (size_t)P * LE));
  CK(cudaMemset(dig, 1, (size_t)NDIG * LE));
  CUtensorMap m_row, m_tile, m_dig;
  // row-major [P][LE]; tiled [TILES*KB*128 rows][128 B] (the same bytes, box = one contiguous block)
  if (!make_map(fn, &m_row, pe, LE, P, LE, 128) || !make_map(fn, &m_tile, pe, 128, (uint64_t)TILES * KB * 128, 128, 128) ||
      !make_map(fn, &m_dig, dig, LE, NDIG, LE, 152)) {
    fprintf(stderr, "tensor map failed\n");
    return 1;
  }
  const int smem = 8 * (128 * 128 + 2 * 152 * 128) + 1024;
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 230400));
  for (int with_dig = 0; with_dig < 2; ++with_dig)
    for (int S : {3, 4, 6, 8})
      for (int tiled = 0; tiled < 2; ++tiled) {
        const int stage = 128 * 128 + (with_dig ? 2 * 152 * 128 : 0);
        const int sm = S * stage + 1024;
        if (sm > 230400) continue;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int w = 0; w < 3; ++w)
          stream_kernel<<<128, 32, sm>>>(tiled ? m_tile : m_row, m_dig, S, tiled, with_dig, sink);
        CK(cudaGetLastError());
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r) stream_kernel<<<128, 32, sm>>>(tiled ? m_tile : m_row, m_dig, S, tiled, with_dig, sink);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)TILES * KB * stage;
        printf("digits %d stages %d %-9s: %.4f ms  %.2f TB/s into shared memory\n", with_dig, S, tiled ? "tiled" : "row-major",
               ms / 20, bytes / (ms / 20 * 1e-3) / 1e12);
      }
  (void)smem;
  return 0;
}
