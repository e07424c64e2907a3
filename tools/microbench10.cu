// Design microbenchmark #10 (not product code): warp-private histogram bins for short-chunk
// count-contract.  Each warp owns R copies of 256 u32 bins (R = 1, 2, 4, 8; copy = lane / (32 / R),
// bin e of copy r at word e * R + r) instead of the CTA-level 32 lane replicas; the question is what
// same-address / bank conflicts under Zipf(1.2) cost per ATOMS, since a warp-private histogram can be
// flushed per chunk with 256 / 32 * R words per lane instead of 32 KB per CTA.
// Trace: 8 distinct Zipf draws per 8-byte record (as the generator produces), 4.64 GB.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__global__ void fill_records_kernel(uint8_t* t, int64_t n, const uint32_t* cdf, uint32_t total, int shuffle) {
  __shared__ uint32_t s_cdf[257];
  for (int i = threadIdx.x; i < 257; i += blockDim.x) s_cdf[i] = cdf[i];
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n / 8; r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t e[8]; int got = 0; uint32_t ctr = 0;
    while (got < 8) {
      uint32_t x = mix32((uint32_t)(r * 64 + ctr++) * 0x9e3779b9U ^ (uint32_t)(r >> 26)) % total;
      int lo = 0, hi = 256;
      while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (s_cdf[mid] <= x) lo = mid; else hi = mid; }
      uint32_t v = (uint32_t)(lo * 167) & 255u; bool dup = false;
      for (int j = 0; j < got; ++j) dup |= e[j] == v;
      if (!dup) e[got++] = v;
    }
    if (shuffle) {  // random order of the 8 picks inside the record
      uint32_t h = mix32((uint32_t)r ^ 0xabcdef01u);
      for (int i = 7; i > 0; --i) { int j = h % (i + 1); h = mix32(h); uint32_t tmp = e[i]; e[i] = e[j]; e[j] = tmp; }
    }
    uint2 w = make_uint2(0, 0);
    for (int j = 0; j < 4; ++j) { w.x |= e[j] << (8 * j); w.y |= e[4 + j] << (8 * j); }
    reinterpret_cast<uint2*>(t)[r] = w;
  }
}
__device__ __forceinline__ int4 ldg_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel)); return r;
}
__device__ __forceinline__ void atoms_inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a)); }

// R copies per warp; R == 32 means the CTA-level lane-replicated layout of the product (rows of 128 B)
template <int R>
__global__ void __launch_bounds__(512, 2) hist_kernel(const int4* __restrict__ v, int64_t nvec, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint32_t* smw = reinterpret_cast<uint32_t*>(sm);
  const int words = R == 32 ? 256 * 32 : 16 * 256 * R;
  for (int i = threadIdx.x; i < words; i += blockDim.x) smw[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t wbase = R == 32 ? base + lane * 4 : base + warp * 256 * R * 4 + (lane / (32 / R)) * 4;
  const int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  const int64_t v0 = blockIdx.x * per, v1 = min(nvec, v0 + per);
  for (int64_t i = v0 + threadIdx.x; i + 15 * 512 < v1; i += 16 * 512) {
    int4 x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = ldg_stream(v + i + u * 512);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const uint32_t wd[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b) atoms_inc(wbase + prmt(wd[q], 0u, 0x4440u | (uint32_t)b) * (R == 32 ? 128u : 4u * R));
    }
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) s += smw[i];
  if (s) atomicAdd(out, (unsigned long long)s);
}

template <int R>
float run(const int4* v, int64_t nvec, unsigned long long* out, int grid) {
  const int smem = (R == 32 ? 256 * 32 : 16 * 256 * R) * 4;
  CK(cudaFuncSetAttribute(hist_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) hist_kernel<R><<<grid, 512, smem>>>(v, nvec, out);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) hist_kernel<R><<<grid, 512, smem>>>(v, nvec, out);
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 10;
}

int main(int argc, char** argv) {
  const double s = argc > 1 ? atof(argv[1]) : 1.2;
  const int shuffle = argc > 2 ? atoi(argv[2]) : 0;
  const int64_t n = (int64_t)10000000 * 58 * 8;
  std::vector<double> w(256); double tot = 0;
  for (int r = 0; r < 256; ++r) { w[r] = s == 0 ? 1.0 : pow(r + 1, -s); tot += w[r]; }
  std::vector<uint32_t> cdf(257); double acc = 0; const uint32_t T = 1u << 30;
  for (int r = 0; r <= 256; ++r) { cdf[r] = (uint32_t)(acc / tot * T); if (r < 256) acc += w[r]; }
  cdf[256] = T;
  uint8_t* t; uint32_t* dc; unsigned long long* out;
  CK(cudaMalloc(&t, n)); CK(cudaMalloc(&dc, 257 * 4)); CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(dc, cdf.data(), 257 * 4, cudaMemcpyHostToDevice));
  fill_records_kernel<<<148 * 8, 256>>>(t, n, dc, T, shuffle);
  CK(cudaDeviceSynchronize());
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * 2; const int64_t nvec = n / 16;
  printf("zipf %.1f shuffle %d  R=1 (1 KB/warp)  %.3f ms\n", s, shuffle, run<1>((int4*)t, nvec, out, grid));
  printf("zipf %.1f shuffle %d  R=2 (2 KB/warp)  %.3f ms\n", s, shuffle, run<2>((int4*)t, nvec, out, grid));
  printf("zipf %.1f shuffle %d  R=4 (4 KB/warp)  %.3f ms\n", s, shuffle, run<4>((int4*)t, nvec, out, grid));
  printf("zipf %.1f shuffle %d  R=8 (8 KB/warp)  %.3f ms\n", s, shuffle, run<8>((int4*)t, nvec, out, grid));
  printf("zipf %.1f shuffle %d  R=32 lane replicas per CTA (product layout)  %.3f ms\n", s, shuffle, run<32>((int4*)t, nvec, out, grid));
  return 0;
}
