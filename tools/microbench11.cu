// Design microbenchmark #11 (not product code): lane-replicated histogram ATOMS into ONE 64 KB set
// (rows of 256 B, the split pipe_kernel layout, half 0) placed at a given offset inside the dynamic
// shared-memory allocation, with the trace streamed by ld.global.nc.L1::no_allocate as in the product.
// Question: why do pipe_kernel's ATOMS count ~18 % extra wavefronts when its three 64 KB sets rotate,
// and almost none when every piece uses the first set?
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
__global__ void fill_records_kernel(uint8_t* t, int64_t n, const uint32_t* cdf, uint32_t total) {
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

// 1024 threads = two halves (half h at bytes h*128 of each 256-B row); the set starts at `off` bytes
__global__ void __launch_bounds__(1024, 1) hist_kernel(const int4* __restrict__ v, int64_t nvec, int off, int smem,
                                                     unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint32_t* smw = reinterpret_cast<uint32_t*>(sm);
  for (int i = threadIdx.x; i < smem / 4; i += blockDim.x) smw[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, half = threadIdx.x >> 9, tid = threadIdx.x & 511;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm) + off + half * 128 + lane * 4;
  const int64_t workers = (int64_t)gridDim.x * 2, w = (int64_t)blockIdx.x * 2 + half;
  const int64_t per = (nvec + workers - 1) / workers;
  const int64_t v0 = w * per, v1 = min(nvec, v0 + per);
  for (int64_t i = v0 + tid; i + 15 * 512 < v1; i += 16 * 512) {
    int4 x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = ldg_stream(v + i + u * 512);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const uint32_t wd[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b) atoms_inc(prmt(wd[q], 0u, 0x4440u | (uint32_t)b) * 256u + sb);
    }
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < smem / 4; i += blockDim.x) s += smw[i];
  if (s) atomicAdd(out, (unsigned long long)s);
}

int main(int argc, char** argv) {
  const int64_t n = (int64_t)10000000 * 58 * 8;
  std::vector<double> wgt(256); double tot = 0;
  for (int r = 0; r < 256; ++r) { wgt[r] = pow(r + 1, -1.2); tot += wgt[r]; }
  std::vector<uint32_t> cdf(257); double acc = 0; const uint32_t T = 1u << 30;
  for (int r = 0; r <= 256; ++r) { cdf[r] = (uint32_t)(acc / tot * T); if (r < 256) acc += wgt[r]; }
  cdf[256] = T;
  uint8_t* t; uint32_t* dc; unsigned long long* out;
  CK(cudaMalloc(&t, n)); CK(cudaMalloc(&dc, 257 * 4)); CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(dc, cdf.data(), 257 * 4, cudaMemcpyHostToDevice));
  fill_records_kernel<<<148 * 8, 256>>>(t, n, dc, T);
  CK(cudaDeviceSynchronize());
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  CK(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608));
  const int cfg[][2] = {{0, 65536}, {0, 196608}, {16384, 196608}, {32768, 196608}, {65536, 196608},
                        {98304, 196608}, {131072, 196608}, {65536, 131072}};
  for (auto& c : cfg) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) hist_kernel<<<nsm, 1024, c[1]>>>((const int4*)t, n / 16, c[0], c[1], out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) hist_kernel<<<nsm, 1024, c[1]>>>((const int4*)t, n / 16, c[0], c[1], out);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("set at offset %6d KB of %3d KB smem: %.3f ms  %.1f GB/s\n", c[0] / 1024, c[1] / 1024, ms / 5, n / (ms / 5 * 1e6));
  }
  return 0;
}
