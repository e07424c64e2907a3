// Design microbenchmark #9 (not product code): shared-memory histogram ATOMS with lane-replicated
// bins under different row pitches / bit-7 placement, on a Zipf(1.2) u8 trace (R1-sized 10M x 58 x 8
// bytes).  Question: why does pipe_kernel (128-byte rows) show ~1.2 shared wavefronts per ATOMS
// (ncu l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom ~ 20 % of ATOMS) while the segmented
// gather's histogram (256-byte rows, replicas in the upper half) shows ~4 %?
//   variant 0: addr = e*128 + lane*4              (pipe_kernel layout)
//   variant 1: addr = e*256 + lane*4              (256-byte pitch, lower half)
//   variant 2: addr = e*256 + 128 + lane*4        (256-byte pitch, upper half: seg_kernel W=1)
//   variant 3: addr = e*128 + ((lane ^ (e & 31))*4)  (128-byte rows, bank rotated by expert)
//   variant 4: addr = (e>>1)*256 + (e&1)*128 + lane*4 == variant 0 (control, different arithmetic)
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
__global__ void fill_kernel(uint8_t* t, int64_t n, const uint32_t* cdf, uint32_t total) {
  __shared__ uint32_t s_cdf[257];
  for (int i = threadIdx.x; i < 257; i += blockDim.x) s_cdf[i] = cdf[i];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n / 4; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t out = 0;
    for (int j = 0; j < 4; ++j) {
      uint32_t r = mix32((uint32_t)(i * 4 + j) * 0x9e3779b9U ^ (uint32_t)((i * 4) >> 32)) % total;
      int lo = 0, hi = 256;
      while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (s_cdf[mid] <= r) lo = mid; else hi = mid; }
      out |= ((uint32_t)(lo * 167) & 255u) << (8 * j);
    }
    reinterpret_cast<uint32_t*>(t)[i] = out;
  }
}
// 8 distinct Zipf draws per aligned 8-byte record (as the trace generator produces), in draw order
// (mode 1) or sorted by expert id (mode 2)
__global__ void fill_records_kernel(uint8_t* t, int64_t n, const uint32_t* cdf, uint32_t total, int mode) {
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
    if (mode == 2)
      for (int i = 1; i < 8; ++i) for (int j = i; j > 0 && e[j - 1] > e[j]; --j) { uint32_t tmp = e[j]; e[j] = e[j - 1]; e[j - 1] = tmp; }
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

template <int V>
__device__ __forceinline__ uint32_t bin_addr(uint32_t word, int b, uint32_t base, uint32_t lane) {
  const uint32_t e = prmt(word, 0u, 0x4440u | (uint32_t)b);
  if constexpr (V == 0) return base + e * 128u + lane * 4u;
  if constexpr (V == 1) return base + e * 256u + lane * 4u;
  if constexpr (V == 2) return base + e * 256u + 128u + lane * 4u;
  if constexpr (V == 3) return base + e * 128u + ((lane ^ (e & 31u)) << 2);
  return base + (e >> 1) * 256u + (e & 1u) * 128u + lane * 4u;
}

template <int V>
__global__ void __launch_bounds__(512, 2) hist_kernel(const int4* __restrict__ v, int64_t nvec, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint32_t* smw = reinterpret_cast<uint32_t*>(sm);
  const int words = (V == 1 || V == 2) ? 256 * 64 : 256 * 32;
  for (int i = threadIdx.x; i < words; i += blockDim.x) smw[i] = 0;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm), lane = threadIdx.x & 31;
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
        for (int b = 0; b < 4; ++b) atoms_inc(bin_addr<V>(wd[q], b, base, lane));
    }
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < words; i += blockDim.x) s += smw[i];
  if (s) atomicAdd(out, (unsigned long long)s);
}

template <int V>
float run(const int4* v, int64_t nvec, unsigned long long* out, int grid) {
  const int smem = (V == 1 || V == 2) ? 65536 : 32768;
  CK(cudaFuncSetAttribute(hist_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) hist_kernel<V><<<grid, 512, smem>>>(v, nvec, out);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) hist_kernel<V><<<grid, 512, smem>>>(v, nvec, out);
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 10;
}

int main(int argc, char** argv) {
  const double s = argc > 1 ? atof(argv[1]) : 1.2;
  const int64_t n = (int64_t)10000000 * 58 * 8;
  std::vector<double> w(256); double tot = 0;
  for (int r = 0; r < 256; ++r) { w[r] = s == 0 ? 1.0 : pow(r + 1, -s); tot += w[r]; }
  std::vector<uint32_t> cdf(257); double acc = 0; const uint32_t T = 1u << 30;
  for (int r = 0; r <= 256; ++r) { cdf[r] = (uint32_t)(acc / tot * T); if (r < 256) acc += w[r]; }
  cdf[256] = T;
  uint8_t* t; uint32_t* dc; unsigned long long* out;
  CK(cudaMalloc(&t, n)); CK(cudaMalloc(&dc, 257 * 4)); CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(dc, cdf.data(), 257 * 4, cudaMemcpyHostToDevice));
  const int mode = argc > 2 ? atoi(argv[2]) : 0;  // 0 i.i.d. bytes, 1 distinct records, 2 sorted records
  if (mode == 0) fill_kernel<<<148 * 8, 256>>>(t, n, dc, T);
  else fill_records_kernel<<<148 * 8, 256>>>(t, n, dc, T, mode);
  CK(cudaDeviceSynchronize());
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * 2; const int64_t nvec = n / 16;
  const char* names[] = {"pitch128 (pipe_kernel)", "pitch256 lower half", "pitch256 upper half (seg W=1)",
                         "pitch128 lane^e rotated", "pitch128 alt arithmetic"};
  float ms[5] = {run<0>((int4*)t, nvec, out, grid), run<1>((int4*)t, nvec, out, grid), run<2>((int4*)t, nvec, out, grid),
                 run<3>((int4*)t, nvec, out, grid), run<4>((int4*)t, nvec, out, grid)};
  const char* modes[] = {"iid bytes", "distinct records", "sorted records"};
  for (int i = 0; i < 5; ++i) printf("zipf %.1f %-17s %-32s %.3f ms  %.1f GB/s\n", s, modes[mode], names[i], ms[i], n / (ms[i] * 1e6));
  return 0;
}
