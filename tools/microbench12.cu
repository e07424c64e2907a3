// Design microbenchmark #12 (not product code): per-chunk histograms for SHORT chunks (140 tokens =
// 1120 B per (layer, chunk) piece, the paper's dialog length) with WARP-private bins instead of the
// CTA's lane-replicated sets.  Each warp owns a contiguous run of pieces; per piece it loads one
// 8-pick record per lane (uint2, 5 rounds of 32 records), ATOMS into its own bins, then "flushes":
// every lane reads 8 bins (x R replicas), folds them into a dummy contraction and zeroes them.
// Question: what does a warp-private histogram + per-piece flush cost per byte, against the
// segmented gather's 4 LDS.128 wavefronts per 32 bytes (16 placements) -- i.e. is a per-chunk
// count + contraction path viable at 140 tokens per chunk?
//   R     replicas per bin (lane % R), bins [256][R] u32 per warp
//   ROT   rotate each lane's record by 8 * (lane & 7) bits, so one ATOMS instruction does not send
//         the hot pick slot (slot 0 = first Zipf draw) of 32 tokens to the same address
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
__device__ __forceinline__ uint2 ldg2(const uint2* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel)); return r;
}
__device__ __forceinline__ void atoms_inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a) : "memory"); }
__device__ __forceinline__ uint32_t lds(uint32_t a) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v; }
__device__ __forceinline__ void sts(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }

constexpr int kChunk = 140;
constexpr int kRounds = (kChunk + 31) / 32;

template <int R, bool ROT>
__global__ void __launch_bounds__(512, 2) wp_kernel(const uint2* __restrict__ rec, int64_t n_pieces, int64_t* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t wb = (uint32_t)__cvta_generic_to_shared(sm) + wid * 256 * R * 4;
  for (int i = lane; i < 256 * R; i += 32) sts(wb + 4 * i, 0);
  __syncwarp();
  const uint32_t rb = wb + (lane % R) * 4;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5), w = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  const int64_t per = (n_pieces + nw - 1) / nw, p0 = w * per, p1 = min(n_pieces, p0 + per);
  const uint32_t rot = 8 * (lane & 7);
  uint32_t acc = 0;
  for (int64_t p = p0; p < p1; ++p) {
    const uint2* pr = rec + p * kChunk;
    uint2 x[kRounds];
#pragma unroll
    for (int r = 0; r < kRounds; ++r) x[r] = (r * 32 + (int)lane < kChunk) ? ldg2(pr + r * 32 + lane) : make_uint2(0, 0);
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      uint32_t a = x[r].x, b = x[r].y;
      if (ROT) {
        const uint32_t a2 = __funnelshift_r(a, b, rot), b2 = __funnelshift_r(b, a, rot);
        a = a2; b = b2;
      }
      if (r * 32 + (int)lane < kChunk) {
#pragma unroll
        for (int k = 0; k < 4; ++k) atoms_inc(rb + prmt(a, 0u, 0x4440u | k) * (4 * R));
#pragma unroll
        for (int k = 0; k < 4; ++k) atoms_inc(rb + prmt(b, 0u, 0x4440u | k) * (4 * R));
      }
    }
    __syncwarp();
    // flush: lane owns bins lane + 32 j; dummy contraction c * (bin + 1)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t e = lane + 32 * j;
      uint32_t c = 0;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        c += lds(wb + (e * R + q) * 4);
        sts(wb + (e * R + q) * 4, 0);
      }
      acc += c * (e + 1);
    }
    __syncwarp();
  }
  if (acc == 0x12345678u) out[0] = acc;
  atomicAdd((unsigned long long*)out + 1, (unsigned long long)acc);
}

template <int R, bool ROT>
void run(const uint2* rec, int64_t n_pieces, int64_t* out, int nsm, const char* name, double bytes) {
  auto k = wp_kernel<R, ROT>;
  const int smem = 16 * 256 * R * 4;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 512, smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) k<<<nsm * per_sm, 512, smem>>>(rec, n_pieces, out);
  CK(cudaGetLastError());
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<nsm * per_sm, 512, smem>>>(rec, n_pieces, out);
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s R=%d rot=%d CTAs/SM=%d: %.3f ms  %.1f GB/s\n", name, R, (int)ROT, per_sm, ms / 5, bytes / (ms / 5 * 1e6));
}

int main() {
  const int64_t n_rec = (int64_t)10000000 * 58 / kChunk * kChunk;  // whole pieces
  const int64_t n = n_rec * 8;
  std::vector<double> wgt(256); double tot = 0;
  for (int r = 0; r < 256; ++r) { wgt[r] = pow(r + 1, -1.2); tot += wgt[r]; }
  std::vector<uint32_t> cdf(257); double acc = 0; const uint32_t T = 1u << 30;
  for (int r = 0; r <= 256; ++r) { cdf[r] = (uint32_t)(acc / tot * T); if (r < 256) acc += wgt[r]; }
  cdf[256] = T;
  uint8_t* t; uint32_t* dc; int64_t* out;
  CK(cudaMalloc(&t, n)); CK(cudaMalloc(&dc, 257 * 4)); CK(cudaMalloc(&out, 16));
  CK(cudaMemcpy(dc, cdf.data(), 257 * 4, cudaMemcpyHostToDevice));
  fill_records_kernel<<<148 * 8, 256>>>(t, n, dc, T);
  CK(cudaDeviceSynchronize());
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int64_t np = n_rec / kChunk;
  printf("# %lld pieces of %d records (%.2f GB)\n", (long long)np, kChunk, n / 1e9);
  run<1, false>((const uint2*)t, np, out, nsm, "warp bins", (double)n);
  run<1, true>((const uint2*)t, np, out, nsm, "warp bins", (double)n);
  run<2, false>((const uint2*)t, np, out, nsm, "warp bins", (double)n);
  run<2, true>((const uint2*)t, np, out, nsm, "warp bins", (double)n);
  run<4, true>((const uint2*)t, np, out, nsm, "warp bins", (double)n);
  return 0;
}
