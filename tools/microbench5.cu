// Design microbenchmark #5 (warp-specialised TMA gather) (not product code): read-ceiling variants and PRMT-addressed gathers.
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
__global__ void fill_kernel(uint8_t* planes, int64_t plane_bytes, int L, const uint32_t* cdf, uint32_t total) {
  __shared__ uint32_t s_cdf[257];
  for (int i = threadIdx.x; i < 257; i += blockDim.x) s_cdf[i] = cdf[i];
  __syncthreads();
  int64_t n = plane_bytes * L / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i * 4; int l = (int)(b / plane_bytes); uint32_t out = 0;
    for (int j = 0; j < 4; ++j) {
      uint32_t r = mix32((uint32_t)(b + j) * 0x9e3779b9U ^ (uint32_t)(b >> 32)) % total;
      int lo = 0, hi = 256;
      while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (s_cdf[mid] <= r) lo = mid; else hi = mid; }
      out |= ((uint32_t)(lo * 167 + l * 31) & 255u) << (8 * j);
    }
    reinterpret_cast<uint32_t*>(planes)[i] = out;
  }
}
__device__ __forceinline__ int4 ldg_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ldg_plain(const int4* p) { return __ldg(p); }


__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) { uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel)); return r; }
__device__ __forceinline__ uint32_t lds32(uint32_t a) { uint32_t r; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a)); return r; }
__device__ __forceinline__ uint4 lds128(uint32_t a) { uint4 r; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a)); return r; }
#define SEL(b) (0x5504u | ((b) << 4))

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(a), "r"(n)); }
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t ph) {
  asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(a), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) { asm volatile("mbarrier.arrive.shared.b64 _, [%0];" :: "r"(a) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint32_t a, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(a), "r"(bytes) : "memory"); }
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// Warp-specialised TMA score: warp 0 = producer (one elected lane issues bulk copies into a ring of
// STAGES x SB bytes), warps 1..NC = consumers (LDS.128 the staged trace, PRMT+LDS.32 gathers).
// The whole trace is one flat byte range here (table reloaded on layer change by consumers).
template <int STAGES, int SB, int NC>
__global__ void __launch_bounds__(32 * (NC + 1)) score_ws_kernel(const uint8_t* __restrict__ src, int64_t plane, int L,
                                                                 const uint32_t* __restrict__ pe, unsigned long long* sums) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* tab = sm;                    // 64 KB table rows (256 B)
  uint8_t* ring = sm + 65536;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nbytes = plane * L;
  const int64_t per = ((nbytes / SB + gridDim.x - 1) / gridDim.x) * SB;
  const int64_t b0 = blockIdx.x * per, b1 = min(nbytes, b0 + per);
  const int nst = b1 > b0 ? (int)((b1 - b0 + SB - 1) / SB) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init((uint32_t)__cvta_generic_to_shared(&full[s]), 1);
      mbar_init((uint32_t)__cvta_generic_to_shared(&empty[s]), NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      for (int it = 0; it < nst; ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait((uint32_t)__cvta_generic_to_shared(&empty[s]), ((it / STAGES) - 1) & 1);
        const int64_t off = b0 + (int64_t)it * SB;
        const uint32_t bytes = (uint32_t)min((int64_t)SB, b1 - off);
        const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
        mbar_expect(fb, bytes);
        bulk_g2s((uint32_t)__cvta_generic_to_shared(ring + s * SB), src + off, bytes, fb);
      }
    }
    return;
  }
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
  const uint32_t slot = (uint32_t)(lane << 2);
  const int ct = threadIdx.x - 32;  // consumer thread index
  int cur_l = -1;
  unsigned long long tot[4] = {0, 0, 0, 0};
  for (int it = 0; it < nst; ++it) {
    const int s = it % STAGES;
    const int64_t off = b0 + (int64_t)it * SB;
    const int l = (int)(off / plane);  // SB divides plane here
    if (l != cur_l) {
      asm volatile("bar.sync 1, %0;" :: "r"(32 * NC));
      for (int i = ct; i < 256 * 32; i += 32 * NC) reinterpret_cast<uint32_t*>(tab + (i >> 5) * 256)[i & 31] = pe[(l * 256 + (i >> 5)) * 4];
      asm volatile("bar.sync 1, %0;" :: "r"(32 * NC));
      cur_l = l;
    }
    mbar_wait((uint32_t)__cvta_generic_to_shared(&full[s]), (it / STAGES) & 1);
    const uint32_t st = (uint32_t)__cvta_generic_to_shared(ring + s * SB);
    uint32_t acc16[2] = {0, 0};
#pragma unroll
    for (int j = 0; j < SB / 16 / (32 * NC); ++j) {
      const uint4 x = lds128(st + (j * 32 * NC + ct) * 16);
      const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
      uint32_t acc8 = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc8 += lds32(prmt(w4[q], slot, SEL(b)) + base);
      acc16[0] += acc8 & 0x00ff00ffu; acc16[1] += (acc8 >> 8) & 0x00ff00ffu;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive((uint32_t)__cvta_generic_to_shared(&empty[s]));
    tot[0] += acc16[0] & 0xffff; tot[2] += acc16[0] >> 16; tot[1] += acc16[1] & 0xffff; tot[3] += acc16[1] >> 16;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) { unsigned long long v = tot[i]; for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o); if (lane == 0) atomicAdd(&sums[i], v); }
}

// LDG reference (production-style inner loop)
template <int UNROLL>
__global__ void __launch_bounds__(512, 3) score_ldg_kernel(const int4* __restrict__ v, int64_t nvec_plane, int L,
                                                          const uint32_t* __restrict__ pe, unsigned long long* sums) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t slot = (uint32_t)(lane << 2);
  unsigned long long tot[4] = {0, 0, 0, 0};
  int64_t total = nvec_plane * L;
  int64_t per = (total + gridDim.x - 1) / gridDim.x;
  int64_t g0 = blockIdx.x * per, g1 = min(total, g0 + per);
  while (g0 < g1) {
    int l = (int)(g0 / nvec_plane);
    int64_t seg_end = min(g1, (int64_t)(l + 1) * nvec_plane);
    __syncthreads();
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) reinterpret_cast<uint32_t*>(sm + (i >> 5) * 256)[i & 31] = pe[(l * 256 + (i >> 5)) * 4];
    __syncthreads();
    const int4* pv = v + g0;
    const uint32_t nv = (uint32_t)(seg_end - g0);
    uint32_t i = threadIdx.x;
    for (; i + (UNROLL - 1) * blockDim.x < nv; i += UNROLL * blockDim.x) {
      int4 x[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) x[u] = ldg_stream(pv + i + u * blockDim.x);
      uint32_t acc16[2] = {0, 0};
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint32_t w4[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
        uint32_t acc8 = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc8 += lds32(prmt(w4[q], slot, SEL(b)) + base);
        acc16[0] += acc8 & 0x00ff00ffu; acc16[1] += (acc8 >> 8) & 0x00ff00ffu;
      }
      tot[0] += acc16[0] & 0xffff; tot[2] += acc16[0] >> 16; tot[1] += acc16[1] & 0xffff; tot[3] += acc16[1] >> 16;
    }
    g0 = seg_end;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) { unsigned long long s = tot[k]; for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o); if (lane == 0) atomicAdd(&sums[k], s); }
}

struct Timer { cudaEvent_t a, b; Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); } float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; } };

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int L = 58, K = 8;
  int64_t N = 10000000LL;
  int64_t plane = N * K, nvec = plane / 16;
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  uint8_t* d; CK(cudaMalloc(&d, plane * L + 4096));
  std::vector<uint32_t> cdf(257); double z = 0; std::vector<double> w(256);
  for (int r = 0; r < 256; ++r) { w[r] = pow(r + 1.0, -1.2); z += w[r]; }
  double c = 0; for (int r = 0; r < 256; ++r) { c += w[r]; cdf[r + 1] = (uint32_t)llround(c / z * (1u << 30)); }
  uint32_t* dcdf; CK(cudaMalloc(&dcdf, 257 * 4)); CK(cudaMemcpy(dcdf, cdf.data(), 257 * 4, cudaMemcpyHostToDevice));
  fill_kernel<<<nsm * 8, 256>>>(d, plane, L, dcdf, cdf[256]); CK(cudaDeviceSynchronize());
  unsigned long long* dout; CK(cudaMalloc(&dout, 4096));
  uint32_t* pe; CK(cudaMalloc(&pe, L * 256 * 16));
  std::vector<uint32_t> hpe(L * 256 * 4);
  for (size_t i = 0; i < hpe.size(); ++i) hpe[i] = ((uint32_t)i * 2654435761u) & 0x0f0f0f0fu;
  CK(cudaMemcpy(pe, hpe.data(), hpe.size() * 4, cudaMemcpyHostToDevice));
  const double bytes = (double)plane * L;
  Timer t;
  unsigned long long ref[4];
  auto bench = [&](const char* name, auto launch, bool setref) {
    CK(cudaMemset(dout, 0, 64)); launch(); CK(cudaDeviceSynchronize()); CK(cudaGetLastError());
    unsigned long long h[4]; CK(cudaMemcpy(h, dout, 32, cudaMemcpyDeviceToHost));
    if (setref) memcpy(ref, h, 32);
    bool ok = !memcmp(ref, h, 32);
    float best = 1e30f;
    for (int i = 0; i < 7; ++i) { t.start(); launch(); float ms = t.stop(); if (ms < best) best = ms; }
    printf("%-36s best %7.3f ms  %7.1f GB/s  %5.1f%% of 6548  %s\n", name, best, bytes / best / 1e6, bytes / best / 1e6 / 6548.2 * 100, ok ? "sums ok" : "SUMS DIFFER");
  };
  CK(cudaFuncSetAttribute(score_ldg_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  bench("ldg u4 (production style) c3", [&] { score_ldg_kernel<4><<<nsm * 3, 512, 65536>>>((const int4*)d, nvec, L, pe, dout); }, true);
#define WS(ST, SB, NC, CPS) { auto k = score_ws_kernel<ST, SB, NC>; int sm_ = 65536 + ST * SB; \
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_)); \
    char nm[80]; snprintf(nm, 80, "ws %dx%dK nc%d c%d", ST, SB / 1024, NC, CPS); \
    bench(nm, [&] { k<<<nsm * CPS, 32 * (NC + 1), sm_>>>(d, plane, L, pe, dout); }, false); }
  WS(4, 16384, 16, 1)
  WS(8, 16384, 16, 1)
  WS(6, 16384, 8, 1)
  WS(4, 8192, 16, 2)
  WS(6, 8192, 8, 2)
  WS(3, 8192, 16, 2)
  WS(8, 8192, 16, 1)
  printf("done\n");
  return 0;
}
