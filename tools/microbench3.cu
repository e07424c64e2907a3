// Design microbenchmark #3 (not product code): read-ceiling variants and PRMT-addressed gathers.
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

template <int UNROLL, bool NA>
__global__ void __launch_bounds__(1024) stream_kernel(const int4* __restrict__ v, int64_t nvec, unsigned long long* out) {
  uint32_t acc = 0;
  int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  int64_t v0 = blockIdx.x * per, v1 = min(nvec, v0 + per);
  for (int64_t i = v0 + threadIdx.x; i < v1; i += (int64_t)blockDim.x * UNROLL) {
    int4 x[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) { int64_t j = i + (int64_t)u * blockDim.x;
      x[u] = j < v1 ? (NA ? ldg_stream(v + j) : ldg_plain(v + j)) : make_int4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += x[u].x ^ x[u].y ^ x[u].z ^ x[u].w;
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}
// grid-stride interleaved (all CTAs sweep together)
template <int UNROLL>
__global__ void __launch_bounds__(1024) stream_gs_kernel(const int4* __restrict__ v, int64_t nvec, unsigned long long* out) {
  uint32_t acc = 0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x * UNROLL + threadIdx.x; i < nvec; i += stride * UNROLL) {
    int4 x[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) { int64_t j = i + (int64_t)u * blockDim.x; x[u] = j < nvec ? ldg_stream(v + j) : make_int4(0,0,0,0); }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += x[u].x ^ x[u].y ^ x[u].z ^ x[u].w;
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}
// bulk-copy (TMA 1D) streaming: one elected thread issues cp.async.bulk into a STAGES ring.
template <int STAGES, int STAGE_BYTES>
__global__ void __launch_bounds__(256) stream_bulk_kernel(const uint8_t* __restrict__ src, int64_t nbytes, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  int64_t per = ((nbytes / STAGE_BYTES + gridDim.x - 1) / gridDim.x) * STAGE_BYTES;
  int64_t b0 = blockIdx.x * per, b1 = min(nbytes, b0 + per);
  int nst = b1 > b0 ? (int)((b1 - b0 + STAGE_BYTES - 1) / STAGE_BYTES) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&full[s])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&empty[s])), "r"(blockDim.x / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int it) {
    int s = it % STAGES;
    int64_t off = b0 + (int64_t)it * STAGE_BYTES;
    uint32_t bytes = (uint32_t)min((int64_t)STAGE_BYTES, b1 - off);
    uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(fb), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((uint32_t)__cvta_generic_to_shared(sm + s * STAGE_BYTES)), "l"(src + off), "r"(bytes), "r"(fb) : "memory");
  };
  if (threadIdx.x == 0) for (int it = 0; it < min(nst, STAGES); ++it) issue(it);
  uint32_t acc = 0;
  for (int it = 0; it < nst; ++it) {
    int s = it % STAGES; uint32_t ph = (it / STAGES) & 1;
    uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(fb), "r"(ph) : "memory");
    const uint4* st = reinterpret_cast<const uint4*>(sm + s * STAGE_BYTES);
    for (int i = threadIdx.x; i < STAGE_BYTES / 16; i += blockDim.x) { uint4 x = st[i]; acc += x.x ^ x.y ^ x.z ^ x.w; }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&empty[s])) : "memory");
    if (threadIdx.x == 0 && it + STAGES < nst) {
      uint32_t eb = (uint32_t)__cvta_generic_to_shared(&empty[s]);
      asm volatile("{ .reg .pred p; W2: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W2; }" :: "r"(eb), "r"(ph) : "memory");
      issue(it + STAGES);
    }
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

// PRMT-addressed gathers. Row stride 256 B per expert; the lane slot is (lane<<2) (W=1) or ((lane&7)<<4) (W=4).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) { uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel)); return r; }
__device__ __forceinline__ uint32_t lds32(uint32_t a) { uint32_t r; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a)); return r; }
__device__ __forceinline__ uint4 lds128(uint32_t a) { uint4 r; asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a)); return r; }
__device__ __forceinline__ void atoms_inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" :: "r"(a)); }
// sel for byte b of a -> result byte1, result byte0 = b.byte0 (lane slot), bytes 2,3 = b.byte1 (zero)
#define SEL(b) (0x5504u | ((b) << 4))


// Fused variants. Row e = 256 B; 32 lane slots of 8 B: low u32 = 4 placement bytes, high u32 = lane count.
__device__ __forceinline__ unsigned long long atoms_add64_ret(uint32_t a, unsigned long long v) {
  unsigned long long r; asm volatile("atom.shared.add.u64 %0, [%1], %2;" : "=l"(r) : "r"(a), "l"(v)); return r; }
__device__ __forceinline__ uint32_t atoms_add32_ret(uint32_t a, uint32_t v) {
  uint32_t r; asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v)); return r; }

template <int MODE, int UNROLL>   // 0: LDS.32 + RED.32 (+128)   1: ATOM.64 ret   2: LDS only   3: RED only
__global__ void __launch_bounds__(512) fused_kernel(const int4* __restrict__ v, int64_t nvec_plane, int L,
                                                   const uint32_t* __restrict__ pe, unsigned long long* sums,
                                                   unsigned long long* counts) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t slot = MODE == 1 ? (uint32_t)(lane << 3) : (uint32_t)(lane << 2);
  uint32_t acc16[2] = {0, 0};
  unsigned long long tot[4] = {0, 0, 0, 0};
  int64_t total = nvec_plane * L;
  int64_t per = (total + gridDim.x - 1) / gridDim.x;
  int64_t g0 = blockIdx.x * per, g1 = min(total, g0 + per);
  while (g0 < g1) {
    int l = (int)(g0 / nvec_plane);
    int64_t seg_end = min(g1, (int64_t)(l + 1) * nvec_plane);
    __syncthreads();
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
      int e = i >> 5, r = i & 31;
      uint32_t* row = reinterpret_cast<uint32_t*>(sm + e * 256);
      uint32_t val = pe[(l * 256 + e) * 4];
      if (MODE == 1) { row[2 * r] = val; row[2 * r + 1] = 0; }
      else { row[r] = val; row[32 + r] = 0; }
    }
    __syncthreads();
    for (int64_t i = g0 + threadIdx.x; i < seg_end; i += (int64_t)blockDim.x * UNROLL) {
      int4 x[UNROLL]; bool ok[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) { int64_t j = i + (int64_t)u * blockDim.x; ok[u] = j < seg_end; x[u] = ok[u] ? ldg_stream(v + j) : make_int4(0,0,0,0); }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (!ok[u]) continue;
        uint32_t w4[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
        uint32_t acc8 = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            uint32_t a = prmt(w4[q], slot, SEL(b)) + base;
            if (MODE == 0) { acc8 += lds32(a); atoms_inc(a + 128); }
            else if (MODE == 1) { acc8 += (uint32_t)atoms_add64_ret(a, 1ull << 32); }
            else if (MODE == 2) { acc8 += lds32(a); }
            else { atoms_inc(a + 128); }
          }
        }
        acc16[0] += acc8 & 0x00ff00ffu; acc16[1] += (acc8 >> 8) & 0x00ff00ffu;
      }
      tot[0] += acc16[0] & 0xffff; tot[2] += acc16[0] >> 16; tot[1] += acc16[1] & 0xffff; tot[3] += acc16[1] >> 16;
      acc16[0] = acc16[1] = 0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 256; e += blockDim.x) {
      const uint32_t* row = reinterpret_cast<const uint32_t*>(sm + e * 256);
      unsigned long long s = 0;
      for (int r = 0; r < 32; ++r) s += MODE == 1 ? row[2 * ((r + e) & 31) + 1] : row[32 + ((r + e) & 31)];
      if (s) atomicAdd(&counts[l * 256 + e], s);
    }
    g0 = seg_end;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) { unsigned long long s = tot[i]; for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o); if (lane == 0) atomicAdd(&sums[i], s); }
}

// TMA-staged score: bulk copies of the CTA's byte range into a STAGES ring; LDS.128 of the staged trace.
template <int STAGES, int STAGE_BYTES>
__global__ void __launch_bounds__(512) score_bulk_kernel(const uint8_t* __restrict__ src, int64_t plane_bytes, int L,
                                                         const uint32_t* __restrict__ pe, unsigned long long* sums) {
  extern __shared__ __align__(128) uint8_t sm[];          // [0,64K): table rows; then ring
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  uint8_t* ring = sm + 65536;
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t slot = (uint32_t)(lane << 2);
  int64_t nbytes = plane_bytes * L;
  int64_t per = ((nbytes / STAGE_BYTES + gridDim.x - 1) / gridDim.x) * STAGE_BYTES;
  int64_t b0 = blockIdx.x * per, b1 = min(nbytes, b0 + per);
  int nst = b1 > b0 ? (int)((b1 - b0 + STAGE_BYTES - 1) / STAGE_BYTES) : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&full[s])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&empty[s])), "r"(blockDim.x / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int it) {
    int s = it % STAGES; int64_t off = b0 + (int64_t)it * STAGE_BYTES;
    uint32_t bytes = (uint32_t)min((int64_t)STAGE_BYTES, b1 - off);
    uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(fb), "r"(bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((uint32_t)__cvta_generic_to_shared(ring + s * STAGE_BYTES)), "l"(src + off), "r"(bytes), "r"(fb) : "memory");
  };
  if (threadIdx.x == 0) for (int it = 0; it < min(nst, STAGES); ++it) issue(it);
  int cur_l = -1;
  unsigned long long tot[4] = {0, 0, 0, 0};
  for (int it = 0; it < nst; ++it) {
    int64_t off = b0 + (int64_t)it * STAGE_BYTES;
    int l = (int)(off / plane_bytes);   // STAGE_BYTES divides plane_bytes in this bench
    if (l != cur_l) {
      __syncthreads();
      for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) reinterpret_cast<uint32_t*>(sm + (i >> 5) * 256)[i & 31] = pe[(l * 256 + (i >> 5)) * 4];
      __syncthreads();
      cur_l = l;
    }
    int s = it % STAGES; uint32_t ph = (it / STAGES) & 1;
    uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" :: "r"(fb), "r"(ph) : "memory");
    const uint32_t st = (uint32_t)__cvta_generic_to_shared(ring + s * STAGE_BYTES);
    uint32_t acc16[2] = {0, 0};
    for (int i = threadIdx.x; i < STAGE_BYTES / 16; i += blockDim.x) {
      uint4 x = lds128(st + i * 16);
      uint32_t w4[4] = {x.x, x.y, x.z, x.w};
      uint32_t acc8 = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc8 += lds32(prmt(w4[q], slot, SEL(b)) + base);
      acc16[0] += acc8 & 0x00ff00ffu; acc16[1] += (acc8 >> 8) & 0x00ff00ffu;
    }
    tot[0] += acc16[0] & 0xffff; tot[2] += acc16[0] >> 16; tot[1] += acc16[1] & 0xffff; tot[3] += acc16[1] >> 16;
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&empty[s])) : "memory");
    if (threadIdx.x == 0 && it + STAGES < nst) {
      uint32_t eb = (uint32_t)__cvta_generic_to_shared(&empty[s]);
      asm volatile("{ .reg .pred p; W2: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W2; }" :: "r"(eb), "r"(ph) : "memory");
      issue(it + STAGES);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) { unsigned long long s = tot[i]; for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o); if (lane == 0) atomicAdd(&sums[i], s); }
}

struct Timer { cudaEvent_t a, b; Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); } float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; } };

int main(int argc, char** argv) {
  const int L = 58, K = 8;
  int64_t N = argc > 1 ? atoll(argv[1]) : 10000000LL;
  double s = argc > 2 ? atof(argv[2]) : 1.2;
  int64_t plane = N * K, nvec = plane / 16;
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  printf("N=%lld L=%d K=%d zipf=%.2f bytes=%.3f GB\n", (long long)N, L, K, s, plane * L / 1e9);
  uint8_t* d; CK(cudaMalloc(&d, plane * L + 4096));
  std::vector<uint32_t> cdf(257); double z = 0; std::vector<double> w(256);
  for (int r = 0; r < 256; ++r) { w[r] = pow(r + 1.0, -s); z += w[r]; }
  double c = 0; for (int r = 0; r < 256; ++r) { c += w[r]; cdf[r + 1] = (uint32_t)llround(c / z * (1u << 30)); }
  uint32_t* dcdf; CK(cudaMalloc(&dcdf, 257 * 4)); CK(cudaMemcpy(dcdf, cdf.data(), 257 * 4, cudaMemcpyHostToDevice));
  fill_kernel<<<nsm * 8, 256>>>(d, plane, L, dcdf, cdf[256]); CK(cudaDeviceSynchronize());
  unsigned long long* dout; CK(cudaMalloc(&dout, 1 << 20));
  uint32_t* pe; CK(cudaMalloc(&pe, L * 256 * 4 * 4));
  std::vector<uint32_t> hpe(L * 256 * 4);
  for (size_t i = 0; i < hpe.size(); ++i) hpe[i] = ((uint32_t)i * 2654435761u) & 0x0f0f0f0fu;
  CK(cudaMemcpy(pe, hpe.data(), hpe.size() * 4, cudaMemcpyHostToDevice));
  const double bytes = (double)plane * L;
  Timer t;
  auto bench = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize()); CK(cudaGetLastError());
    float best = 1e30f, sum = 0;
    for (int i = 0; i < 7; ++i) { t.start(); launch(); float ms = t.stop(); sum += ms; if (ms < best) best = ms; }
    CK(cudaGetLastError());
    printf("%-34s best %7.3f ms avg %7.3f  %7.1f GB/s  %5.1f%% of 6548\n", name, best, sum / 7, bytes / best / 1e6, bytes / best / 1e6 / 6548.2 * 100);
  };
  char nm[80];
  const int SM = 65536;
#define SETUP(K_) CK(cudaFuncSetAttribute(K_, cudaFuncAttributeMaxDynamicSharedMemorySize, SM))
  SETUP((fused_kernel<0, 4>)); SETUP((fused_kernel<1, 4>)); SETUP((fused_kernel<2, 4>)); SETUP((fused_kernel<3, 4>));
  for (int cpsm : {2, 3}) {
    int grid = nsm * cpsm;
    snprintf(nm, 80, "fused LDS+RED c%d", cpsm); bench(nm, [&] { fused_kernel<0, 4><<<grid, 512, SM>>>((const int4*)d, nvec, L, pe, dout, dout + 64); });
    snprintf(nm, 80, "fused ATOM64ret c%d", cpsm); bench(nm, [&] { fused_kernel<1, 4><<<grid, 512, SM>>>((const int4*)d, nvec, L, pe, dout, dout + 64); });
    snprintf(nm, 80, "LDS only c%d", cpsm); bench(nm, [&] { fused_kernel<2, 4><<<grid, 512, SM>>>((const int4*)d, nvec, L, pe, dout, dout + 64); });
    snprintf(nm, 80, "RED only c%d", cpsm); bench(nm, [&] { fused_kernel<3, 4><<<grid, 512, SM>>>((const int4*)d, nvec, L, pe, dout, dout + 64); });
  }
  const int SMB = 65536 + 4 * 16384;
  CK(cudaFuncSetAttribute(score_bulk_kernel<4, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMB));
  CK(cudaFuncSetAttribute(score_bulk_kernel<2, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2 * 16384));
  CK(cudaFuncSetAttribute(score_bulk_kernel<3, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 3 * 8192));
  for (int cpsm : {1, 2}) {
    snprintf(nm, 80, "score bulk 4x16K c%d", cpsm); bench(nm, [&] { score_bulk_kernel<4, 16384><<<nsm * cpsm, 512, SMB>>>(d, plane, L, pe, dout); });
    snprintf(nm, 80, "score bulk 2x16K c%d", cpsm); bench(nm, [&] { score_bulk_kernel<2, 16384><<<nsm * cpsm, 512, 65536 + 2 * 16384>>>(d, plane, L, pe, dout); });
    snprintf(nm, 80, "score bulk 3x8K c%d", cpsm); bench(nm, [&] { score_bulk_kernel<3, 8192><<<nsm * cpsm, 512, 65536 + 3 * 8192>>>(d, plane, L, pe, dout); });
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
