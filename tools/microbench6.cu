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



// Histogram variants (one byte = one increment), all over layer-major u8 planes:
//  0: 32 lane replicas, PRMT address, RED.ADD (production design)
//  1: __match_any_sync warp aggregation per byte position, leader adds popc(mask) to a single
//     (non-replicated) bin: one ATOMS per distinct expert per warp instruction
//  2: match_any aggregation into 32-replica bins (leader lane's replica)
template <int MODE, int UNROLL>
__global__ void __launch_bounds__(512) hist_variant(const int4* __restrict__ v, int64_t nvec_plane, int L,
                                                   unsigned long long* counts, uint32_t one) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint32_t* h = reinterpret_cast<uint32_t*>(sm);
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const uint32_t slot = (uint32_t)(lane << 2);
  uint32_t sink = 0;
  int64_t total = nvec_plane * L;
  int64_t per = (total + gridDim.x - 1) / gridDim.x;
  int64_t g0 = blockIdx.x * per, g1 = min(total, g0 + per);
  while (g0 < g1) {
    int l = (int)(g0 / nvec_plane);
    int64_t seg_end = min(g1, (int64_t)(l + 1) * nvec_plane);
    __syncthreads();
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) h[i] = 0;
    __syncthreads();
    // warp-uniform loop: every lane of a warp runs the same iterations (match_any needs all 32)
    for (int64_t iw = g0 + (threadIdx.x & ~31); iw < seg_end; iw += (int64_t)blockDim.x * UNROLL) {
      const int64_t i = iw + lane;
      int4 x[UNROLL]; bool ok[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) { int64_t j = i + (int64_t)u * blockDim.x; ok[u] = j < seg_end; x[u] = ok[u] ? ldg_stream(v + j) : make_int4(0,0,0,0); }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        uint32_t w4[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            uint32_t e = (w4[q] >> (8 * b)) & 0xffu;
            if (MODE == 0) {
              if (ok[u]) atoms_inc(prmt(w4[q], slot, SEL(b)) + base);
            } else if (MODE == 3) {
              if (ok[u]) asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(prmt(w4[q], slot, SEL(b)) + base), "r"(one));
            } else if (MODE == 4) {
              uint32_t old;
              if (ok[u]) { asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(prmt(w4[q], slot, SEL(b)) + base), "r"(one)); sink ^= old; }
            } else {
              uint32_t key = ok[u] ? e : 0x100u;   // all lanes take part in the match
              uint32_t m = __match_any_sync(0xffffffffu, key);
              int leader = __ffs(m) - 1;
              if (lane == leader && key < 0x100u) {
                uint32_t a = MODE == 1 ? base + e * 4 : base + ((e << 8) | slot);
                asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(a), "r"((uint32_t)__popc(m)));
              }
            }
          }
        }
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 256; e += blockDim.x) {
      unsigned long long s = 0;
      if (MODE == 1) s = h[e];
      else for (int r = 0; r < 32; ++r) s += h[e * 64 + ((r + e) & 31)];
      if (s) atomicAdd(&counts[l * 256 + e], s);
    }
    g0 = seg_end;
  }
  if (sink == 0x12345678u) counts[0] = 0;
}

struct Timer { cudaEvent_t a, b; Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); } float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; } };

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int L = 58, K = 8;
  int64_t N = argc > 1 ? atoll(argv[1]) : 10000000LL;
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  int64_t plane = N * K, nvec = plane / 16;
  uint8_t* d; CK(cudaMalloc(&d, plane * L + 4096));
  unsigned long long* dout; CK(cudaMalloc(&dout, 1 << 20));
  uint32_t* dcdf; CK(cudaMalloc(&dcdf, 257 * 4));
  const double bytes = (double)plane * L;
  Timer t;
  for (double s : {1.2}) {
    std::vector<uint32_t> cdf(257); double z = 0; std::vector<double> w(256);
    for (int r = 0; r < 256; ++r) { w[r] = pow(r + 1.0, -s); z += w[r]; }
    double c = 0; for (int r = 0; r < 256; ++r) { c += w[r]; cdf[r + 1] = (uint32_t)llround(c / z * (1u << 30)); }
    CK(cudaMemcpy(dcdf, cdf.data(), 257 * 4, cudaMemcpyHostToDevice));
    fill_kernel<<<nsm * 8, 256>>>(d, plane, L, dcdf, cdf[256]); CK(cudaDeviceSynchronize());
    auto bench = [&](const char* name, auto launch) {
      launch();
      CK(cudaDeviceSynchronize()); CK(cudaGetLastError());
      float best = 1e30f;
      for (int i = 0; i < 3; ++i) { t.start(); launch(); float ms = t.stop(); if (ms < best) best = ms; }
      printf("zipf %.1f %-34s best %7.3f ms  %7.1f GB/s  %5.1f%% of 6548\n", s, name, best, bytes / best / 1e6, bytes / best / 1e6 / 6548.2 * 100);
    };
    const int SM = 65536;
    CK(cudaFuncSetAttribute(hist_variant<0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
    CK(cudaFuncSetAttribute(hist_variant<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
    CK(cudaFuncSetAttribute(hist_variant<3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
    CK(cudaFuncSetAttribute(hist_variant<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
    bench("replicated RED +1 (POPC.INC)", [&] { hist_variant<0, 4><<<nsm * 3, 512, SM>>>((const int4*)d, nvec, L, dout, 1u); });
    bench("replicated RED +r (ATOMS.ADD)", [&] { hist_variant<3, 4><<<nsm * 3, 512, SM>>>((const int4*)d, nvec, L, dout, 1u); });
    bench("replicated ATOM ret +r", [&] { hist_variant<4, 4><<<nsm * 3, 512, SM>>>((const int4*)d, nvec, L, dout, 1u); });
  }
  printf("done\n");
  return 0;
}
