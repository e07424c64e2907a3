// Design microbenchmark (not product code): measures, on one B200, the rates that
// decide the hist/score kernel designs for layer-major u8 traces.
//   * stream: LDG.128 read of the whole trace (HBM ceiling for this access pattern)
//   * hist_rep<R>: shared-memory ATOMS histogram, R replicas per bin (bank = lane % R)
//   * score_pw<W>: replicated-table LDS gather, W u32 words (4W u8 placement lanes) per entry
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/microbench tools/microbench.cu
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

// Quick skewed filler: rank from a 256-entry integer CDF, per-layer affine permutation.
__global__ void fill_kernel(uint8_t* planes, int64_t plane_bytes, int L, const uint32_t* cdf, uint32_t total) {
  __shared__ uint32_t s_cdf[257];
  for (int i = threadIdx.x; i < 257; i += blockDim.x) s_cdf[i] = cdf[i];
  __syncthreads();
  int64_t n = plane_bytes * L / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i * 4;
    int l = (int)(b / plane_bytes);
    uint32_t out = 0;
    for (int j = 0; j < 4; ++j) {
      uint32_t r = mix32((uint32_t)(b + j) * 0x9e3779b9U ^ (uint32_t)(b >> 32)) % total;
      int lo = 0, hi = 256;
      while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (s_cdf[mid] <= r) lo = mid; else hi = mid; }
      uint32_t e = (uint32_t)(lo * 167 + l * 31) & 255u;
      out |= e << (8 * j);
    }
    reinterpret_cast<uint32_t*>(planes)[i] = out;
  }
}

__device__ __forceinline__ int4 ldg_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int UNROLL>
__global__ void __launch_bounds__(512) stream_kernel(const int4* __restrict__ v, int64_t nvec, unsigned long long* out) {
  uint32_t acc = 0;
  int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  int64_t v0 = blockIdx.x * per, v1 = min(nvec, v0 + per);
  for (int64_t i = v0 + threadIdx.x; i < v1; i += (int64_t)blockDim.x * UNROLL) {
    int4 x[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      int64_t j = i + (int64_t)u * blockDim.x;
      x[u] = j < v1 ? ldg_stream(v + j) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += x[u].x ^ x[u].y ^ x[u].z ^ x[u].w;
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

// hist: flattened [L][nvec] vector space; CTA-contiguous ranges; R replicas per bin.
template <int R, int UNROLL>
__global__ void __launch_bounds__(512) hist_kernel(const int4* __restrict__ v, int64_t nvec_plane, int L,
                                                  unsigned long long* counts) {
  extern __shared__ uint32_t h[];  // [256][R]
  const int lane = threadIdx.x & 31;
  const int rep = lane % R;
  for (int i = threadIdx.x; i < 256 * R; i += blockDim.x) h[i] = 0;
  __syncthreads();
  int64_t total = nvec_plane * L;
  int64_t per = (total + gridDim.x - 1) / gridDim.x;
  int64_t g0 = blockIdx.x * per, g1 = min(total, g0 + per);
  while (g0 < g1) {
    int l = (int)(g0 / nvec_plane);
    int64_t seg_end = min(g1, (int64_t)(l + 1) * nvec_plane);
    for (int64_t i = g0 + threadIdx.x; i < seg_end; i += (int64_t)blockDim.x * UNROLL) {
      int4 x[UNROLL];
      bool ok[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        int64_t j = i + (int64_t)u * blockDim.x;
        ok[u] = j < seg_end;
        x[u] = ok[u] ? ldg_stream(v + j) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (!ok[u]) continue;
        uint32_t w[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            uint32_t e = (w[q] >> (8 * b)) & 0xffu;
            atomicAdd(&h[e * R + rep], 1u);
          }
        }
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 256; e += blockDim.x) {
      uint32_t s = 0;
      for (int r = 0; r < R; ++r) { int rr = (r + e) % R; s += h[e * R + rr]; h[e * R + rr] = 0; }
      if (s) atomicAdd(&counts[l * 256 + e], (unsigned long long)s);
    }
    __syncthreads();
    g0 = seg_end;
  }
}

// score: table entry = W u32 words = 4W u8 placement lanes; replicas so LDS is conflict-free.
template <int W> struct VecT;
template <> struct VecT<1> { using T = uint32_t; };
template <> struct VecT<2> { using T = uint2; };
template <> struct VecT<4> { using T = uint4; };

template <int W, int UNROLL>
__global__ void __launch_bounds__(512) score_kernel(const int4* __restrict__ v, int64_t nvec_plane, int L,
                                                   const uint32_t* __restrict__ pe /*[L][256][W]*/,
                                                   unsigned long long* sums /*[4W]*/) {
  constexpr int R = 32 / W;  // replicas: 32/16/8 for LDS.32/64/128
  using T = typename VecT<W>::T;
  extern __shared__ uint4 smem_raw[];
  T* tbl = reinterpret_cast<T*>(smem_raw);  // [256][R]
  const int lane = threadIdx.x & 31;
  const T* my = tbl + (lane % R);
  uint32_t acc16[2 * W];
#pragma unroll
  for (int i = 0; i < 2 * W; ++i) acc16[i] = 0;
  unsigned long long tot[4 * W];
#pragma unroll
  for (int i = 0; i < 4 * W; ++i) tot[i] = 0;

  int64_t total = nvec_plane * L;
  int64_t per = (total + gridDim.x - 1) / gridDim.x;
  int64_t g0 = blockIdx.x * per, g1 = min(total, g0 + per);
  while (g0 < g1) {
    int l = (int)(g0 / nvec_plane);
    int64_t seg_end = min(g1, (int64_t)(l + 1) * nvec_plane);
    __syncthreads();
    for (int i = threadIdx.x; i < 256 * R; i += blockDim.x) {
      int e = i / R;
      tbl[i] = reinterpret_cast<const T*>(pe)[l * 256 + e];
    }
    __syncthreads();
    for (int64_t i = g0 + threadIdx.x; i < seg_end; i += (int64_t)blockDim.x * UNROLL) {
      int4 x[UNROLL];
      bool ok[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        int64_t j = i + (int64_t)u * blockDim.x;
        ok[u] = j < seg_end;
        x[u] = ok[u] ? ldg_stream(v + j) : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        if (!ok[u]) continue;
        uint32_t w4[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
        uint32_t acc8[W];
#pragma unroll
        for (int k = 0; k < W; ++k) acc8[k] = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            uint32_t e = (w4[q] >> (8 * b)) & 0xffu;
            T t = my[e * R];
            if constexpr (W == 1) acc8[0] += t;
            else if constexpr (W == 2) { acc8[0] += t.x; acc8[1] += t.y; }
            else { acc8[0] += t.x; acc8[1] += t.y; acc8[2] += t.z; acc8[3] += t.w; }
          }
        }
#pragma unroll
        for (int k = 0; k < W; ++k) {
          acc16[2 * k] += acc8[k] & 0x00ff00ffu;
          acc16[2 * k + 1] += (acc8[k] >> 8) & 0x00ff00ffu;
        }
      }
      // widen u16 -> u64 once per outer iteration (<= UNROLL*16*15 per lane)
#pragma unroll
      for (int k = 0; k < 2 * W; ++k) {
        tot[2 * k] += acc16[k] & 0xffffu;
        tot[2 * k + 1] += acc16[k] >> 16;
        acc16[k] = 0;
      }
    }
    g0 = seg_end;
  }
#pragma unroll
  for (int i = 0; i < 4 * W; ++i) {
    unsigned long long s = tot[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) atomicAdd(&sums[i], s);
  }
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

int main(int argc, char** argv) {
  const int L = 58, K = 8;
  int64_t N = argc > 1 ? atoll(argv[1]) : 10000000LL;
  double s = argc > 2 ? atof(argv[2]) : 1.2;
  int64_t plane = N * K;  // multiple of 16 for K=8
  int64_t nvec = plane / 16;
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  printf("N=%lld L=%d K=%d zipf=%.2f bytes=%.3f GB sms=%d\n", (long long)N, L, K, s, plane * L / 1e9, nsm);
  uint8_t* d; CK(cudaMalloc(&d, plane * L));
  std::vector<uint32_t> cdf(257); double z = 0; std::vector<double> w(256);
  for (int r = 0; r < 256; ++r) { w[r] = pow(r + 1.0, -s); z += w[r]; }
  double c = 0; cdf[0] = 0; for (int r = 0; r < 256; ++r) { c += w[r]; cdf[r + 1] = (uint32_t)llround(c / z * (1u << 30)); }
  uint32_t* dcdf; CK(cudaMalloc(&dcdf, 257 * 4)); CK(cudaMemcpy(dcdf, cdf.data(), 257 * 4, cudaMemcpyHostToDevice));
  fill_kernel<<<nsm * 8, 256>>>(d, plane, L, dcdf, cdf[256]);
  CK(cudaDeviceSynchronize());
  unsigned long long* dout; CK(cudaMalloc(&dout, 1 << 20));
  uint32_t* pe; CK(cudaMalloc(&pe, L * 256 * 4 * 4));
  std::vector<uint32_t> hpe(L * 256 * 4);
  for (size_t i = 0; i < hpe.size(); ++i) hpe[i] = ((uint32_t)i * 2654435761u) & 0x0f0f0f0fu;  // lanes <= 15
  CK(cudaMemcpy(pe, hpe.data(), hpe.size() * 4, cudaMemcpyHostToDevice));
  const double bytes = (double)plane * L;
  Timer t;
  auto report = [&](const char* name, float ms) {
    printf("%-28s %8.3f ms  %8.1f GB/s  %6.1f%% of 6548\n", name, ms, bytes / ms / 1e6, bytes / ms / 1e6 / 6548.2 * 100);
  };
  auto bench = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int i = 0; i < 5; ++i) { t.start(); launch(); float ms = t.stop(); if (ms < best) best = ms; }
    CK(cudaGetLastError());
    report(name, best);
  };
  for (int thr : {256, 512}) {
    for (int cpsm : {2, 4, 8}) {
      if (thr * cpsm > 2048) continue;
      int grid = nsm * cpsm;
      char nm[64];
      snprintf(nm, 64, "stream u4 t%d c%d", thr, cpsm);
      bench(nm, [&] { stream_kernel<4><<<grid, thr>>>((const int4*)d, nvec * L, dout); });
      snprintf(nm, 64, "hist rep32 u4 t%d c%d", thr, cpsm);
      CK(cudaFuncSetAttribute(hist_kernel<32, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
      bench(nm, [&] { hist_kernel<32, 4><<<grid, thr, 256 * 32 * 4>>>((const int4*)d, nvec, L, dout); });
      snprintf(nm, 64, "hist rep8 u4 t%d c%d", thr, cpsm);
      bench(nm, [&] { hist_kernel<8, 4><<<grid, thr, 256 * 8 * 4>>>((const int4*)d, nvec, L, dout); });
      snprintf(nm, 64, "hist rep1 u4 t%d c%d", thr, cpsm);
      bench(nm, [&] { hist_kernel<1, 4><<<grid, thr, 256 * 4>>>((const int4*)d, nvec, L, dout); });
      snprintf(nm, 64, "score W1(P4) u4 t%d c%d", thr, cpsm);
      CK(cudaFuncSetAttribute(score_kernel<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
      bench(nm, [&] { score_kernel<1, 4><<<grid, thr, 32768>>>((const int4*)d, nvec, L, pe, dout); });
      snprintf(nm, 64, "score W2(P8) u4 t%d c%d", thr, cpsm);
      CK(cudaFuncSetAttribute(score_kernel<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
      bench(nm, [&] { score_kernel<2, 4><<<grid, thr, 32768>>>((const int4*)d, nvec, L, pe, dout); });
      snprintf(nm, 64, "score W4(P16) u4 t%d c%d", thr, cpsm);
      CK(cudaFuncSetAttribute(score_kernel<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
      bench(nm, [&] { score_kernel<4, 4><<<grid, thr, 32768>>>((const int4*)d, nvec, L, pe, dout); });
    }
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
