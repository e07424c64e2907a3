// Design microbenchmark #8 (not product code): does counting a piece's hottest experts in
// registers (SIMD byte compares + popc) and predicating their lanes off the ATOMS make the
// replicated-bin histogram cheaper?  The question is whether an ATOMS instruction with fewer
// active lanes costs fewer L1TEX wavefronts.  Trace: layer-major u8 planes, K = 8 distinct picks
// per (token, layer) drawn without replacement from Zipf(s) (rejection = sequential draws).
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
__host__ __device__ __forceinline__ uint32_t expert_of(int rank, int l) { return (uint32_t)(rank * 167 + l * 31) & 255u; }

// one thread per (token, layer) record of 8 distinct picks
__global__ void fill_kernel(uint8_t* planes, int64_t N, int L, const uint32_t* cdf, uint32_t total) {
  __shared__ uint32_t s_cdf[257];
  for (int i = threadIdx.x; i < 257; i += blockDim.x) s_cdf[i] = cdf[i];
  __syncthreads();
  const int64_t n = N * L;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / N);
    const int64_t t = i - (int64_t)l * N;
    uint32_t picked[8];
    const uint32_t key = mix32((uint32_t)i * 0x9e3779b9U ^ mix32((uint32_t)(i >> 32) + 0x85ebca6bU));
    uint32_t draw = 0;
    for (int k = 0; k < 8; ++k) {
      uint32_t e;
      for (;;) {
        const uint32_t h = mix32(key ^ mix32(++draw * 0x6d2b79f5U));
        const uint32_t r = h % total;
        int lo = 0, hi = 256;
        while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (s_cdf[mid] <= r) lo = mid; else hi = mid; }
        e = expert_of(lo, l);
        bool dup = false;
        for (int j = 0; j < k; ++j) dup |= picked[j] == e;
        if (!dup) break;
      }
      picked[k] = e;
    }
    uint32_t lo4 = picked[0] | picked[1] << 8 | picked[2] << 16 | picked[3] << 24;
    uint32_t hi4 = picked[4] | picked[5] << 8 | picked[6] << 16 | picked[7] << 24;
    reinterpret_cast<uint2*>(planes + (int64_t)l * N * 8)[t] = make_uint2(lo4, hi4);
  }
}
__device__ __forceinline__ int4 ldg_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) { uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel)); return r; }
__device__ __forceinline__ void atoms_inc(uint32_t a) { asm volatile("red.shared.add.u32 [%0], 1;" :: "r"(a)); }
__device__ __forceinline__ void atoms_inc_if(uint32_t a, bool p) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %1, 0; @q red.shared.add.u32 [%0], 1; }" :: "r"(a), "r"((uint32_t)p));
}
#define SEL(b) (0x5504u | ((b) << 4))

// MODE 0: production (every byte one ATOMS)
// MODE 1: H hot experts counted in registers (vcmpeq4 + popc), their lanes predicated off the ATOMS
// MODE 2: the same register counting, ATOMS unconditional (ALU overhead alone; counts are wrong)
template <int MODE, int H, int UNROLL>
__global__ void __launch_bounds__(512, 3) hist_variant(const int4* __restrict__ v, int64_t nvec_plane, int L,
                                                       unsigned long long* counts) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint32_t* h = reinterpret_cast<uint32_t*>(sm);
  const int lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + 128;
  const uint32_t slot = (uint32_t)(lane << 2);
  int64_t total = nvec_plane * L;
  int64_t per = (total + gridDim.x - 1) / gridDim.x;
  int64_t g0 = blockIdx.x * per, g1 = min(total, g0 + per);
  while (g0 < g1) {
    const int l = (int)(g0 / nvec_plane);
    const int64_t seg_end = min(g1, (int64_t)(l + 1) * nvec_plane);
    __syncthreads();
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) h[i] = 0;
    __syncthreads();
    uint32_t hp[H > 0 ? H : 1], hc[H > 0 ? H : 1];
#pragma unroll
    for (int j = 0; j < (H > 0 ? H : 1); ++j) { hp[j] = expert_of(j, l) * 0x01010101u; hc[j] = 0; }
    int64_t i = g0 + threadIdx.x;
    for (; i + (UNROLL - 1) * (int64_t)blockDim.x < seg_end; i += (int64_t)blockDim.x * UNROLL) {
      int4 x[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) x[u] = ldg_stream(v + i + (int64_t)u * blockDim.x);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint32_t w4[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t any = 0;
          if constexpr (MODE != 0) {
#pragma unroll
            for (int j = 0; j < H; ++j) {
              const uint32_t m = __vcmpeq4(w4[q], hp[j]);
              hc[j] += __popc(m);
              any |= m;
            }
          }
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const uint32_t a = prmt(w4[q], slot, SEL(b)) + base;
            if constexpr (MODE == 1) atoms_inc_if(a, ((any >> (8 * b)) & 1u) == 0);
            else atoms_inc(a);
          }
        }
      }
    }
    for (; i < seg_end; i += blockDim.x) {  // tail: production path
      const int4 x = ldg_stream(v + i);
      const uint32_t w4[4] = {(uint32_t)x.x, (uint32_t)x.y, (uint32_t)x.z, (uint32_t)x.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b) atoms_inc(prmt(w4[q], slot, SEL(b)) + base);
    }
    if constexpr (MODE == 1) {
#pragma unroll
      for (int j = 0; j < H; ++j)
        if (hc[j]) asm volatile("red.shared.add.u32 [%0], %1;" :: "r"(base + (((hp[j] & 255u) << 8) | slot)), "r"(hc[j] >> 3));
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 256; e += blockDim.x) {
      unsigned long long s = 0;
      for (int r = 0; r < 32; ++r) s += h[e * 64 + 32 + ((r + e) & 31)];
      if (s) atomicAdd(&counts[l * 256 + e], s);
    }
    g0 = seg_end;
  }
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
  unsigned long long* dout; CK(cudaMalloc(&dout, 256 * L * 8));
  uint32_t* dcdf; CK(cudaMalloc(&dcdf, 257 * 4));
  const double bytes = (double)plane * L;
  Timer t;
  std::vector<unsigned long long> ref(256 * L), got(256 * L);
  for (double s : {1.2, 0.0, 2.0}) {
    std::vector<uint32_t> cdf(257); double z = 0; std::vector<double> w(256);
    for (int r = 0; r < 256; ++r) { w[r] = pow(r + 1.0, -s); z += w[r]; }
    double c = 0; for (int r = 0; r < 256; ++r) { c += w[r]; cdf[r + 1] = (uint32_t)llround(c / z * (1u << 30)); }
    CK(cudaMemcpy(dcdf, cdf.data(), 257 * 4, cudaMemcpyHostToDevice));
    fill_kernel<<<nsm * 8, 256>>>(d, N, L, dcdf, cdf[256]); CK(cudaDeviceSynchronize());
    const int SM = 65536;
    auto bench = [&](const char* name, auto kern, int check) {  // 0 = set reference, 1 = compare, 2 = neither
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
      CK(cudaMemset(dout, 0, 256 * L * 8));
      kern<<<nsm * 3, 512, SM>>>((const int4*)d, nvec, L, dout);
      CK(cudaDeviceSynchronize()); CK(cudaGetLastError());
      CK(cudaMemcpy(got.data(), dout, 256 * L * 8, cudaMemcpyDeviceToHost));
      const char* ok = "";
      if (check == 0) { ref = got; ok = "(reference)"; }
      else if (check == 2) ok = "(timing only)";
      else ok = (got == ref) ? "counts identical" : "COUNTS DIFFER";
      unsigned long long top = 0;
      for (int l = 0; l < L; ++l) top += got[l * 256 + expert_of(0, l)];
      float best = 1e30f;
      for (int i = 0; i < 5; ++i) { t.start(); kern<<<nsm * 3, 512, SM>>>((const int4*)d, nvec, L, dout); float ms = t.stop(); if (ms < best) best = ms; }
      printf("zipf %.1f %-40s best %7.3f ms  %7.1f GB/s  %5.1f%% of 6548  top1 share %.3f  %s\n", s, name, best,
             bytes / best / 1e6, bytes / best / 1e6 / 6548.2 * 100, (double)top / bytes, ok);
    };
    bench("production (all ATOMS)", hist_variant<0, 0, 16>, 0);
    bench("hot 1 in registers, lanes predicated off", hist_variant<1, 1, 16>, 1);
    bench("hot 2 in registers, lanes predicated off", hist_variant<1, 2, 16>, 1);
    bench("hot 4 in registers, lanes predicated off", hist_variant<1, 4, 16>, 1);
    bench("hot 8 in registers, lanes predicated off", hist_variant<1, 8, 16>, 1);
    bench("production unroll 8", hist_variant<0, 0, 8>, 1);
    bench("hot 1 unroll 8", hist_variant<1, 1, 8>, 1);
    bench("hot 2 unroll 8", hist_variant<1, 2, 8>, 1);
    bench("hot 4 unroll 8", hist_variant<1, 4, 8>, 1);
    bench("hot 2 unroll 4", hist_variant<1, 2, 4>, 1);
    bench("hot 4 unroll 4", hist_variant<1, 4, 4>, 1);
    bench("hot 4 ALU only (ATOMS unconditional)", hist_variant<2, 4, 16>, 2);
  }
  printf("done\n");
  return 0;
}
