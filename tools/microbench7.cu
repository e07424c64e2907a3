// Design microbenchmark #7 (not product code): replicated shared-memory histogram with
// red.shared (ATOMS) vs red.async (REDAS, mbarrier complete_tx accounting), same layout as the
// product (256 rows x 256 B, 32 u32 replicas of bin e at +128 + lane*4), 16 vectors per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench7 tools/microbench7.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s)); return r;
}
__device__ __forceinline__ int4 ldg_stream(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <int MODE>  // 0: red.shared (ATOMS), 1: red.async (REDAS)
__device__ __forceinline__ void inc(uint32_t a, uint32_t bar) {
  if (MODE == 0) asm volatile("red.shared.add.u32 [%0], 1;" :: "r"(a) : "memory");
  else asm volatile("red.async.relaxed.cluster.shared::cluster.mbarrier::complete_tx::bytes.add.u32 [%0], 1, [%1];"
                    :: "r"(a), "r"(bar) : "memory");
}

template <int MODE, int UNROLL>
__global__ void __cluster_dims__(1, 1, 1) __launch_bounds__(512, 3) hist(const int4* __restrict__ v, int64_t nvec, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[16];
  uint32_t* smw = (uint32_t*)sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) smw[i] = 0;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[warp]);
  if (MODE == 1 && lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar));
  __syncthreads();
  const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(sm) + 128, hslot = lane << 2;
  const int64_t per = (nvec + gridDim.x - 1) / gridDim.x;
  const int64_t a = blockIdx.x * per, b = min(nvec, a + per);
  const uint32_t T = blockDim.x;
  for (int64_t i = a + threadIdx.x; i + (UNROLL - 1) * T < b; i += UNROLL * T) {
    if (MODE == 1 && lane == 0)  // this warp's batch: 32 lanes x UNROLL x 16 picks x 4 bytes
      asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(32u * UNROLL * 16u * 4u) : "memory");
    __syncwarp();
    int4 x[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) x[u] = ldg_stream(v + i + u * T);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint32_t w[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) inc<MODE>(hbase + prmt(w[q], hslot, 0x5504u | (bb << 4)), bar);
    }
  }
  if (MODE == 1) {
    if (lane == 0) asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" :: "r"(bar) : "memory");
    asm volatile("{ .reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W%=; }" :: "r"(bar) : "memory");
  }
  __syncthreads();
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) s += smw[(i >> 5) * 64 + 32 + (i & 31)];
  atomicAdd(out, s);
}

int main() {
  const int64_t bytes = 4640000000LL;
  const int64_t nvec = bytes / 16;
  uint8_t* d; CK(cudaMalloc(&d, bytes));
  std::vector<uint8_t> h(1 << 24);
  uint64_t st = 88172645463325252ull;
  for (auto& x : h) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; double u = (st >> 11) * (1.0 / 9007199254740992.0); x = (uint8_t)(255.0 * u * u * u); }
  for (int64_t o = 0; o < bytes; o += h.size()) CK(cudaMemcpy(d + o, h.data(), std::min<int64_t>(h.size(), bytes - o), cudaMemcpyHostToDevice));
  unsigned long long* out; CK(cudaMalloc(&out, 8));
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int SM = 256 * 256;
  CK(cudaFuncSetAttribute(hist<0, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  CK(cudaFuncSetAttribute(hist<1, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  CK(cudaFuncSetAttribute(hist<0, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  CK(cudaFuncSetAttribute(hist<1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto bench = [&](const char* name, auto launch) {
    float best = 1e9; unsigned long long got = 0;
    for (int r = 0; r < 6; ++r) {
      CK(cudaMemset(out, 0, 8));
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) best = std::min(best, ms);
      CK(cudaMemcpy(&got, out, 8, cudaMemcpyDeviceToHost));
    }
    printf("%-34s best %7.3f ms  %8.1f GB/s  %5.1f%% of 6548   count %llu (expect %lld)\n", name, best, bytes / best / 1e6,
           100.0 * bytes / best / 1e6 / 6548.2, got, (long long)(nvec / (16 * 512 * 3 * nsm) * (16 * 512 * 3 * nsm)) * 16);
  };
  bench("red.shared (ATOMS), unroll 16", [&] { hist<0, 16><<<nsm * 3, 512, SM>>>((const int4*)d, nvec, out); });
  bench("red.async (REDAS), unroll 16", [&] { hist<1, 16><<<nsm * 3, 512, SM>>>((const int4*)d, nvec, out); });
  bench("red.shared (ATOMS), unroll 8", [&] { hist<0, 8><<<nsm * 3, 512, SM>>>((const int4*)d, nvec, out); });
  bench("red.async (REDAS), unroll 8", [&] { hist<1, 8><<<nsm * 3, 512, SM>>>((const int4*)d, nvec, out); });
  CK(cudaGetLastError());
  printf("done\n");
  return 0;
}
