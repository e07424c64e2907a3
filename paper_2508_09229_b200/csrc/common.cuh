// Shared device helpers for the moeplace sm_100a kernels.
#pragma once
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>
#include <cuda_runtime.h>
#include "../../include/moeplace_cuda.h"

namespace mp {

constexpr int kMaxE = 256;     // one-byte expert ids
constexpr int kThreads = 512;  // streaming kernels: 16 warps per CTA

// Streaming 128-bit load that does not allocate in L1 (each trace byte is read once).
__device__ __forceinline__ int4 ldg_stream(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// prmt.b32: builds a word from the bytes of (a, b).  Used to turn an expert byte into a
// shared-memory row offset in ONE instruction: selector SEL_ROW(b) puts byte b of `a` into
// result byte 1 (=> e << 8) and byte 0 of `b` (the lane's slot offset) into result byte 0.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// result = { byte0: b.byte0, byte1: a.byte[k], byte2: b.byte1 (=0), byte3: b.byte1 (=0) }
__host__ __device__ constexpr uint32_t sel_row(int k) { return 0x5504u | ((uint32_t)k << 4); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a));
  return r;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}

// shared-memory increment without return (ATOMS)
__device__ __forceinline__ void atoms_inc(uint32_t a) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(a));
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Bulk L2 prefetch of [p, p + bytes) (bytes a multiple of 16, p 16-byte aligned): raises the
// number of DRAM requests in flight without spending registers on them.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Warp reduce-scatter of P per-lane values (P = 4, 8, 16): after log2(P) halving exchanges at
// offsets 16, 8, ... every lane holds one value index q, then the remaining offsets finish the
// warp sum.  Cost: P - 1 + log2(32 / P) SHFLs instead of P * 5.  Lanes with
// (lane & (32/P - 1)) == 0 hold the complete warp sum of value q (returned in *q).
template <int P>
__device__ __forceinline__ uint32_t warp_reduce_scatter(uint32_t (&v)[P], int lane, int* q) {
  int idx = 0;
#pragma unroll
  for (int m = P, o = 16; m > 1; m >>= 1, o >>= 1) {
    const int h = m >> 1;
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const uint32_t send = up ? v[i] : v[i + h];
      const uint32_t keep = up ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
    idx = idx * 2 + (up ? 1 : 0);
  }
#pragma unroll
  for (int o = 16 / P; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
  *q = idx;
  return v[0];
}

// Record a data error: the first writer sets {code, a, b}; every writer bumps the count.
__device__ __forceinline__ void report_err(int64_t* err, int code, int64_t a, int64_t b, int64_t n = 1) {
  if (!err) return;
  unsigned long long* e = reinterpret_cast<unsigned long long*>(err);
  if (atomicCAS(e, 0ull, (unsigned long long)code) == 0ull) {
    e[1] = (unsigned long long)a;
    e[2] = (unsigned long long)b;
  }
  atomicAdd(e + 3, (unsigned long long)n);
}

__device__ __forceinline__ void atomic_add_i64(int64_t* p, int64_t v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// Work split shared by the streaming kernels: the byte space of all L planes restricted to
// [b0, b1) is flattened (plane-major) and cut into gridDim.x contiguous ranges; each CTA then
// walks the per-plane segments of its range.
struct Flat {
  int64_t nb;     // bytes per plane in range
  int64_t b0;     // first byte (within a plane)
  int64_t g0, g1; // this CTA's flattened range
  __device__ Flat(int64_t b0_, int64_t b1_, int L) : Flat(b0_, b1_, L, (int)blockIdx.x, (int)gridDim.x) {}
  // range `idx` of `n` (a kernel whose CTAs hold several independent workers)
  __device__ Flat(int64_t b0_, int64_t b1_, int L, int idx, int n) {
    b0 = b0_;
    nb = b1_ - b0_;
    int64_t total = nb * (int64_t)L;
    int64_t per = (total + n - 1) / n;
    per = (per + 15) & ~(int64_t)15;
    g0 = min(total, (int64_t)idx * per);
    g1 = min(total, g0 + per);
  }
};

// ---- host-side launch facts, queried once per device (and kernel) instead of on every launch:
// the streamed end-to-end path launches once per 1M-token slice.  The cache holds only device
// properties and occupancy results; it never owns device memory.
inline int device_sm_count() {
  int dev = 0;
  cudaGetDevice(&dev);
  static int cache[64] = {0};  // benign race: every writer stores the same value
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cache[dev] = n;
  return n;
}

// The kernel's max-dynamic-shared-memory attribute is raised (never lowered: it is per-function state,
// and a smaller later value would break a cached larger launch) once per (device, kernel, larger
// size); *per_sm = resident CTAs per SM at (threads, smem), from
// cudaOccupancyMaxActiveBlocksPerMultiprocessor (cached per (device, kernel, threads, smem)).
inline cudaError_t prepare_kernel(const void* kern, int threads, int smem, int* per_sm, bool occupancy = true) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, int>, int> occ;
  static std::map<std::tuple<int, const void*>, int> attr;  // largest size set so far
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, kern, threads, smem);
  std::lock_guard<std::mutex> g(mu);
  int& cur = attr[std::make_tuple(dev, kern)];
  if (smem > cur) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cur = smem;
  }
  const auto it = occ.find(key);
  if (it != occ.end()) {
    *per_sm = it->second;
    return cudaSuccess;
  }
  int n = 1;  // cluster kernels (CTA pairs) skip the occupancy query: one CTA per SM by construction
  if (occupancy) {
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem);
    if (e != cudaSuccess) return e;
  }
  occ[key] = n;
  *per_sm = n;
  return cudaSuccess;
}

}  // namespace mp
