// Cross-GPU sum of the packed int64 result vector [counts | hop sums] over NVLink / NVSwitch peer
// memory (the path's one exchange step), replacing the NCCL all_reduce after the fused
// pass.  The vector lives in symmetric memory (torch.distributed._symmetric_memory): every rank's
// buffer is mapped into every other rank's address space, and on NVSwitch systems a multicast object
// covers all copies, so ONE `multimem.ld_reduce.add.u64` per element returns the sum over the world
// computed in the switch (NVLS); without multicast each element is summed from the peers' copies
// with plain P2P loads.
//
// One kernel, G CTAs (as many slices as the signal pad allows: 61 for the config-2 vector at 8 GPUs,
// one element per thread), CTA b owns a contiguous slice of the vector:
//   1. barrier: each thread t < world stores the epoch into rank t's signal pad (st.release.sys),
//      then waits until every rank's store for slice b arrived in its own pad (ld.acquire.sys):
//      all ranks' partials of slice b are complete and visible;
//   2. sums slice b of the world's copies (NVLS or P2P loads, all in flight) into `out`, a private
//      buffer.
// The symmetric inputs are double-buffered by the caller (even / odd epochs), so no second barrier
// is needed: a rank rewrites an input half only two calls later, after the next call's barrier,
// which every peer reaches only once its reads of this call are done (stream order).  Slices
// synchronise independently, so there is no grid-wide barrier.  Spins are bounded (~2 s of clock):
// a missing peer raises MP_DATA_UNREACHABLE in err instead of hanging the GPU.
#include <algorithm>

#include "common.cuh"

namespace mp {
namespace {

constexpr int kArThreads = 256;
constexpr int kArMaxPerThread = 8;  // elements per thread, loads issued together (latency-bound)
constexpr int kArPadWords = 1024;   // signal-pad words available: 2 * world * slices <= this
constexpr int kArPadBase = 1024;    // first signal-pad word used (torch's own barrier uses the low words)

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int64_t ld_reduce_add_u64(const int64_t* mc) {
  uint64_t v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u64 %0, [%1];" : "=l"(v) : "l"(mc) : "memory");
  return (int64_t)v;
}

// returns false on timeout
__device__ __forceinline__ bool pad_barrier(uint32_t* const* pads, int rank, int world, int slot0, uint32_t epoch) {
  bool ok = true;
  if ((int)threadIdx.x < world) {
    // st.release.sys orders this rank's earlier writes (the partials, written by the preceding kernel
    // on this stream) before the flag at system scope
    st_release_sys(pads[threadIdx.x] + kArPadBase + slot0 + rank, epoch);
    const uint32_t* mine = pads[rank] + kArPadBase + slot0 + threadIdx.x;
    const long long t0 = clock64();
    // at least this epoch: a fast peer may already have moved on to the next call and stored a larger
    // one (it can only do so after its own part of this call is complete)
    while ((int)(ld_acquire_sys(mine) - epoch) < 0) {
      if (clock64() - t0 > (1ll << 32)) {
        ok = false;
        break;
      }
    }
  }
  return __syncthreads_and(ok) != 0;
}

__global__ void __launch_bounds__(kArThreads) allreduce_kernel(int64_t* __restrict__ out, int64_t n, int slice,
                                                               const int64_t* mc, const int64_t* const* peers,
                                                               uint32_t* const* pads, int rank, int world,
                                                               uint32_t epoch, int64_t* err) {
  const int b = blockIdx.x;
  const int64_t i0 = (int64_t)b * slice, i1 = min(n, i0 + slice);
  if (i0 >= n) return;
  if (!pad_barrier(pads, rank, world, b * world, epoch)) {
    if (threadIdx.x == 0) report_err(err, MP_DATA_UNREACHABLE, rank, b);
    return;
  }
  // every load of this thread in flight at once: each is a round trip through NVLink / the switch
  int64_t v[kArMaxPerThread];
#pragma unroll
  for (int j = 0; j < kArMaxPerThread; ++j) {
    const int64_t i = i0 + threadIdx.x + (int64_t)j * kArThreads;
    v[j] = 0;
    if (i < i1) {
      if (mc) {
        v[j] = ld_reduce_add_u64(mc + i);  // summed in the NVSwitch
      } else {
        for (int r = 0; r < world; ++r) v[j] += peers[r][i];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kArMaxPerThread; ++j) {
    const int64_t i = i0 + threadIdx.x + (int64_t)j * kArThreads;
    if (i < i1) out[i] = v[j];
  }
}

}  // namespace

// slices: as many as the signal pad allows (one element per thread when possible), each CTA's loads
// all in flight; 0 if the vector is too long for kArMaxPerThread elements per thread
static int ar_slice(int64_t n, int world) {
  const int max_slices = kArPadWords / world;
  int64_t slice = std::max<int64_t>(kArThreads, (n + max_slices - 1) / max_slices);
  slice = (slice + kArThreads - 1) / kArThreads * kArThreads;
  return slice > (int64_t)kArThreads * kArMaxPerThread ? 0 : (int)slice;
}

int allreduce_supported(int64_t n, int world) { return ar_slice(n, world) > 0; }

cudaError_t launch_allreduce_i64(int64_t* out, int64_t n, const int64_t* mc, const int64_t* const* peers,
                                 uint32_t* const* pads, int rank, int world, uint32_t epoch, int64_t* err,
                                 cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int slice = ar_slice(n, world);
  if (!slice) return cudaErrorInvalidValue;
  const int g = (int)((n + slice - 1) / slice);
  allreduce_kernel<<<g, kArThreads, 0, s>>>(out, n, slice, mc, peers, pads, rank, world, epoch, err);
  return cudaGetLastError();
}

}  // namespace mp
