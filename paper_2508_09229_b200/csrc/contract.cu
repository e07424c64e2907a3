// Exact per-chunk hop sums of many placements on the 5th-generation tensor cores:
//   out[q][c] += sum_i pe[q][i] * counts[c][i]       (i = l*E + e; SPEC.md:383 linearity)
//
// pe (uint8, the per-expert round-trip costs of placement q) is the A operand as it is (u8, K-major).
// The per-chunk counts are split into 8-bit digits (mp_count_digits_u8): B row n = c*ndig + a holds
// digit a of chunk c's counts, so ONE u8 x u8 GEMM with int32 accumulation gives every digit's
// partial side by side in TMEM, and the epilogue recombines them into int64 (sum_a part << 8a)
// before one atomic add per (q, c).  Exact: a u8*u8 product is <= 65025 and each CTA sums at most
// 32768 products into one int32 accumulator (its split-K range), < 2^31.
//
// Kernel (one CTA per SM, 128 threads): TMA (cp.async.bulk.tensor, 128-byte swizzle) streams
// 128 x 128 B pe tiles and NT x 128 B digit tiles into a `stages`-deep shared-memory ring guarded by
// full/empty mbarriers; one elected thread issues tcgen05.mma.cta_group::1.kind::i8 (M = 128,
// N <= 256 per instruction, K = 32) into TMEM accumulators (NT <= 512 columns) and frees each slot
// with tcgen05.commit; after the last k-block the four warps read their 32 TMEM lanes with
// tcgen05.ld.32x32b, recombine the digits and add to out with red.global.add.u64.  The grid is
// (M tiles, N tiles, split-K) sized to the 148 SMs; pe is read from HBM exactly once.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include "common.cuh"

namespace mp {
namespace {

constexpr int kBM = 128;               // pe rows per tile (MMA M)
constexpr int kBK = 128;               // K bytes per stage (one 128-byte swizzle row)
constexpr int kMaxStages = 8;
constexpr int kTcThreads = 128;
constexpr int kSmemLimit = 232448;     // 227 KB opt-in per CTA
constexpr int kMaxKPerSplit = 32768;   // int32 exactness bound: 65025 * 32768 < 2^31

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
// K-major operand tile with 128-byte swizzle: 8-row atoms of 1024 B (SBO = 1024 B), LBO unused (1),
// descriptor version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// instruction descriptor: D = S32 (c_format 2), A = B = U8 (format 0), both K-major, N >> 3, M >> 4
__device__ __forceinline__ uint32_t idesc_i8(int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct TcArgs {
  int P, C, ndig, n_cols;   // n_cols = C * ndig rows of the digit operand
  int NT;                   // digit rows per CTA (multiple of 16, <= 512)
  int kblocks, kb_per_split, stages, box_rows, n_loads;
  uint32_t tmem_cols;
  int64_t* out;
};

__global__ void __launch_bounds__(kTcThreads, 1)
    contract_tc_kernel(const __grid_constant__ CUtensorMap tm_pe, const __grid_constant__ CUtensorMap tm_dig, TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[2 * kMaxStages + 1];
  __shared__ uint32_t tmem_slot;
  const uint32_t base = (smem_addr(smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.stages;
  const uint32_t a_bytes = kBM * kBK, b_bytes = (uint32_t)a.NT * kBK, stage_bytes = a_bytes + b_bytes;
  const uint32_t full0 = smem_addr(&bars[0]), empty0 = smem_addr(&bars[kMaxStages]), done = smem_addr(&bars[2 * kMaxStages]);
  const int m0 = blockIdx.x * kBM;
  const int n0 = blockIdx.y * a.NT;                          // first digit row of this CTA
  const int kb0 = blockIdx.z * a.kb_per_split;
  const int kb1 = min(a.kblocks, kb0 + a.kb_per_split);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_pe)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dig)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                 "r"(a.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0 && lane == 0) {  // ---- TMA producer ----
    for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
      const int s = i % S;
      if (i >= S) mbar_wait(empty0 + 8 * s, ((i / S) - 1) & 1);
      const uint32_t dst = base + (uint32_t)s * stage_bytes;
      mbar_expect_tx(full0 + 8 * s, a_bytes + (uint32_t)a.n_loads * a.box_rows * kBK);
      tma_load_2d(dst, &tm_pe, kb * kBK, m0, full0 + 8 * s);
      for (int j = 0; j < a.n_loads; ++j)
        tma_load_2d(dst + a_bytes + (uint32_t)j * a.box_rows * kBK, &tm_dig, kb * kBK, n0 + j * a.box_rows,
                    full0 + 8 * s);
    }
  } else if (warp == 1 && lane == 0) {  // ---- MMA issuer (one thread) ----
    for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
      const int s = i % S;
      mbar_wait(full0 + 8 * s, (i / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = base + (uint32_t)s * stage_bytes, sb = sa + a_bytes;
#pragma unroll
      for (int k = 0; k < kBK / 32; ++k) {
        for (int j = 0; j * 256 < a.NT; ++j) {
          const int nj = min(256, a.NT - 256 * j);
          mma_i8(tmem + 256 * j, sw128_desc(sa + 32 * k), sw128_desc(sb + (uint32_t)j * 256 * kBK + 32 * k), idesc_i8(nj),
                 (i > 0 || k > 0) ? 1u : 0u);
        }
      }
      mma_commit(empty0 + 8 * s);  // the slot is free once these MMAs have read it
    }
    mma_commit(done);
  }
  __syncwarp();
  // ---- epilogue: TMEM -> registers -> digit recombine -> int64 atomics ----
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = m0 + warp * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  const int nd = a.ndig;
  for (int c0 = 0; c0 < a.NT; c0 += 16) {
    uint32_t v[16];
    tmem_ld16(trow + c0, v);
    if (row < a.P) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j % nd) continue;  // nd in {1, 2, 4} divides 16: column j starts a chunk's digit group
        const int n = n0 + c0 + j;
        if (n >= a.n_cols) break;
        int64_t val = 0;
        for (int d = 0; d < nd; ++d) val += (int64_t)v[j + d] << (8 * d);
        if (val) atomic_add_i64(a.out + (int64_t)row * a.C + n / nd, val);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
}

__global__ void count_digits_u8_kernel(const int64_t* __restrict__ counts, int C, int64_t LE, int ndig, int64_t ldd,
                                       uint8_t* __restrict__ out, int64_t* err) {
  // out[(c*ndig + a)*ldd + i] = byte a of counts[c*LE + i]; columns [LE, ldd) are zero
  const int64_t n = (int64_t)C * ldd;
  const int sh = 8 * ndig;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(j / ldd);
    const int64_t i = j - (int64_t)c * ldd;
    int64_t v = i < LE ? counts[(int64_t)c * LE + i] : 0;
    if (v < 0 || (sh < 64 && (v >> sh) != 0)) {
      report_err(err, MP_DATA_EXPERT_RANGE, c, i);
      v = 0;
    }
    for (int d = 0; d < ndig; ++d) out[((int64_t)c * ndig + d) * ldd + i] = (uint8_t)(v >> (8 * d));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;  // resolved once (a driver entry point)
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* ptr, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t box_rows) {
  auto fn = encode_tiled();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld};
  cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t launch_count_digits_u8(const int64_t* counts, int C, int64_t LE, int ndig, int64_t ldd, uint8_t* out,
                                   int64_t* err, cudaStream_t s) {
  const int64_t n = (int64_t)C * ldd;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  count_digits_u8_kernel<<<grid, 256, 0, s>>>(counts, C, LE, ndig, ldd, out, err);
  return cudaGetLastError();
}

// splits: 0 = choose (fill the SMs), else the split-K factor
cudaError_t launch_contract_tc(const uint8_t* pe, int P, int64_t ldpe, const uint8_t* digits, int C, int ndig,
                               int64_t LE, int64_t ldd, int64_t* out, int splits, cudaStream_t s) {
  if (P <= 0 || C <= 0 || LE <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  TcArgs a;
  a.P = P;
  a.C = C;
  a.ndig = ndig;
  a.n_cols = C * ndig;
  const int n_tiles = (a.n_cols + 511) / 512;
  const int per = (a.n_cols + n_tiles - 1) / n_tiles;
  a.NT = (per + 15) / 16 * 16;
  a.n_loads = (a.NT + 255) / 256;
  a.box_rows = ((a.NT + a.n_loads - 1) / a.n_loads + 7) / 8 * 8;
  a.tmem_cols = a.NT <= 32 ? 32 : a.NT <= 64 ? 64 : a.NT <= 128 ? 128 : a.NT <= 256 ? 256 : 512;
  a.kblocks = (int)((LE + kBK - 1) / kBK);
  const int m_tiles = (P + kBM - 1) / kBM;
  int sp = splits > 0 ? splits : std::max(1, sms / (m_tiles * n_tiles));
  sp = std::min(sp, a.kblocks);
  a.kb_per_split = (a.kblocks + sp - 1) / sp;
  a.kb_per_split = std::min(a.kb_per_split, kMaxKPerSplit / kBK);
  sp = (a.kblocks + a.kb_per_split - 1) / a.kb_per_split;
  const int stage_bytes = kBM * kBK + a.n_loads * a.box_rows * kBK;
  a.stages = std::min(kMaxStages, (kSmemLimit - 1024) / stage_bytes);
  if (a.stages < 2) return cudaErrorInvalidValue;
  a.out = out;
  CUtensorMap tm_pe, tm_dig;
  if (!make_map(&tm_pe, pe, (uint64_t)LE, (uint64_t)P, (uint64_t)ldpe, kBM)) return cudaErrorInvalidValue;
  if (!make_map(&tm_dig, digits, (uint64_t)LE, (uint64_t)a.n_cols, (uint64_t)ldd, (uint32_t)a.box_rows))
    return cudaErrorInvalidValue;
  const int smem = a.stages * stage_bytes + 1024;
  cudaError_t e = cudaFuncSetAttribute(contract_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  contract_tc_kernel<<<dim3((unsigned)m_tiles, (unsigned)n_tiles, (unsigned)sp), kTcThreads, smem, s>>>(tm_pe, tm_dig,
                                                                                                       a);
  return cudaGetLastError();
}

}  // namespace mp
