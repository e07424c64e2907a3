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
// Kernel (one CTA per SM, 6 warps): warp 4 streams 128 x 128 B pe tiles and NT x 128 B digit tiles
// with TMA (cp.async.bulk.tensor, 128-byte swizzle) into a `stages`-deep shared-memory ring guarded
// by full/empty mbarriers; one thread of warp 5 issues tcgen05.mma.cta_group::1.kind::i8 (M = 128,
// N <= 256 per instruction, K = 32) into TMEM accumulators (NT <= 512 columns) and frees each slot
// with tcgen05.commit; at the end of a segment warps 0-3 read their 32 TMEM lanes with
// tcgen05.ld.32x32b, recombine the digits and add to out with red.global.add.u64.  Work split:
// blockIdx.y = N tile, and the (pe tile, k-block) units are divided evenly over gridDim.x (stream-K;
// by default aligned so each CTA's range stays inside one pe tile); pe is read from HBM once.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include "common.cuh"

namespace mp {
namespace {

constexpr int kBM = 128;               // pe rows per tile (MMA M)
constexpr int kBK = 128;               // K bytes per stage (one 128-byte swizzle row)
constexpr int kMaxStages = 8;
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

template <int ND>
__device__ __forceinline__ void stage_values(const uint32_t (&v)[16], int64_t* row) {
#pragma unroll
  for (int j = 0; j < 16 / ND; ++j) {
    int64_t val = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d) val += (int64_t)v[j * ND + d] << (8 * d);
    row[j] = val;
  }
}

struct TcArgs {
  int P, C, ndig, n_cols;   // n_cols = C * ndig rows of the digit operand
  int NT;                   // digit rows per CTA (multiple of 16, <= 512)
  int kblocks, m_tiles;     // k-blocks of 128 B per row; 128-row tiles of pe
  int64_t units;            // m_tiles * kblocks (unit = one k-block of one pe tile), split evenly over gridDim.x
  int max_seg;              // k-blocks one accumulation may span (int32 exactness: 256)
  int stages, box_rows, n_loads;
  uint32_t tmem_cols;
  int64_t* out;
};

// Stream-K work split: CTA i owns units [i*U/G, (i+1)*U/G) of the (tile, k-block) sequence; a run of
// units of one pe tile (at most max_seg long) accumulates in TMEM and is flushed by one epilogue.
struct Seg {
  int64_t u, end;
  __device__ bool next(const TcArgs& a, int64_t u1, int64_t* s0, int64_t* s1) {
    if (u >= u1) return false;
    const int64_t tile_end = (u / a.kblocks + 1) * a.kblocks;
    *s0 = u;
    *s1 = min(min(u1, tile_end), u + a.max_seg);
    u = *s1;
    return true;
  }
};

constexpr int kEpiWarps = 4;                  // warps 0-3: epilogue (TMEM lane quadrants 0-3)
constexpr int kTcThreads2 = 32 * (kEpiWarps + 2);  // + warp 4: TMA producer, warp 5: MMA issuer
constexpr int kEpiTileBytes = 32 * 17 * 8;    // per warp: 32 rows x <= 16 int64 values, pitch 17

__global__ void __launch_bounds__(kTcThreads2, 1)
    contract_tc_kernel(const __grid_constant__ CUtensorMap tm_pe, const __grid_constant__ CUtensorMap tm_dig, TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[2 * kMaxStages + 2];
  __shared__ uint32_t tmem_slot;
  const uint32_t base = (smem_addr(smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.stages;
  const uint32_t a_bytes = kBM * kBK, b_bytes = (uint32_t)a.n_loads * a.box_rows * kBK, stage_bytes = a_bytes + b_bytes;
  const uint32_t full0 = smem_addr(&bars[0]), empty0 = smem_addr(&bars[kMaxStages]);
  const uint32_t tmem_full = smem_addr(&bars[2 * kMaxStages]), tmem_empty = smem_addr(&bars[2 * kMaxStages + 1]);
  const int n0 = blockIdx.y * a.NT;  // first digit row of this CTA's N tile
  const int64_t u0 = blockIdx.x * a.units / gridDim.x, u1 = (blockIdx.x + 1) * a.units / gridDim.x;

  if (warp == 4 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, kEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_pe)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dig)) : "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                 "r"(a.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 4) {  // ---- TMA producer ----
    if (lane == 0) {
      int i = 0;
      for (int64_t u = u0; u < u1; ++u, ++i) {
        const int s = i % S;
        if (i >= S) mbar_wait(empty0 + 8 * s, ((i / S) - 1) & 1);
        const int m0 = (int)(u / a.kblocks) * kBM, kb = (int)(u % a.kblocks);
        const uint32_t dst = base + (uint32_t)s * stage_bytes;
        mbar_expect_tx(full0 + 8 * s, stage_bytes);
        tma_load_2d(dst, &tm_pe, kb * kBK, m0, full0 + 8 * s);
        for (int j = 0; j < a.n_loads; ++j)
          tma_load_2d(dst + a_bytes + (uint32_t)j * a.box_rows * kBK, &tm_dig, kb * kBK, n0 + j * a.box_rows,
                      full0 + 8 * s);
      }
    }
  } else if (warp == 5) {  // ---- MMA issuer (one thread) ----
    if (lane == 0) {
      Seg sg{u0, u1};
      int64_t s0, s1;
      int i = 0, seg = 0;
      while (sg.next(a, u1, &s0, &s1)) {
        if (seg > 0) mbar_wait(tmem_empty, (seg - 1) & 1);  // the epilogue has drained the accumulators
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int64_t u = s0; u < s1; ++u, ++i) {
          const int s = i % S;
          mbar_wait(full0 + 8 * s, (i / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = base + (uint32_t)s * stage_bytes, sb = sa + a_bytes;
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k) {
            for (int j = 0; j * 256 < a.NT; ++j) {
              const int nj = min(256, a.NT - 256 * j);
#ifdef MP_TC_EXPERIMENT_NO_MMA
              if (u >= 0) continue;
#endif
              mma_i8(tmem + 256 * j, sw128_desc(sa + 32 * k), sw128_desc(sb + (uint32_t)j * 256 * kBK + 32 * k),
                     idesc_i8(nj), (u > s0 || k > 0) ? 1u : 0u);
            }
          }
          mma_commit(empty0 + 8 * s);  // the slot is free once these MMAs have read it
        }
        mma_commit(tmem_full);
        ++seg;
      }
    }
  } else {  // ---- epilogue warps 0-3: TMEM -> registers -> digit recombine -> coalesced int64 atomics ----
    uint8_t* tile = smem_raw + (base - smem_addr(smem_raw)) + (uint32_t)S * stage_bytes + warp * kEpiTileBytes;
    int64_t* t64 = reinterpret_cast<int64_t*>(tile);
    const int nd = a.ndig, V = 16 / nd;  // chunk values per 16 columns
    Seg sg{u0, u1};
    int64_t s0, s1;
    int seg = 0;
    while (sg.next(a, u1, &s0, &s1)) {
      mbar_wait(tmem_full, seg & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row0 = (int)(s0 / a.kblocks) * kBM + warp * 32;
      const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
      for (int c0 = 0; c0 < a.NT; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(trow + c0, v);
        if (c0 + 16 >= a.NT) {  // last TMEM read of this segment: hand the accumulators back
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tmem_empty) : "memory");
        }
        // digit recombine: value j of this row = sum_d v[j*nd + d] << 8d, staged as tile[row][j]
        if (nd == 1) stage_values<1>(v, t64 + lane * 17);
        else if (nd == 2) stage_values<2>(v, t64 + lane * 17);
        else stage_values<4>(v, t64 + lane * 17);
        __syncwarp();
        // write-out: instruction r covers rows 32/V * r .. and V consecutive chunks per row
        const int cbase = (n0 + c0) / nd;
        for (int r = 0; r < V; ++r) {
          const int idx = r * 32 + lane;
          const int rr = idx / V, j = idx % V;
          const int row = row0 + rr, ch = cbase + j;
          const int64_t val = t64[rr * 17 + j];
#ifdef MP_TC_EXPERIMENT_NO_ATOMICS
          if (val == 0x7fffffffffffll) a.out[0] = val;
#else
          if (val && row < a.P && ch < a.C && (n0 + c0) + j * nd < a.n_cols)
            atomic_add_i64(a.out + (int64_t)row * a.C + ch, val);
#endif
        }
        __syncwarp();
      }
      ++seg;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 5)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
}

// ---- CTA-pair variant (tcgen05 cta_group::2) ------------------------------------------------
// Two CTAs of a cluster on one TPC form an M = 256 tile: CTA r loads pe rows m0 + 128r (A) and HALF of
// the N tile's digit rows (B rows n0 + H*r .. + H, H = NT/2) into its own shared memory, both with
// `cp.async.bulk.tensor.cta_group::2` signalling the leader's full barrier; the leader's single
// thread issues `tcgen05.mma.cta_group::2.kind::i8`, which reads A and B from both CTAs and writes
// D rows 128r.. into CTA r's TMEM; commits multicast to both CTAs' barriers.  Per k-block an SM
// receives 128 + H rows instead of 128 + 2H (config 4: 35.5 KB instead of 55 KB).  Measured
// (tools/probe_contract.py, config 4): bit-exact, but 0.058 ms with 64 pairs against 0.039 ms for
// 128 single CTAs -- operand bytes were not the single-CTA kernel's limit (ncu: TMA/L2 reads at 6 % of
// peak; the pair waits for the slower CTA's loads and the leader's thread issues M = 256 MMAs for
// both) -- so AUTO keeps single CTAs and the pair kernel runs on request (ctas < 0).  TMEM column j holds digit row map(j): the first MMA
// covers B rows [0, h1) of each half (columns [0, h1) from CTA 0, [h1, 2h1) from CTA 1), a second
// one the remaining H - h1 rows of each half.
struct Tc2Args {
  int P, C, ndig, n_cols;
  int NT, H, h1;            // digit rows per N tile, per CTA half (NT / 2), per half in the first MMA
  int kblocks, m_tiles;     // k-blocks of 128 B; 256-row pe tiles
  int64_t units;            // m_tiles * kblocks, split evenly over the pairs
  int max_seg, stages;
  uint32_t tmem_cols;
  int64_t* out;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ uint32_t idesc_i8_m256(int n) {
  return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}
// digit row (relative to the N tile) held by TMEM column j
__device__ __forceinline__ int pair_col_row(int j, int H, int h1) {
  if (j < 2 * h1) return (j >= h1 ? H : 0) + (j % h1);
  const int jj = j - 2 * h1, h2 = H - h1;
  return (jj >= h2 ? H : 0) + h1 + (jj % h2);
}

struct Seg2 {
  int64_t u;
  __device__ bool next(const Tc2Args& a, int64_t u1, int64_t* s0, int64_t* s1) {
    if (u >= u1) return false;
    const int64_t tile_end = (u / a.kblocks + 1) * a.kblocks;
    *s0 = u;
    *s1 = min(min(u1, tile_end), u + a.max_seg);
    u = *s1;
    return true;
  }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads2, 1)
    contract_tc2_kernel(const __grid_constant__ CUtensorMap tm_pe, const __grid_constant__ CUtensorMap tm_dig,
                        Tc2Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[2 * kMaxStages + 2];
  __shared__ uint32_t tmem_slot;
  const uint32_t base = (smem_addr(smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int S = a.stages;
  const uint32_t a_bytes = 128 * kBK, b_bytes = (uint32_t)a.H * kBK, stage_bytes = a_bytes + b_bytes;
  const uint32_t full0 = smem_addr(&bars[0]), empty0 = smem_addr(&bars[kMaxStages]);
  const uint32_t tmem_full = smem_addr(&bars[2 * kMaxStages]), tmem_empty = smem_addr(&bars[2 * kMaxStages + 1]);
  const int n0 = blockIdx.y * a.NT;
  const int pair = (int)(blockIdx.x >> 1), npairs = (int)(gridDim.x >> 1);
  const int64_t u0 = pair * a.units / npairs, u1 = (pair + 1) * a.units / npairs;

  if (warp == 4 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 2 * kEpiWarps);  // the epilogue warps of both CTAs
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_pe)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dig)) : "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                 "r"(a.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // both CTAs' barriers initialised and TMEM allocated
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 4) {  // ---- TMA producer (each CTA loads its own A rows and B half) ----
    if (lane == 0) {
      const uint32_t full_lead = mapa_shared(full0, 0);
      int i = 0;
      for (int64_t u = u0; u < u1; ++u, ++i) {
        const int s = i % S;
        if (i >= S) mbar_wait(empty0 + 8 * s, ((i / S) - 1) & 1);
        const int m0 = (int)(u / a.kblocks) * 256 + (int)rank * 128, kb = (int)(u % a.kblocks);
        const uint32_t dst = base + (uint32_t)s * stage_bytes;
        if (rank == 0) mbar_expect_tx(full0 + 8 * s, 2 * stage_bytes);  // both CTAs' bytes
        tma_load_2d_pair(dst, &tm_pe, kb * kBK, m0, full_lead + 8 * s);
        tma_load_2d_pair(dst + a_bytes, &tm_dig, kb * kBK, n0 + (int)rank * a.H, full_lead + 8 * s);
      }
    }
  } else if (warp == 5) {  // ---- MMA issuer: one thread of the leader CTA ----
    if (rank == 0 && lane == 0) {
      Seg2 sg{u0};
      int64_t s0, s1;
      int i = 0, seg = 0;
      const int h2 = a.H - a.h1;
      while (sg.next(a, u1, &s0, &s1)) {
        if (seg > 0) mbar_wait(tmem_empty, (seg - 1) & 1);  // both epilogues have drained TMEM
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int64_t u = s0; u < s1; ++u, ++i) {
          const int s = i % S;
          mbar_wait(full0 + 8 * s, (i / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = base + (uint32_t)s * stage_bytes, sb = sa + a_bytes;
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k) {
            const uint32_t acc = (u > s0 || k > 0) ? 1u : 0u;
            mma_i8_pair(tmem, sw128_desc(sa + 32 * k), sw128_desc(sb + 32 * k), idesc_i8_m256(2 * a.h1), acc);
            if (h2 > 0)
              mma_i8_pair(tmem + 2 * a.h1, sw128_desc(sa + 32 * k), sw128_desc(sb + (uint32_t)a.h1 * kBK + 32 * k),
                          idesc_i8_m256(2 * h2), acc);
          }
          mma_commit_pair(empty0 + 8 * s);  // frees slot s in both CTAs
        }
        mma_commit_pair(tmem_full);
        ++seg;
      }
    }
  } else {  // ---- epilogue warps 0-3 of each CTA: own TMEM lanes = pe rows m0 + 128 * rank + ... ----
    uint8_t* tile = smem_raw + (base - smem_addr(smem_raw)) + (uint32_t)S * stage_bytes + warp * kEpiTileBytes;
    int64_t* t64 = reinterpret_cast<int64_t*>(tile);
    const int nd = a.ndig, V = 16 / nd;
    const uint32_t empty_lead = mapa_shared(tmem_empty, 0);
    Seg2 sg{u0};
    int64_t s0, s1;
    int seg = 0;
    while (sg.next(a, u1, &s0, &s1)) {
      mbar_wait(tmem_full, seg & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row0 = (int)(s0 / a.kblocks) * 256 + (int)rank * 128 + warp * 32;
      const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
      for (int c0 = 0; c0 < 2 * a.H; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(trow + c0, v);
        if (c0 + 16 >= 2 * a.H) {  // last TMEM read of this segment: tell the leader
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(empty_lead) : "memory");
        }
        if (nd == 1) stage_values<1>(v, t64 + lane * 17);
        else if (nd == 2) stage_values<2>(v, t64 + lane * 17);
        else stage_values<4>(v, t64 + lane * 17);
        __syncwarp();
        for (int r = 0; r < V; ++r) {
          const int idx = r * 32 + lane;
          const int rr = idx / V, j = idx % V;
          const int row = row0 + rr;
          const int drow = n0 + pair_col_row(c0 + j * nd, a.H, a.h1);  // first digit row of this value
          const int ch = drow / nd;
          const int64_t val = t64[rr * 17 + j];
          if (val && row < a.P && ch < a.C && drow < a.n_cols) atomic_add_i64(a.out + (int64_t)row * a.C + ch, val);
        }
        __syncwarp();
      }
      ++seg;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // neither CTA frees TMEM while the pair's MMAs may still target it
  if (warp == 5)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
}

// out[(c*ndig + a)*ldd + i] = byte a of counts[c*LE + i]; columns [LE, ldd) are zero.  One thread per
// 8 consecutive columns of one chunk row (blockIdx.y = chunk): eight int64 loads, ndig u64 stores.
__global__ void count_digits_u8_kernel(const int64_t* __restrict__ counts, int C, int64_t LE, int ndig, int64_t ldd,
                                       uint8_t* __restrict__ out, int64_t* err) {
  const int c = blockIdx.y;
  const int sh = 8 * ndig;
  const int64_t* row = counts + (int64_t)c * LE;
  for (int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8; i0 < ldd;
       i0 += (int64_t)gridDim.x * blockDim.x * 8) {
    uint64_t w[4] = {0, 0, 0, 0};
    int64_t vv[8];
    if (i0 + 8 <= LE && (reinterpret_cast<uintptr_t>(row) & 15) == 0) {  // 16-byte loads when the row is aligned
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const longlong2 p = __ldg(reinterpret_cast<const longlong2*>(row + i0 + k));
        vv[k] = p.x;
        vv[k + 1] = p.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) vv[k] = i0 + k < LE ? __ldg(row + i0 + k) : 0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t i = i0 + k;
      int64_t v = vv[k];
      if (v < 0 || (sh < 64 && (v >> sh) != 0)) {
        report_err(err, MP_DATA_EXPERT_RANGE, c, i);
        v = 0;
      }
#pragma unroll
      for (int d = 0; d < 4; ++d) w[d] |= (uint64_t)((v >> (8 * d)) & 0xff) << (8 * k);
    }
    if (i0 + 8 <= ldd) {  // ldd is a multiple of 16: every 8-column group is whole
#pragma unroll
      for (int d = 0; d < 4; ++d)
        if (d < ndig) *reinterpret_cast<uint64_t*>(out + ((int64_t)c * ndig + d) * ldd + i0) = w[d];
    }
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
  const int gx = (int)std::min<int64_t>((ldd / 8 + 127) / 128, 64);
  count_digits_u8_kernel<<<dim3(gx, C), 128, 0, s>>>(counts, C, LE, ndig, ldd, out, err);
  return cudaGetLastError();
}

static cudaError_t launch_contract_tc2(const uint8_t* pe, int P, int64_t ldpe, const uint8_t* digits, int C, int ndig,
                                       int64_t LE, int64_t ldd, int64_t* out, int pairs, int sms, cudaStream_t s) {
  Tc2Args a;
  a.P = P;
  a.C = C;
  a.ndig = ndig;
  a.n_cols = C * ndig;
  const int n_tiles = (a.n_cols + 511) / 512;
  const int per = (a.n_cols + n_tiles - 1) / n_tiles;
  a.NT = (per + 31) / 32 * 32;  // H = NT / 2 a multiple of 16 (swizzle atoms, digit groups)
  a.H = a.NT / 2;
  a.h1 = std::min(128, a.H);
  a.tmem_cols = a.NT <= 32 ? 32 : a.NT <= 64 ? 64 : a.NT <= 128 ? 128 : a.NT <= 256 ? 256 : 512;
  a.kblocks = (int)((LE + kBK - 1) / kBK);
  a.m_tiles = (P + 255) / 256;
  a.units = (int64_t)a.m_tiles * a.kblocks;
  a.max_seg = kMaxKPerSplit / kBK;
  const int per_n = std::max(1, sms / 2 / n_tiles);  // pairs per N tile
  int64_t g = pairs > 0 ? pairs : (a.m_tiles <= per_n ? (int64_t)a.m_tiles * (per_n / a.m_tiles) : per_n);
  g = std::min(g, a.units);
  const int stage_bytes = 128 * kBK + a.H * kBK;
  const int epi_bytes = kEpiWarps * kEpiTileBytes;
  a.stages = std::min(kMaxStages, (kSmemLimit - 2048 - epi_bytes) / stage_bytes);
  if (a.stages < 2) return cudaErrorInvalidValue;
  a.out = out;
  CUtensorMap tm_pe, tm_dig;
  if (!make_map(&tm_pe, pe, (uint64_t)LE, (uint64_t)P, (uint64_t)ldpe, 128)) return cudaErrorInvalidValue;
  if (!make_map(&tm_dig, digits, (uint64_t)LE, (uint64_t)a.n_cols, (uint64_t)ldd, (uint32_t)a.H))
    return cudaErrorInvalidValue;
  const int smem = a.stages * stage_bytes + epi_bytes + 1024;
  int per_sm = 0;
  cudaError_t e = prepare_kernel((const void*)contract_tc2_kernel, kTcThreads2, smem, &per_sm, false);
  if (e != cudaSuccess) return e;
  contract_tc2_kernel<<<dim3((unsigned)(2 * g), (unsigned)n_tiles), kTcThreads2, smem, s>>>(tm_pe, tm_dig, a);
  return cudaGetLastError();
}

// ctas: 0 = auto (single CTAs, tile-aligned split), > 0 = that many single CTAs per N tile
// (stream-K), < 0 = -ctas CTA pairs per N tile (cta_group::2; measured slower, see above)
cudaError_t launch_contract_tc(const uint8_t* pe, int P, int64_t ldpe, const uint8_t* digits, int C, int ndig,
                               int64_t LE, int64_t ldd, int64_t* out, int ctas, cudaStream_t s) {
  if (P <= 0 || C <= 0 || LE <= 0) return cudaSuccess;
  const int sms = device_sm_count();
  if (ctas < 0) return launch_contract_tc2(pe, P, ldpe, digits, C, ndig, LE, ldd, out, -ctas, sms, s);
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
  a.m_tiles = (P + kBM - 1) / kBM;
  a.units = (int64_t)a.m_tiles * a.kblocks;
  a.max_seg = kMaxKPerSplit / kBK;
  // auto: split every pe tile's k-blocks into the same number of ranges so that no CTA's range
  // crosses a tile (one epilogue per CTA): g = m_tiles * floor(SMs per N tile / m_tiles); with more
  // tiles than SMs, plain stream-K over all units.  Config 4 (32 tiles): 128 CTAs, 0.039 ms, against
  // 0.050 ms for 148 CTAs whose ranges straddle tiles (two serialized epilogues each).
  const int per_n = std::max(1, sms / n_tiles);
  int64_t g = ctas > 0 ? ctas : (a.m_tiles <= per_n ? (int64_t)a.m_tiles * (per_n / a.m_tiles) : per_n);
  g = std::min(g, a.units);
  const int stage_bytes = kBM * kBK + a.n_loads * a.box_rows * kBK;
  const int epi_bytes = kEpiWarps * kEpiTileBytes;
  a.stages = std::min(kMaxStages, (kSmemLimit - 2048 - epi_bytes) / stage_bytes);
  if (a.stages < 2) return cudaErrorInvalidValue;
  a.out = out;
  CUtensorMap tm_pe, tm_dig;
  if (!make_map(&tm_pe, pe, (uint64_t)LE, (uint64_t)P, (uint64_t)ldpe, kBM)) return cudaErrorInvalidValue;
  if (!make_map(&tm_dig, digits, (uint64_t)LE, (uint64_t)a.n_cols, (uint64_t)ldd, (uint32_t)a.box_rows))
    return cudaErrorInvalidValue;
  const int smem = a.stages * stage_bytes + epi_bytes + 1024;
  int per_sm = 0;
  cudaError_t e = prepare_kernel((const void*)contract_tc_kernel, kTcThreads2, smem, &per_sm);
  if (e != cudaSuccess) return e;
  contract_tc_kernel<<<dim3((unsigned)g, (unsigned)n_tiles), kTcThreads2, smem, s>>>(tm_pe, tm_dig, a);
  return cudaGetLastError();
}

}  // namespace mp
