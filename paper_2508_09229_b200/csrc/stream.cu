// Streaming kernels over layer-major u8 traces: load statistics (hist), placement traffic
// (score) and the fused pass.  One kernel template serves all of them, with two of the three
// exact hop-sum algorithms (gather, count-contract; the token-tiled one is in tokens.cu).
//
// Design: the byte space of the L planes is cut into gridDim.x contiguous
// ranges; a CTA walks its range plane segment by plane segment, and chunk boundaries cut a
// segment into pieces (one layer x one chunk).  Per segment it stages layer l's state in shared
// memory as 256 rows of 256 B, one row per expert id e:
//   * gather: P = 4W placement hop costs (u8 lanes), replicated per lane slot so the 32 lanes
//     of a warp never bank-conflict (slot = lane*4 | lane*8 | (lane&7)*16 for W = 1 | 2 | 4 ->
//     one LDS.32 | LDS.64 | LDS.128 wavefront per 32 | 16 | 8 lanes);
//   * histogram: 32 u32 replicas of bin e at bytes 128 + lane*4 (bank = lane), so the ATOMS of
//     one warp hit 32 distinct banks and no address is shared between lanes; count-contract
//     alternates pieces between this set and a second one at bytes 0..127.
// An expert byte b of a loaded word becomes its row offset (e << 8) | slot with a single
// PRMT, so a lookup costs PRMT + LDS (gather) and/or PRMT + ATOMS (histogram).  The trace is
// streamed with 128-bit L1-no-allocate loads, UNROLL vectors per thread per main-loop batch.
// The count-contract and per-chunk-histogram instances run pipe_kernel instead (three rotating
// replica sets of 128-byte rows and per-set mbarriers in place of a CTA barrier per piece; see
// the comment above pipe_kernel); stream_kernel keeps the gather, the plain histogram and the
// MP_PIPE_FLUSH=0 comparison build.
#include <algorithm>
#include "common.cuh"

namespace mp {

template <int W>
struct ScoreAcc {
  static constexpr int P = 4 * W;
  uint32_t tot[P];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < P; ++q) tot[q] = 0;
  }
};

// one table lookup at row offset `a` (shared address), returning W words
template <int W>
__device__ __forceinline__ void table_load(uint32_t a, uint32_t (&t)[W]) {
  if constexpr (W == 1) {
    t[0] = lds32(a);
  } else if constexpr (W == 2) {
    uint2 v = lds64(a);
    t[0] = v.x; t[1] = v.y;
  } else {
    uint4 v = lds128(a);
    t[0] = v.x; t[1] = v.y; t[2] = v.z; t[3] = v.w;
  }
}

// L2 bulk-prefetch lookahead in main-loop iterations (0 = off, the default).  Measured on B200
// (R1, 10M tokens): at 2 iterations it speeds the ATOMS-bound histogram kernels by 1-3 % (hist
// 0.902 -> 0.878 ms, fused 1.370 -> 1.354 ms) but raises their DRAM traffic to 1.09-1.13x the
// algorithmic bytes (ncu), and slows the gather (0.799 -> 0.903 ms); kept as a build option only.
#ifndef MP_PF_AHEAD
#define MP_PF_AHEAD 0
#endif
// Vectors per thread per main-loop iteration (R1, 10M tokens, B200): histogram / count-contract
// instances 2: 0.894 / 4: 0.895 / 8: 0.846 / 16: 0.840 / 32: 0.843 ms (hist), fused step 0.936 ->
// 0.886 ms at 16; gather instances 2: 0.963 / 4: 0.795 / 8: 0.770-0.787 / 16: 0.796 ms (score W=1).
#ifndef MP_FLUSH_SNAPSHOT
#define MP_FLUSH_SNAPSHOT 1
#endif
#ifndef MP_COUNT_UNROLL
#define MP_COUNT_UNROLL 16
#endif
#ifndef MP_GATHER_UNROLL
#define MP_GATHER_UNROLL 8
#endif

template <bool HIST, int W, int WIDEN, int UNROLL>
struct Stream {
  static constexpr int P = 4 * W;
  uint32_t base;   // shared address of row 0
  uint32_t hbase;  // shared address of row 0's histogram replicas (base + 128, or base for set B)
  uint32_t slot;   // lane's score slot (byte 0 of the row offset)
  uint32_t hslot;  // lane's histogram slot
  uint32_t tid;    // this thread's index among the streaming threads
  uint32_t nth;    // number of streaming threads

  // single byte (heads/tails of ranges; rare)
  __device__ __forceinline__ void one(uint32_t e, ScoreAcc<(W > 0 ? W : 1)>& acc) {
    if constexpr (HIST) atoms_inc(hbase + ((e << 8) | hslot));
    if constexpr (W > 0) {
      uint32_t t[W];
      table_load<W>(base + ((e << 8) | slot), t);
#pragma unroll
      for (int w = 0; w < W; ++w)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc.tot[4 * w + j] += (t[w] >> (8 * j)) & 0xffu;
    }
  }

  // 16 bytes -> lookups; u8-lane sums widened into u16-lane accumulators every WIDEN lookups
  __device__ __forceinline__ void vec(const int4& x, uint32_t (&acc16)[2 * (W > 0 ? W : 1)]) {
    const uint32_t wd[4] = {(uint32_t)x.x, (uint32_t)x.y, (uint32_t)x.z, (uint32_t)x.w};
    constexpr int WW = W > 0 ? W : 1;
    uint32_t acc8[WW];
#pragma unroll
    for (int w = 0; w < WW; ++w) acc8[w] = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if constexpr (W > 0) {
          const uint32_t off = prmt(wd[q], slot, sel_row(b));
          uint32_t t[W];
          table_load<W>(base + off, t);
#pragma unroll
          for (int w = 0; w < W; ++w) acc8[w] += t[w];
          if constexpr (HIST) {
            const uint32_t hoff = (W == 1) ? off : prmt(wd[q], hslot, sel_row(b));
            atoms_inc(hbase + hoff);
          }
          if (((q * 4 + b + 1) % WIDEN) == 0) {
#pragma unroll
            for (int w = 0; w < W; ++w) {
              acc16[2 * w] += acc8[w] & 0x00ff00ffu;
              acc16[2 * w + 1] += (acc8[w] >> 8) & 0x00ff00ffu;
              acc8[w] = 0;
            }
          }
        } else {
          const uint32_t off = prmt(wd[q], hslot, sel_row(b));
          atoms_inc(hbase + off);
        }
      }
    }
  }

  __device__ __forceinline__ void widen(uint32_t (&acc16)[2 * (W > 0 ? W : 1)], ScoreAcc<(W > 0 ? W : 1)>& acc) {
    if constexpr (W > 0) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        acc.tot[4 * w + 0] += acc16[2 * w] & 0xffffu;
        acc.tot[4 * w + 2] += acc16[2 * w] >> 16;
        acc.tot[4 * w + 1] += acc16[2 * w + 1] & 0xffffu;
        acc.tot[4 * w + 3] += acc16[2 * w + 1] >> 16;
        acc16[2 * w] = 0;
        acc16[2 * w + 1] = 0;
      }
    }
  }

  // all bytes [xa, xb) of one plane (xb - xa <= kMaxPiece, so vector offsets fit in 32 bits)
  __device__ __forceinline__ void range(const uint8_t* __restrict__ plane, int64_t xa, int64_t xb,
                                        ScoreAcc<(W > 0 ? W : 1)>& acc) {
    constexpr int WW = W > 0 ? W : 1;
    const int64_t ha = min(xb, (xa + 15) & ~(int64_t)15);
    const int64_t tb = max(ha, xb & ~(int64_t)15);
    for (int64_t x = xa + tid; x < ha; x += nth) one(plane[x], acc);
    for (int64_t x = tb + tid; x < xb; x += nth) one(plane[x], acc);
    const int4* __restrict__ pv = reinterpret_cast<const int4*>(plane + ha);
    const uint32_t nv = (uint32_t)((tb - ha) >> 4);
    const uint32_t T = nth;
    uint32_t acc16[2 * WW];
#pragma unroll
    for (int i = 0; i < 2 * WW; ++i) acc16[i] = 0;
    uint32_t v = tid;
    // main loop: UNROLL vectors in flight per thread, no bounds checks; one thread keeps the
    // CTA's trace region PF_AHEAD iterations ahead prefetched into L2
    const uint32_t step_bytes = UNROLL * T * 16u;
    for (; v + (UNROLL - 1) * T < nv; v += UNROLL * T) {
      constexpr int PF_AHEAD = HIST ? MP_PF_AHEAD : 0;
      if constexpr (PF_AHEAD > 0) {
        if (threadIdx.x == 0) {
          const uint64_t pf = (uint64_t)(v + PF_AHEAD * UNROLL * T) * 16u;
          if (pf + step_bytes <= (uint64_t)nv * 16u) prefetch_l2(reinterpret_cast<const uint8_t*>(pv) + pf, step_bytes);
        }
      }
      int4 x[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) x[u] = ldg_stream(pv + v + u * T);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) vec(x[u], acc16);
      widen(acc16, acc);
    }
    // tail: fewer than UNROLL vectors left for this thread -- guard-free batches of 4 first (several
    // loads per round trip), then single vectors
    if constexpr (UNROLL > 4) {
      for (; v + 3 * T < nv; v += 4 * T) {
        int4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = ldg_stream(pv + v + u * T);
#pragma unroll
        for (int u = 0; u < 4; ++u) vec(x[u], acc16);
        widen(acc16, acc);
      }
    }
    for (; v < nv; v += T) {
      vec(ldg_stream(pv + v), acc16);
      widen(acc16, acc);
    }
  }
};

__device__ __forceinline__ int chunk_of(const int64_t* __restrict__ bounds, int C, int64_t t) {
  // largest c in [0, C) with bounds[c] <= t
  int lo = 0, hi = C;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(bounds + mid) <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// Pieces are capped so one warp's hop sum over a piece fits u32 (64 MB / 16 warps x 255 < 2^32),
// which lets the per-piece flush reduce-scatter u32 values.
constexpr int64_t kMaxPiece = (int64_t)1 << 26;
// Count-contract pieces are capped at 16 MB: a bin total times a u8 cost then fits u32, and so does
// any warp's partial hop sum over a piece (2^24 * 255 < 2^32).
constexpr int64_t kMaxContractPiece = (int64_t)1 << 24;

// WC > 0 selects the count-contract algorithm (requires HIST, W == 0, CHUNKED): the trace is only
// histogrammed, and at every piece flush (one layer x one chunk) the piece's bin totals are
// contracted with the WC-word placement tables: hop_sums[q][c] += sum_e n[e] * pe[q][l][e].  Exact
// by linearity, and the per-byte cost no longer depends on the number of placements.
template <bool HIST, int W, int WIDEN, int UNROLL, bool CHUNKED = false, int WC = 0>
__global__ void __launch_bounds__(kThreads, (W == 4 || W == 2) ? 2 : 3)
stream_kernel(const uint8_t* __restrict__ planes, int64_t stride, int64_t t0, int64_t t1, int L, int K, int E,
              const int64_t* __restrict__ bounds, int C, const uint32_t* __restrict__ tables,
              int64_t* __restrict__ counts, int64_t* __restrict__ hop_sums, int64_t* __restrict__ err) {
  extern __shared__ __align__(128) uint8_t sm[];  // 256 rows x 256 B
  constexpr int WW = W > 0 ? W : 1;
  constexpr int P = 4 * WW;
  const int lane = threadIdx.x & 31;
  Stream<HIST, W, WIDEN, UNROLL> st;
  st.base = smem_addr(sm);
  st.hbase = st.base + 128;
  st.tid = threadIdx.x;
  st.nth = blockDim.x;
  st.slot = W == 4 ? (uint32_t)((lane & 7) << 4) : W == 2 ? (uint32_t)(lane << 3) : (uint32_t)(lane << 2);
  st.hslot = (uint32_t)(lane << 2);
  uint32_t* smw = reinterpret_cast<uint32_t*>(sm);

  // count-contract alternates pieces between two replica sets (set A = bytes 128..255 of each row,
  // set B = bytes 0..127, free since there are no gather tables): a piece's flush reads and zeroes
  // its set while the next piece already counts into the other one, so one barrier per piece
  // suffices and no per-segment zeroing is needed.
  // The per-chunk histogram (CHUNKED, W == 0, WC == 0) alternates the two sets the same way.
  constexpr bool kAltSets = CHUNKED && W == 0;
  int hset = 0;
  // Flushes read a set without zeroing it: each flush thread keeps its 16-replica partial of both
  // sets from the previous flush and reports the difference (exact mod 2^32, and a piece's true
  // count is < 2^32), which halves the flush's shared-memory traffic (L1TEX is the bound).
  uint32_t snap0 = 0u, snap1 = 0u;  // two scalars, not an array: no local memory
  if constexpr (kAltSets) {
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) smw[i] = 0;
  }
  Flat f(t0 * K, t1 * K, L);
  for (int64_t g = f.g0; g < f.g1;) {
    const int l = (int)(g / f.nb);
    const int64_t off_in = g - (int64_t)l * f.nb;
    const int64_t seg = min(f.g1 - g, f.nb - off_in);
    const int64_t x0 = f.b0 + off_in, x1 = x0 + seg;
    const uint8_t* plane = planes + (int64_t)l * stride;

    __syncthreads();  // previous segment is done with shared memory
    if constexpr (W > 0) {
      // row e, word j (< WPR) <- tables[(l*256 + e)*W + j % W]
      constexpr int WPR = (W == 2) ? 64 : 32;
      const uint32_t* tl = tables + (int64_t)l * 256 * W;
      for (int i = threadIdx.x; i < 256 * WPR; i += blockDim.x) {
        const int e = i / WPR, j = i % WPR;
        smw[e * 64 + j] = __ldg(tl + e * W + (j % W));
      }
    }
    if constexpr (HIST && !kAltSets) {
      for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) smw[(i >> 5) * 64 + 32 + (i & 31)] = 0;
    }
    __syncthreads();

    // histogram flush: replica sums of every bin -> dst[l*E + e] (and zero the replicas)
    auto flush_hist = [&](int64_t* dst) {
      for (int e = threadIdx.x; e < 256; e += blockDim.x) {
        uint32_t* row = smw + e * 64 + 32;
        uint32_t s = 0;
#pragma unroll 8
        for (int r = 0; r < 32; ++r) {
          const int rr = (r + e) & 31;  // rotate: no bank conflicts
          s += row[rr];
          if (CHUNKED) row[rr] = 0;
        }
        if (s) {
          if (e < E) atomic_add_i64(dst + (int64_t)l * E + e, (int64_t)s);
          else report_err(err, MP_DATA_EXPERT_RANGE, l, e, s);
        }
      }
    };

    // count-contract flush: two threads per bin (16 replicas each, rotated so a warp's 32 loads hit
    // 32 banks), bin total -> counts (if requested) and x pe of every placement -> hop_sums[q][c]
    constexpr int PC = 4 * (WC > 0 ? WC : 1);
    const int fe = threadIdx.x >> 1, fh = threadIdx.x & 1;
    uint32_t tw[WC > 0 ? WC : 1];
    if constexpr (WC > 0) {
#pragma unroll
      for (int w = 0; w < WC; ++w) tw[w] = fe < 256 ? __ldg(tables + ((int64_t)l * 256 + fe) * WC + w) : 0u;
    }
    // per-chunk histogram flush: the same two threads per bin, bin total -> dst[l*E + e] (set zeroed)
    // bin total of the piece just counted into `set` (two threads per bin, 16 replicas each, rotated so
    // a warp's 32 loads hit 32 banks); valid in the even lane of each pair
    auto piece_bin_total = [&](int set) -> uint32_t {
      uint32_t part = 0;
      if (fe < 256) {
        const uint32_t* row = smw + fe * 64 + (set ? 0 : 32);
#pragma unroll
        for (int i = 0; i < 16; ++i) part += row[(fh * 16 + i + fe) & 31];
      }
#if MP_FLUSH_SNAPSHOT
      const uint32_t d = part - (set ? snap1 : snap0);
      if (set) snap1 = part; else snap0 = part;
#else
      const uint32_t d = part;
      if (fe < 256) {
        uint32_t* row = smw + fe * 64 + (set ? 0 : 32);
#pragma unroll
        for (int i = 0; i < 16; ++i) row[(fh * 16 + i + fe) & 31] = 0;
      }
#endif
      const uint32_t n = d + __shfl_xor_sync(0xffffffffu, d, 1);
      return fh ? 0u : n;  // even lane of each pair owns the bin
    };

    // per-chunk histogram flush: bin total -> dst[l*E + e]
    auto flush_counts = [&](int64_t* dst, int set) {
      const uint32_t n = piece_bin_total(set);
      if (n) {
        if (fe < E) atomic_add_i64(dst + (int64_t)l * E + fe, (int64_t)n);
        else report_err(err, MP_DATA_EXPERT_RANGE, l, fe, n);
      }
    };

    auto flush_contract = [&](int c, int set) {
      const uint32_t n = piece_bin_total(set);
      if (n && counts) {
        if (fe < E) atomic_add_i64(counts + (int64_t)l * E + fe, (int64_t)n);
        else report_err(err, MP_DATA_EXPERT_RANGE, l, fe, n);
      }
      if (__any_sync(0xffffffffu, n != 0)) {
        uint32_t v[PC];
#pragma unroll
        for (int w = 0; w < (WC > 0 ? WC : 1); ++w)
#pragma unroll
          for (int j = 0; j < 4; ++j) v[4 * w + j] = n * ((tw[w] >> (8 * j)) & 0xffu);
        int q = 0;
        const uint32_t tot = warp_reduce_scatter<PC>(v, lane, &q);
        if ((lane & (32 / PC - 1)) == 0 && tot) atomic_add_i64(hop_sums + (int64_t)q * C + c, (int64_t)tot);
      }
    };

    if constexpr (W > 0 || CHUNKED) {
      // chunk of the segment's first byte by binary search, then walk forward (pieces are in order)
      int c = chunk_of(bounds, C, x0 / K);
      int64_t cend = __ldg(bounds + c + 1) * K;
      for (int64_t x = x0; x < x1;) {
        while (cend <= x && c + 1 < C) cend = __ldg(bounds + (++c) + 1) * K;  // skips empty chunks
        const int64_t xe = min(min(x1, cend), x + (WC > 0 ? kMaxContractPiece : kMaxPiece));
        ScoreAcc<WW> acc;
        acc.zero();
        if constexpr (kAltSets) st.hbase = st.base + (hset ? 0u : 128u);
        st.range(plane, x, xe, acc);
        if constexpr (W > 0) {
          int q = 0;
          const uint32_t tot = warp_reduce_scatter<P>(acc.tot, lane, &q);
          if ((lane & (32 / P - 1)) == 0 && tot) atomic_add_i64(hop_sums + (int64_t)q * C + c, (int64_t)tot);
        }
        if constexpr (CHUNKED && WC > 0) {
          __syncthreads();  // every warp's ATOMS into set hset are done
          flush_contract(c, hset);
          hset ^= 1;        // the next piece counts into the other set; no second barrier
        } else if constexpr (CHUNKED) {  // per-chunk histogram: counts is [C][L][E]
          __syncthreads();  // every warp's ATOMS into set hset are done
          flush_counts(counts + (int64_t)c * L * E, hset);
          hset ^= 1;
        }
        x = xe;
      }
    } else {
      ScoreAcc<1> dummy;
      st.range(plane, x0, x1, dummy);
    }

    if constexpr (HIST && !CHUNKED) {
      __syncthreads();
      flush_hist(counts);
    }
    g += seg;
  }
}

constexpr int kSmemBytes = 256 * 256;

template <bool HIST, int W, int WIDEN, bool CHUNKED = false, int WC = 0>
static cudaError_t launch_t(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K, int E,
                            const int64_t* bounds, int C, const uint32_t* tables, int64_t* counts,
                            int64_t* hop_sums, int64_t* err, cudaStream_t s) {
  constexpr int UNROLL = W == 0 ? MP_COUNT_UNROLL : MP_GATHER_UNROLL;  // vectors per thread per iteration
  auto kern = stream_kernel<HIST, W, WIDEN, UNROLL, CHUNKED, WC>;
  int per_sm = 0;
  cudaError_t e = prepare_kernel((const void*)kern, kThreads, kSmemBytes, &per_sm);
  if (e != cudaSuccess) return e;
  const int nsm = device_sm_count();
  if (per_sm < 1) per_sm = 1;
  // grid: persistent, one wave of resident CTAs; small inputs get fewer CTAs
  const int64_t total = (t1 - t0) * (int64_t)K * L;
  int64_t grid = (int64_t)nsm * per_sm;
  const int64_t min_bytes_per_cta = 64 * 1024;
  grid = max((int64_t)1, min(grid, (total + min_bytes_per_cta - 1) / min_bytes_per_cta));
  kern<<<(unsigned)grid, kThreads, kSmemBytes, s>>>(planes, stride, t0, t1, L, K, E, bounds, C, tables, counts,
                                                     hop_sums, err);
  return cudaGetLastError();
}

// ---- pipelined-flush streaming kernel (per-chunk histogram and count-contract) ----------------
// The two-set kernel above needs one CTA barrier per (layer, chunk) piece: every warp waits for the
// slowest one before the piece is flushed.  Here three replica sets rotate and the barrier is split:
// a warp counts piece k into set k%3, then waits for piece k-1's completion (all threads arrived on
// its mbarrier, normally long done), flushes piece k-1 and arrives on piece k's mbarrier.  Arriving
// after the flush makes "phase k complete" imply "set (k-1)%3 flushed", which is what counting
// piece k+2 into that set needs, so warps run up to one piece apart and never idle at a barrier.
// Rows are 128 B (32 lane replicas) per set, so a bin's address is e*128 + set + lane*4 (PRMT byte
// extract + IMAD on the FMA pipe); 3 x 32 KB of sets -> 2 CTAs/SM.
#ifndef MP_PIPE_FLUSH
#define MP_PIPE_FLUSH 1
#endif
#ifndef MP_PIPE_GTAIL4
#define MP_PIPE_GTAIL4 1  // guarded 4-vector tail batches (C = 3000: hist_chunks 1.905 -> 1.472, W = 4 pass 2.10 -> 1.80 ms)
#endif
// MP_PIPE_SPLIT (default): one CTA of 1024 threads per SM made of two independent 512-thread halves
// whose sets interleave in 256-byte rows (half h at bytes h*128..h*128+127 of row e), so the bins of
// one warp's ATOMS are 256 B apart and share address bit 7.  microbench9 (i.i.d. Zipf bytes,
// profiles/r2_microbench9_atoms_pitch.txt): 128-byte pitch 0.763 ms per 4.64 GB, 256-byte pitch
// 0.731 ms.  In this kernel the gain is smaller (fused step 0.854 -> 0.846 ms, W = 4 at C = 1500
// 1.329 -> 1.238; hist+8 placements at C = 150 0.870 -> 0.901), and ncu's aggregate ATOMS conflict
// counter stays at ~18 % of ATOMS while the per-instruction source view shows ideal wavefronts.
// Occupancy is unchanged (32 warps per SM).  MP_PIPE_SPLIT=0 builds the 2 x 512-thread CTA kernel.
#ifndef MP_PIPE_SPLIT
#define MP_PIPE_SPLIT 1
#endif
// Replica sets per worker: 3 rotate with one piece of slack between warps; 2 need a wait per piece
// (piece k reuses piece k-2's set) but fit below 128 KB of shared memory, where shared atomics are
// fast -- sets placed above ~96 KB of the allocation count ~40 % extra ATOMS wavefronts and run
// ~30 % slower (tools/microbench11.cu, profiles/r2_smem_atoms.txt).  The launcher takes 2 sets for
// pieces of >= kTwoSetPiece bytes on average (R1 10M / 150 chunks, 533 KB pieces: fused step
// 0.845 -> 0.805 ms) and 3 for shorter ones (1500 chunks: 1.215 vs 1.335 ms with 2 sets).
constexpr int kPipeHalves = MP_PIPE_SPLIT ? 2 : 1;  // workers per CTA (count-contract, per-chunk histogram)
// A CTA of HALVES workers of WT threads; one set = 256 expert rows of HALVES x 128 bytes (worker h's
// 32 lane replicas at bytes h*128 .. h*128+127 of each row).
template <int WT, int HALVES>
struct PipeShape {
  static constexpr int kWT = WT, kHalves = HALVES, kThreads = WT * HALVES;
  static constexpr int kRow = 128 * HALVES;
  static constexpr int kSetBytes = 256 * kRow;
};
using PipeCC = PipeShape<kThreads, kPipeHalves>;  // count-contract / per-chunk histogram: 2 x 512 threads
// ONE 1024-thread worker whose three 32 KB sets all sit below 96 KB of shared memory: the plain
// histogram (one chunk: a handful of flushes; 0.769 -> 0.726 ms for 10M R1 tokens, 98.9 % of HBM)
// and the chunked instances when their pieces average >= kSingleWorkerPiece, there with the two
// halves staggered (see launch_pipe).  With short pieces the single worker is slower (one piece at
// a time for the whole SM: 1500 chunks 1.20 -> 1.57 ms), so those keep two 512-thread workers
// (profiles/r2_pipe_workers.txt, r2_pipe_single_stagger.txt).
using PipeHist = PipeShape<1024, 1>;

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}

// ATOMS increments for bytes [xa, xb) of one plane by the T threads of a worker; sb = shared address
// of this lane's replica of bin 0 in the piece's set (bin e at sb + e * ROW)
template <int UNROLL, uint32_t T, uint32_t ROW>
__device__ __forceinline__ void pipe_count(const uint8_t* __restrict__ plane, int64_t xa, int64_t xb, uint32_t sb,
                                           uint32_t tid) {
  const int64_t ha = min(xb, (xa + 15) & ~(int64_t)15);
  const int64_t tb = max(ha, xb & ~(int64_t)15);
  // the < 16 unaligned bytes at each end (one per thread, T >= 16): loaded now, counted after the
  // vectors -- counting them first put two dependent load round trips ahead of warp 0's vector
  // loads at every piece, and the pipelined flush then waited for warp 0 every piece
  // packed into one register (bits 0-8 head, 16-24 tail; 0x100 = none) to stay off the loop's budget
  const uint32_t ends = (xa + tid < ha ? (uint32_t)__ldg(plane + xa + tid) : 0x100u) |
                        ((tb + tid < xb ? (uint32_t)__ldg(plane + tb + tid) : 0x100u) << 16);
  const int4* __restrict__ pv = reinterpret_cast<const int4*>(plane + ha);
  const uint32_t nv = (uint32_t)((tb - ha) >> 4);
  auto vec = [&](const int4& x) {
    const uint32_t wd[4] = {(uint32_t)x.x, (uint32_t)x.y, (uint32_t)x.z, (uint32_t)x.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int b = 0; b < 4; ++b) atoms_inc(prmt(wd[q], 0u, 0x4440u | (uint32_t)b) * ROW + sb);
  };
  uint32_t v = tid;
  for (; v + (UNROLL - 1) * T < nv; v += UNROLL * T) {
    int4 x[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) x[u] = ldg_stream(pv + v + u * T);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) vec(x[u]);
  }
#if MP_PIPE_GTAIL4
  // tail: guarded batches of 4 (a short piece's rest in one or two load round trips)
  for (; v < nv; v += 4 * T) {
    int4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = v + u * T < nv ? ldg_stream(pv + v + u * T) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v + u * T < nv) vec(x[u]);
  }
#else
  for (; v + 3 * T < nv; v += 4 * T) {
    int4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = ldg_stream(pv + v + u * T);
#pragma unroll
    for (int u = 0; u < 4; ++u) vec(x[u]);
  }
  for (; v < nv; v += T) vec(ldg_stream(pv + v));
#endif
  if (!(ends & 0x100u)) atoms_inc(sb + (ends & 0xffu) * ROW);
  if (!(ends & 0x1000000u)) atoms_inc(sb + ((ends >> 16) & 0xffu) * ROW);
}

// WC == 0: per-chunk histogram, counts is int64 [C][L][E].  WC > 0: count-contract with WC-word
// tables; counts (nullable) is int64 [L][E] and hop_sums int64 [4*WC][C].
template <int WC, int UNROLL, int kPipeSets, class Shape>
__global__ void __launch_bounds__(Shape::kThreads, 1024 / Shape::kThreads)
pipe_kernel(const uint8_t* __restrict__ planes, int64_t stride, int64_t t0, int64_t t1, int L, int K, int E,
            const int64_t* __restrict__ bounds, int C, const uint32_t* __restrict__ tables,
            int64_t* __restrict__ counts, int64_t* __restrict__ hop_sums, int64_t* __restrict__ err,
            unsigned stagger_ns) {
  constexpr int kPipeWT = Shape::kWT, kPipeHalves = Shape::kHalves;
  constexpr int kPipeRow = Shape::kRow, kPipeSetBytes = Shape::kSetBytes;
  extern __shared__ __align__(128) uint8_t sm[];  // kPipeSets x 256 rows x kPipeRow B
  __shared__ __align__(8) uint64_t bar[kPipeHalves][kPipeSets];
  constexpr int PC = 4 * (WC > 0 ? WC : 1);
  const int lane = threadIdx.x & 31;
  const int half = kPipeHalves > 1 ? (int)(threadIdx.x / kPipeWT) : 0;  // independent workers
  const uint32_t tid = threadIdx.x & (kPipeWT - 1);
  const uint32_t base0 = smem_addr(sm);
  const uint32_t bar0 = smem_addr(&bar[half][0]);
  uint32_t* smw = reinterpret_cast<uint32_t*>(sm) + half * 32;
  for (int i = threadIdx.x; i < kPipeSets * kPipeSetBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (tid == 0)
    for (int b = 0; b < kPipeSets; ++b) mbar_init(bar0 + 8 * b, kPipeWT);
  __syncthreads();
  // one 1024-thread worker: its upper half starts stagger_ns later, so the halves reach the piece
  // boundaries (where a warp's loads have drained) out of phase and the SM keeps loads in flight
  // (they may drift apart by up to a piece: the pipelined flush allows it)
  if (stagger_ns && tid >= (uint32_t)kPipeWT / 2) __nanosleep(stagger_ns);

  // flush roles: two threads per bin (16 replicas each, rotated: a warp's 32 loads hit 32 banks)
  const int fe = (int)(tid >> 1), fh = (int)(tid & 1);
  uint32_t snap[kPipeSets];
#pragma unroll
  for (int b = 0; b < kPipeSets; ++b) snap[b] = 0u;
  // piece k-1 awaiting its flush
  int pk = -1, pl = 0, pc = 0;
  // table words of piece k-1 held in registers for WC <= 4; WC = 8 reads them at the flush (L1)
  // instead, which would otherwise pin 16 registers across the count loop at the 64-register budget
  // (reading at the flush for every WC cost 5 % with short pieces: 1500 chunks 1.22 -> 1.28 ms)
  constexpr bool kRegTables = WC > 0 && WC <= 4;
  uint32_t ptw[kRegTables ? WC : 1];
  auto flush_prev = [&]() {
    const int set = pk % kPipeSets;
    mbar_wait(bar0 + 8 * set, (uint32_t)((pk / kPipeSets) & 1));  // every thread finished counting piece pk
    uint32_t part = 0;
    if (fe < 256) {
      const uint32_t* row = smw + set * (kPipeSetBytes / 4) + fe * (kPipeRow / 4);
#pragma unroll
      for (int i = 0; i < 16; ++i) part += row[(fh * 16 + i + fe) & 31];
    }
    uint32_t prev = snap[0];
#pragma unroll
    for (int b = 1; b < kPipeSets; ++b)
      if (set == b) prev = snap[b];
#pragma unroll
    for (int b = 0; b < kPipeSets; ++b)
      if (set == b) snap[b] = part;
    const uint32_t d = part - prev;  // exact mod 2^32: the piece's count is < 2^32
    uint32_t n = d + __shfl_xor_sync(0xffffffffu, d, 1);
    if (fh) n = 0;  // even lane of each pair owns the bin
    if constexpr (WC == 0) {
      if (n) {
        if (fe < E) atomic_add_i64(counts + ((int64_t)pc * L + pl) * E + fe, (int64_t)n);
        else report_err(err, MP_DATA_EXPERT_RANGE, pl, fe, n);
      }
    } else {
      if (n && counts) {
        if (fe < E) atomic_add_i64(counts + (int64_t)pl * E + fe, (int64_t)n);
        else report_err(err, MP_DATA_EXPERT_RANGE, pl, fe, n);
      }
      if (__any_sync(0xffffffffu, n != 0)) {
        const uint32_t* tp = tables + ((int64_t)pl * 256 + (fe < 256 ? fe : 0)) * WC;
        uint32_t v[PC];
#pragma unroll
        for (int w = 0; w < WC; ++w) {
          uint32_t tw;
          if constexpr (kRegTables) tw = ptw[w < WC ? w : 0];
          else tw = n ? __ldg(tp + w) : 0u;
#pragma unroll
          for (int j = 0; j < 4; ++j) v[4 * w + j] = n * ((tw >> (8 * j)) & 0xffu);
        }
        int q = 0;
        const uint32_t tot = warp_reduce_scatter<PC>(v, lane, &q);
        if ((lane & (32 / PC - 1)) == 0 && tot) atomic_add_i64(hop_sums + (int64_t)q * C + pc, (int64_t)tot);
      }
    }
  };

  int k = 0;  // this (half-)CTA's piece counter
  Flat f(t0 * K, t1 * K, L, (int)blockIdx.x * kPipeHalves + half, (int)gridDim.x * kPipeHalves);
  for (int64_t g = f.g0; g < f.g1;) {
    const int l = (int)(g / f.nb);
    const int64_t off_in = g - (int64_t)l * f.nb;
    const int64_t seg = min(f.g1 - g, f.nb - off_in);
    const int64_t x0 = f.b0 + off_in, x1 = x0 + seg;
    const uint8_t* plane = planes + (int64_t)l * stride;
    uint32_t tw[kRegTables ? WC : 1];
    if constexpr (kRegTables) {
#pragma unroll
      for (int w = 0; w < WC; ++w) tw[w] = fe < 256 ? __ldg(tables + ((int64_t)l * 256 + fe) * WC + w) : 0u;
    }
    // bounds == nullptr: the whole range is one chunk (mp_hist_u8: counts is [L][E])
    int c = bounds ? chunk_of(bounds, C, x0 / K) : 0;
    int64_t cend = bounds ? __ldg(bounds + c + 1) * K : INT64_MAX;
    for (int64_t x = x0; x < x1;) {
      while (cend <= x && c + 1 < C) cend = __ldg(bounds + (++c) + 1) * K;  // skips empty chunks
      const int64_t xe = min(min(x1, cend), x + (WC > 0 ? kMaxContractPiece : kMaxPiece));
      const int set = k % kPipeSets;
      if constexpr (kPipeSets == 2) {  // piece k reuses piece k-2's set: every thread must have flushed it
        if (k >= 2) mbar_wait(bar0 + 8 * ((k - 1) % 2), (uint32_t)(((k - 1) / 2) & 1));
      }
      pipe_count<UNROLL, (uint32_t)kPipeWT, (uint32_t)kPipeRow>(plane, x, xe, base0 + (uint32_t)(set * kPipeSetBytes + half * 128 + (lane << 2)), tid);
      if (pk >= 0) flush_prev();
      mbar_arrive(bar0 + 8 * set);  // counted piece k, flushed piece k-1
      pk = k++;
      pl = l;
      pc = c;
      if constexpr (kRegTables) {
#pragma unroll
        for (int w = 0; w < WC; ++w) ptw[w] = tw[w];
      }
      x = xe;
    }
    g += seg;
  }
  if (pk >= 0) flush_prev();
}

constexpr int64_t kTwoSetPiece = 128 * 1024;  // crossover measured between 133 KB (C = 600) and 89 KB
// Long pieces: ONE 1024-thread worker per SM whose three 32 KB sets sit below 96 KB, its halves
// staggered by kStaggerNs (R1 10M: C = 150 / 533 KB pieces: fused step 0.809 -> 0.781 ms, C = 50:
// 0.755 -> 0.692 ms; at C = 300 / 267 KB pieces two 512-thread workers stay faster, 0.878 vs 0.901;
// profiles/r2_pipe_single_stagger.txt)
constexpr int64_t kSingleWorkerPiece = 400 * 1024;
constexpr unsigned kStaggerNs = 4000;

template <int WC, int SETS, class Shape = PipeCC>
static cudaError_t launch_pipe_t(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K, int E,
                                 const int64_t* bounds, int C, const uint32_t* tables, int64_t* counts,
                                 int64_t* hop_sums, int64_t* err, cudaStream_t s, unsigned stagger_ns = 0) {
  auto kern = pipe_kernel<WC, MP_COUNT_UNROLL, SETS, Shape>;
  constexpr int smem = SETS * Shape::kSetBytes;
  int per_sm = 0;
  cudaError_t e = prepare_kernel((const void*)kern, Shape::kThreads, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const int nsm = device_sm_count();
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 1024 / Shape::kThreads) per_sm = 1024 / Shape::kThreads;  // 1024 threads per SM
  const int64_t total = (t1 - t0) * (int64_t)K * L;
  int64_t grid = (int64_t)nsm * per_sm;
  const int64_t min_bytes_per_cta = 64 * 1024 * Shape::kHalves;
  grid = max((int64_t)1, min(grid, (total + min_bytes_per_cta - 1) / min_bytes_per_cta));
  kern<<<(unsigned)grid, Shape::kThreads, smem, s>>>(planes, stride, t0, t1, L, K, E, bounds, C, tables, counts,
                                                     hop_sums, err, stagger_ns);
  return cudaGetLastError();
}

// {span, non-empty chunks} of a chunk-bounds array, written to host-mapped memory
__global__ void chunk_stats_kernel(const int64_t* __restrict__ bounds, int C, int64_t* out) {
  __shared__ int part[32];
  int n = 0;
  for (int i = threadIdx.x; i < C; i += blockDim.x) n += __ldg(bounds + i + 1) > __ldg(bounds + i);
  n = __reduce_add_sync(0xffffffffu, n);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    out[0] = __ldg(bounds + C) - __ldg(bounds);
    out[1] = t;
  }
}

// Average bytes per NON-EMPTY (layer, chunk) piece, which picks the kernel shape (results never
// depend on it).  (t1 - t0) * K / C is right for a whole trace, but a shard of a larger trace keeps
// every chunk of the global bounds, clipped (rank r of G sees C / G non-empty chunks), which would
// make the pieces look G times shorter.  So the first call with a given bounds array launches a
// one-block kernel on the launch stream that counts the non-empty chunks into host-mapped memory;
// later calls use that count once its event has completed (a query, never a wait).  Entries are
// keyed by (device, pointer, C); a reused pointer with other contents can only cost speed.
static int64_t avg_piece_bytes(const int64_t* bounds, int C, int64_t t0, int64_t t1, int K, cudaStream_t s) {
  const int64_t est = (t1 - t0) * (int64_t)K / (bounds ? C : 1);
  if (!bounds || C <= 1) return est;
  constexpr int kSlots = 256;
  struct Entry {
    int slot;
    cudaEvent_t ev;
  };
  static std::mutex mu;
  static std::map<std::tuple<int, const int64_t*, int>, Entry> cache;
  static int64_t* pool = nullptr;  // host-mapped, 2 words per slot
  static int used = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  const auto key = std::make_tuple(dev, bounds, C);
  auto it = cache.find(key);
  if (it != cache.end()) {
    if (cudaEventQuery(it->second.ev) != cudaSuccess) {
      cudaGetLastError();  // not ready yet
      return est;
    }
    const volatile int64_t* h = pool + 2 * it->second.slot;
    const int64_t span = h[0], nonempty = h[1];
    return (span > 0 && nonempty > 0) ? span * (int64_t)K / nonempty : est;
  }
  if (!pool && cudaHostAlloc((void**)&pool, 2 * kSlots * sizeof(int64_t), cudaHostAllocMapped | cudaHostAllocPortable) !=
                   cudaSuccess) {
    cudaGetLastError();
    pool = nullptr;
    return est;
  }
  if (used == kSlots) {  // bounded: start over (the next calls re-count)
    for (auto& kv : cache) {
      cudaEventSynchronize(kv.second.ev);
      cudaEventDestroy(kv.second.ev);
    }
    cache.clear();
    used = 0;
  }
  Entry e{used, nullptr};
  int64_t* d = nullptr;
  if (cudaHostGetDevicePointer((void**)&d, pool + 2 * e.slot, 0) != cudaSuccess ||
      cudaEventCreateWithFlags(&e.ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    if (e.ev) cudaEventDestroy(e.ev);
    return est;
  }
  chunk_stats_kernel<<<1, 256, 0, s>>>(bounds, C, d);
  if (cudaGetLastError() != cudaSuccess || cudaEventRecord(e.ev, s) != cudaSuccess) {
    cudaGetLastError();
    cudaEventDestroy(e.ev);
    return est;
  }
  ++used;
  cache.emplace(key, e);
  return est;
}

template <int WC>
static cudaError_t launch_pipe(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K, int E,
                               const int64_t* bounds, int C, const uint32_t* tables, int64_t* counts,
                               int64_t* hop_sums, int64_t* err, cudaStream_t s) {
  const int64_t piece = avg_piece_bytes(bounds, C, t0, t1, K, s);  // average (layer, chunk) piece
  if (piece >= kSingleWorkerPiece)  // one 1024-thread worker, three 32 KB sets, staggered halves
    return launch_pipe_t<WC, 3, PipeHist>(planes, stride, t0, t1, L, K, E, bounds, C, tables, counts, hop_sums, err, s,
                                          kStaggerNs);
#ifdef MP_PIPE_FORCE_SETS
  if (MP_PIPE_FORCE_SETS == 2)
#else
  if (piece >= kTwoSetPiece)
#endif
    return launch_pipe_t<WC, 2>(planes, stride, t0, t1, L, K, E, bounds, C, tables, counts, hop_sums, err, s);
  return launch_pipe_t<WC, 3>(planes, stride, t0, t1, L, K, E, bounds, C, tables, counts, hop_sums, err, s);
}

cudaError_t launch_hist_chunks(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K, int E,
                               const int64_t* bounds, int C, int64_t* counts, int64_t* err, cudaStream_t s) {
#if MP_PIPE_FLUSH
  return launch_pipe<0>(planes, stride, t0, t1, L, K, E, bounds, C, nullptr, counts, nullptr, err, s);
#else
  return launch_t<true, 0, 16, true>(planes, stride, t0, t1, L, K, E, bounds, C, nullptr, counts, nullptr, err, s);
#endif
}

// ---- exact contraction of per-chunk counts with per-expert costs (factorized evaluator) ----
// out[q*C + c] += sum_i counts[c*LE + i] * pe[q*LE + i]; tiles of 64 placements x 16 chunks,
// LE streamed in 128-wide slices through shared memory; int64 accumulation (exact).
constexpr int kCtP = 64, kCtC = 16, kCtI = 128;

__global__ void __launch_bounds__(256) contract_kernel(const int64_t* __restrict__ counts, int C,
                                                       const uint8_t* __restrict__ pe, int P, int64_t LE,
                                                       int64_t* __restrict__ out) {
  __shared__ uint8_t s_pe[kCtP][kCtI];
  __shared__ int32_t s_cnt[kCtC][kCtI + 1];
  const int q0 = blockIdx.x * kCtP, c0 = blockIdx.y * kCtC;
  const int tq = threadIdx.x & 63;   // placement within tile
  const int tc = threadIdx.x >> 6;   // 4 chunk lanes: chunks tc, tc+4, tc+8, tc+12
  int64_t acc[4] = {0, 0, 0, 0};
  for (int64_t i0 = 0; i0 < LE; i0 += kCtI) {
    __syncthreads();
    for (int k = threadIdx.x; k < kCtP * kCtI; k += blockDim.x) {
      const int qq = k / kCtI, ii = k % kCtI;
      s_pe[qq][ii] = (q0 + qq < P && i0 + ii < LE) ? pe[(int64_t)(q0 + qq) * LE + i0 + ii] : 0;
    }
    for (int k = threadIdx.x; k < kCtC * kCtI; k += blockDim.x) {
      const int cc = k / kCtI, ii = k % kCtI;
      s_cnt[cc][ii] = (c0 + cc < C && i0 + ii < LE) ? (int32_t)counts[(int64_t)(c0 + cc) * LE + i0 + ii] : 0;
    }
    __syncthreads();
#pragma unroll 4
    for (int ii = 0; ii < kCtI; ++ii) {
      const int32_t w = s_pe[tq][ii];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] += (int64_t)w * s_cnt[tc + 4 * j][ii];
    }
  }
  if (q0 + tq < P)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tc + 4 * j;
      if (c < C && acc[j]) atomic_add_i64(out + (int64_t)(q0 + tq) * C + c, acc[j]);
    }
}

cudaError_t launch_contract(const int64_t* counts, int C, const uint8_t* pe, int P, int64_t LE, int64_t* out,
                            cudaStream_t s) {
  if (P <= 0 || C <= 0 || LE <= 0) return cudaSuccess;
  dim3 grid((unsigned)((P + kCtP - 1) / kCtP), (unsigned)((C + kCtC - 1) / kCtC));
  contract_kernel<<<grid, 256, 0, s>>>(counts, C, pe, P, LE, out);
  return cudaGetLastError();
}

// Which exact algorithm computes the hop sums: the per-byte gather costs one LDS per
// lookup (1/2/4 wavefronts per 32 lookups for W = 1/2/4) on top of the histogram's ATOMS when both are
// needed; count-contract costs only the histogram.  Measured (R1, 10M tokens): gather W=1 0.80 ms,
// W=2 1.25, W=4 2.25, fused hist+gather 1.36; count-contract 0.91-0.93 for any W, with or without counts.
// Token-tiled wins below a per-shape tokens-per-chunk threshold (R1, 10M tokens, crossovers measured
// in profiles/r1_chunk_granularity.txt): its cost is flat in C but grows with W (1.31 / 2.61 / 5.2 ms
// for W = 1 / 2 / 4, + 0.83 ms histogram), while the streaming algorithms pay per (layer, chunk) piece.
int token_threshold(bool hist, int W) {
  if (W <= 1) return hist ? MP_TOKEN_CHUNK_TOKENS : 2 * MP_TOKEN_CHUNK_TOKENS - 1024;  // 2560 / 4096
  if (W == 2) return hist ? MP_TOKEN_CHUNK_TOKENS / 2 : 1600;                         // 1280 / 1600
  return hist ? 700 : 800;
}

int choose_algo(bool hist, int W, int algo, int64_t tokens, int C, int L, int K, int max_p) {
  if (algo != MP_ALGO_AUTO) return algo;
  if (W == 8) return MP_ALGO_COUNT;  // 32 placements per pass: the count-contract kernel only
  const bool tok_ok = (int64_t)L * K * max_p <= 65535;
  // Segmented gather (K = 8, max_p <= 31; with a histogram W = 1): C-independent and cheaper than
  // the token walk for W >= 2 and for the fused pass, so it takes the short-chunk range from
  // MP_SEG_CHUNK_TOKENS down to where the token walk's flat cost wins again (crossovers measured
  // at R1, profiles/r1_chunk_granularity.txt).
  if (K == 8 && max_p <= 31) {
    // SEG below seg_hi tokens per chunk, TOKEN below tok_lo (R1, 10M tokens, forced algorithms,
    // after the redux.sync flush; profiles/r2_crossovers.txt): hist+W=1 count 1.300 / seg 1.310 ms
    // at 5000 tokens per chunk, 1.220 / 1.308 at 6667; the token walk (2.13 ms) never wins with a
    // histogram; score W=1 seg 0.770 / gather 0.774 at 33,333 tokens per chunk, seg 1.20 vs token
    // 1.32 at 67 and 1.04 vs 1.32 at 100 (seg ~ 0.77 + 28 / tokens-per-chunk ms: even at ~50);
    // W=2 count 1.185 / seg 1.222 at 6667, 1.302 / 1.227 at 5000; W=4 count 1.929 / 2.433 vs seg
    // 2.31 at 3333 / 2000; hist+W=2 count 1.836 vs seg 1.794 at 3000; hist+W=4 count ~0.88 + 3240 /
    // tokens-per-chunk vs seg 3.03: even at ~1500.
    const int seg_hi = hist ? (W == 1 ? 5000 : W == 2 ? 3000 : 1500) : W == 1 ? 40000 : W == 2 ? 6000 : 2400;
    const int tok_lo = hist ? 0 : W == 1 ? 50 : 0;
    if (tok_ok && tokens < (int64_t)tok_lo * C) return MP_ALGO_TOKEN;
    if (tokens < (int64_t)seg_hi * C) return MP_ALGO_SEG;
    return (hist || W > 1) ? MP_ALGO_COUNT : MP_ALGO_GATHER;
  }
  if (tokens < (int64_t)token_threshold(hist, W) * C && tok_ok) return MP_ALGO_TOKEN;
  return (hist || W > 1) ? MP_ALGO_COUNT : MP_ALGO_GATHER;
}

cudaError_t launch_score_tok(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K,
                             const int64_t* bounds, int C, const uint32_t* tables, int W, int max_p, int64_t* hop_sums,
                             cudaStream_t s);
cudaError_t launch_seg(bool hist, int W, const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int E,
                       const int64_t* bounds, int C, const uint32_t* tables, int64_t* counts, int64_t* hop_sums,
                       int64_t* err, cudaStream_t s);

cudaError_t launch_stream(bool hist, int W, int max_p, const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1,
                          int L, int K, int E, const int64_t* bounds, int C, const uint32_t* tables, int64_t* counts,
                          int64_t* hop_sums, int64_t* err, cudaStream_t s, int algo) {
#define MP_ARGS planes, stride, t0, t1, L, K, E, bounds, C, tables, counts, hop_sums, err, s
  const int widen = max_p <= 15 ? 16 : max_p <= 63 ? 4 : 1;
  // plain histogram: the pipelined-flush kernel with the whole range as one chunk (pieces end only at
  // layer ends): 0.836 -> 0.754 ms for 10M R1 tokens against the two-set streaming kernel, 0.726 ms
  // with one 1024-thread worker per SM
#if MP_PIPE_FLUSH
  if (W == 0)  // one 1024-thread worker, three 32 KB sets (PipeHist)
    return launch_pipe_t<0, 3, PipeHist>(planes, stride, t0, t1, L, K, E, nullptr, 1, nullptr, counts, nullptr, err, s);
#else
  if (W == 0) return launch_hist_chunks(planes, stride, t0, t1, L, K, E, nullptr, 1, counts, err, s);
#endif
  // AUTO decides by tokens per chunk; a shard of a larger trace carries the global (clipped) chunk
  // list, so count only its non-empty chunks (avg_piece_bytes: cached, never waits)
  int C_eff = C;
  if (algo == MP_ALGO_AUTO && bounds && C > 1 && K > 0) {
    const int64_t piece = avg_piece_bytes(bounds, C, t0, t1, K, s);
    if (piece > 0) C_eff = (int)std::max<int64_t>(1, std::min<int64_t>(C, (t1 - t0) * K / piece));
  }
  const int chosen = choose_algo(hist, W, algo, t1 - t0, C_eff, L, K, max_p);
  if (chosen == MP_ALGO_SEG)
    return launch_seg(hist, W, planes, stride, t0, t1, L, E, bounds, C, tables, counts, hop_sums, err, s);
  if (chosen == MP_ALGO_TOKEN) {
    if (hist) {  // histogram pass (per-layer flushes only) + the token-tiled scorer
      const cudaError_t e = launch_t<true, 0, 16>(planes, stride, t0, t1, L, K, E, nullptr, 1, nullptr, counts, nullptr,
                                                   err, s);
      if (e != cudaSuccess) return e;
    }
    return launch_score_tok(planes, stride, t0, t1, L, K, bounds, C, tables, W, max_p, hop_sums, s);
  }
  if (chosen == MP_ALGO_COUNT) {
    if (!hist) counts = nullptr;  // histogram stays in shared memory
#if MP_PIPE_FLUSH
    if (W == 1) return launch_pipe<1>(MP_ARGS);
    if (W == 2) return launch_pipe<2>(MP_ARGS);
    if (W == 4) return launch_pipe<4>(MP_ARGS);
    if (W == 8) return launch_pipe<8>(MP_ARGS);
#else
    if (W == 1) return launch_t<true, 0, 16, true, 1>(MP_ARGS);
    if (W == 2) return launch_t<true, 0, 16, true, 2>(MP_ARGS);
    if (W == 4) return launch_t<true, 0, 16, true, 4>(MP_ARGS);
#endif
    return cudaErrorInvalidValue;
  }
  if (hist) {
    if (W == 1) {
      if (widen == 16) return launch_t<true, 1, 16>(MP_ARGS);
      if (widen == 4) return launch_t<true, 1, 4>(MP_ARGS);
      return launch_t<true, 1, 1>(MP_ARGS);
    }
    return cudaErrorInvalidValue;
  }
  if (W == 1) {
    if (widen == 16) return launch_t<false, 1, 16>(MP_ARGS);
    if (widen == 4) return launch_t<false, 1, 4>(MP_ARGS);
    return launch_t<false, 1, 1>(MP_ARGS);
  }
  if (W == 2) {
    if (widen == 16) return launch_t<false, 2, 16>(MP_ARGS);
    if (widen == 4) return launch_t<false, 2, 4>(MP_ARGS);
    return launch_t<false, 2, 1>(MP_ARGS);
  }
  if (W == 4) {
    if (widen == 16) return launch_t<false, 4, 16>(MP_ARGS);
    if (widen == 4) return launch_t<false, 4, 4>(MP_ARGS);
    return launch_t<false, 4, 1>(MP_ARGS);
  }
#undef MP_ARGS
  return cudaErrorInvalidValue;
}

}  // namespace mp
