// Segmented gather (MP_ALGO_SEG): per-chunk hop sums whose cost does not depend on the chunk count,
// as a layer-major stream (no per-layer table re-staging per token tile, unlike the token-tiled
// scorer).  K = 8, max_p <= 31.
//
// A CTA walks its byte range plane segment by plane segment like the streaming kernels and stages
// the layer's W-word table replicated per lane slot (conflict-free PRMT-addressed lookups).  The
// segment's tokens are then split into 32 contiguous warp sub-ranges; a warp streams its
// sub-range in windows of 64 tokens (one 16-byte vector = two 8-pick records per lane, four
// windows in flight) and keeps running per-lane sums of the current chunk.  Chunk boundaries are
// detected per window from the chunk bounds (warp-uniform): the tokens before the boundary are
// added, the warp sums its running sums (redux.sync) and adds them to hop_sums[q][c] (one int64
// atomic per placement), and the sums restart for the next chunk.  The streaming kernels instead
// spread every (layer, chunk) piece over the whole CTA, so short chunks leave most threads idle;
// here a boundary costs one warp reduction wherever it falls.
// Per-token sums of 8 lookups fit u8 lanes (8 * 31 < 256); running sums are u16 lanes widened
// into u32 every 64 windows and at each flush.  With HIST every byte also increments the
// lane-replicated histogram (W = 1: in the table rows' free half, one PRMT per address; W = 2 / 4:
// a separate region of 128-byte rows, PRMT byte extract + IMAD), flushed per segment.
#include <type_traits>

#include "common.cuh"

namespace mp {

// One 1024-thread CTA per SM: its tables + histogram (64 / 96 KB) stay below the upper part of the
// shared-memory carve-out, where atomics run ~30 % slower (profiles/r2_smem_atoms.txt); two 512-thread
// CTAs put the second one's there.  140 tokens per chunk: fused 1.387 -> 1.322 ms, hist + W = 2
// 1.929 -> 1.816, hist + W = 4 3.267 -> 3.171, score W = 1 0.950 -> 0.928 (profiles/r2_seg_cta1024.txt).
#ifndef MP_SEG_THREADS
#define MP_SEG_THREADS 1024
#endif
constexpr int kSegThreads = MP_SEG_THREADS;
constexpr int kSegWarps = kSegThreads / 32;
// windows in flight per warp for W = 1 (R1 10M tokens, 4 placements, 1500 / 15k / 150k chunks):
// 2: 1.035 / 1.112 / 1.895 ms, 4: 0.985 / 1.052 / 1.841 ms, 8: 1.014 / 1.087 / 1.853 ms (spills)
#ifndef MP_SEG_U1
#define MP_SEG_U1 4
#endif
template <int W>
__host__ __device__ constexpr int seg_unroll() { return W == 4 ? 2 : W == 2 ? 4 : MP_SEG_U1; }  // windows (64 tokens) in flight per warp

template <int W>
__device__ __forceinline__ void seg_lookup(uint32_t a, uint32_t (&t)[W]) {
  if constexpr (W == 1) {
    t[0] = lds32(a);
  } else if constexpr (W == 2) {
    const uint2 v = lds64(a);
    t[0] = v.x; t[1] = v.y;
  } else {
    const uint4 v = lds128(a);
    t[0] = v.x; t[1] = v.y; t[2] = v.z; t[3] = v.w;
  }
}

template <int W, bool HIST>
__global__ void __launch_bounds__(kSegThreads, 1024 / kSegThreads)
seg_kernel(const uint8_t* __restrict__ planes, int64_t stride, int64_t t0, int64_t t1, int L, int E,
           const int64_t* __restrict__ bounds, int C, const uint32_t* __restrict__ tables,
           int64_t* __restrict__ counts, int64_t* __restrict__ hop_sums, int64_t* __restrict__ err) {
  constexpr int P = 4 * W;
  constexpr int U = seg_unroll<W>();
  // 256 rows x 256 B of tables (W = 1: bytes 128-255 of each row hold the histogram replicas);
  // W > 1 with HIST: + a 256 rows x 128 B histogram region; then a 128-byte trash row
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr bool kHistRegion = HIST && W > 1;
  constexpr int kHistWords = 256 * 256 / 4;  // word offset of the separate histogram region
  uint32_t* smw = reinterpret_cast<uint32_t*>(sm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = smem_addr(sm);
  const uint32_t slot = W == 4 ? (uint32_t)((lane & 7) << 4) : W == 2 ? (uint32_t)(lane << 3) : (uint32_t)(lane << 2);
  const uint32_t hslot = (uint32_t)(lane << 2);
  const uint32_t hreg = base + 256 * 256 + hslot;  // W > 1: bin e of this lane at hreg + e * 128
  const uint32_t trash = base + 256 * 256 + (kHistRegion ? 256 * 128 : 0) + hslot;  // masked-out tokens

  // running sums of the current chunk in u16 lanes (acc16[2w] = placements {4w, 4w+2}, acc16[2w+1] =
  // {4w+1, 4w+3}); they are widened only inside a flush, which runs at every chunk boundary and
  // at least every 128 windows (128 x 2 tokens x 248 < 2^16), so no u32 sums stay live
  uint32_t acc16[2 * W];
#pragma unroll
  for (int i = 0; i < 2 * W; ++i) acc16[i] = 0;
  // two tokens' u8-lane sums into the u16 lanes: one PRMT per half and word, one IADD3 each
  auto add2 = [&](const uint32_t (&a)[W], const uint32_t (&b)[W]) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      acc16[2 * w] += prmt(a[w], 0u, 0x7270u) + prmt(b[w], 0u, 0x7270u);      // bytes 0, 2
      acc16[2 * w + 1] += prmt(a[w], 0u, 0x7371u) + prmt(b[w], 0u, 0x7371u);  // bytes 1, 3
    }
  };
  int64_t* hp = nullptr;  // &hop_sums[p][c] of this lane's placement p = lane & (P - 1) (set per warp range)
  int since = 0;          // windows started since the last flush (warp-uniform)
  // warp-uniform: running sums of the current chunk -> hop_sums[.][c].  The warp sums come from
  // redux.sync, one instruction per word with no shuffle traffic through the shared-memory pipe
  // (a P = 16 reduce-scatter took 16 SHFL per boundary: 140 tokens per chunk, score W = 4 2.74 ->
  // 2.49 ms, W = 1 1.04 -> 0.95 ms, fused 1.49 -> 1.39 ms); lane p < P then adds placement p.  Within 3 windows of the
  // last flush (at most 4 windows of sums: the flushed window's rest + 3) the u16 lanes of the warp
  // sum cannot overflow (32 lanes x 4 x 2 tokens x 248 < 2^16), so the 2W packed words are summed
  // as they are; otherwise each u16 lane is summed on its own.
  auto flush = [&]() {
    const int pl = lane & (P - 1), j = 2 * (pl >> 2) + (pl & 1);  // word of placement pl; bit 1: high half
    uint32_t t = 0;
    if (since <= 3) {
#pragma unroll
      for (int i = 0; i < 2 * W; ++i) {
        const uint32_t v = __reduce_add_sync(0xffffffffu, acc16[i]);
        t = i == j ? v : t;
        acc16[i] = 0;
      }
      t = (pl & 2) ? t >> 16 : t & 0xffffu;
    } else {
#pragma unroll
      for (int i = 0; i < 2 * W; ++i) {
        const uint32_t lo = __reduce_add_sync(0xffffffffu, acc16[i] & 0xffffu);
        const uint32_t hi = __reduce_add_sync(0xffffffffu, acc16[i] >> 16);
        t = i == j ? ((pl & 2) ? hi : lo) : t;
        acc16[i] = 0;
      }
    }
    since = 0;
    if (lane < P && t) atomic_add_i64(hp, (int64_t)t);
  };
  // the 8 lookups (+ histogram increments) of one token record: u8-lane sums per table word
  auto record = [&](uint32_t w0, uint32_t w1, bool valid, uint32_t (&sum)[W]) {
#pragma unroll
    for (int w = 0; w < W; ++w) sum[w] = 0;
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      const uint32_t word = k < 4 ? w0 : w1;
      const uint32_t a0 = base + prmt(word, slot, sel_row(k & 3));
      const uint32_t a1 = base + prmt(word, slot, sel_row((k + 1) & 3));
      uint32_t x0[W], x1[W];
      seg_lookup<W>(a0, x0);
      seg_lookup<W>(a1, x1);
#pragma unroll
      for (int w = 0; w < W; ++w) sum[w] = sum[w] + x0[w] + x1[w];
      if constexpr (HIST) {
        if constexpr (kHistRegion) {
          atoms_inc(valid ? prmt(word, 0u, 0x4440u | (uint32_t)(k & 3)) * 128u + hreg : trash);
          atoms_inc(valid ? prmt(word, 0u, 0x4440u | (uint32_t)((k + 1) & 3)) * 128u + hreg : trash);
        } else {  // W = 1: the lane's replica sits 128 bytes after its table slot in the same row
          atoms_inc(valid ? a0 + 128u : trash);
          atoms_inc(valid ? a1 + 128u : trash);
        }
      }
    }
    if (!valid) {
#pragma unroll
      for (int w = 0; w < W; ++w) sum[w] = 0;
    }
  };

  Flat f(t0 * 8, t1 * 8, L);
  for (int64_t g = f.g0; g < f.g1;) {
    const int l = (int)(g / f.nb);
    const int64_t off_in = g - (int64_t)l * f.nb;
    const int64_t seg = min(f.g1 - g, f.nb - off_in);
    const int64_t x0 = f.b0 + off_in, x1 = x0 + seg;  // multiples of 8: whole records
    const uint8_t* plane = planes + (int64_t)l * stride;

    __syncthreads();  // previous segment is done with shared memory
    {
      constexpr int WPR = (W == 2) ? 64 : 32;  // table words per row
      const uint32_t* tl = tables + (int64_t)l * 256 * W;
      for (int i = threadIdx.x; i < 256 * WPR; i += blockDim.x) {
        const int e = i / WPR, j = i % WPR;
        smw[e * 64 + j] = __ldg(tl + e * W + (j % W));
      }
      if constexpr (kHistRegion)
        for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) smw[kHistWords + i] = 0;
      else if constexpr (HIST)
        for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) smw[(i >> 5) * 64 + 32 + (i & 31)] = 0;
    }
    __syncthreads();

    // tokens [ta, tb) of this segment; vector (token pair) m covers tokens 2m, 2m+1
    const int64_t ta = x0 / 8, tb = x1 / 8;
    const int64_t m0 = ta >> 1, m1 = (tb + 1) >> 1;
    const int64_t per = (m1 - m0 + kSegWarps - 1) / kSegWarps;
    const int64_t wm0 = min(m1, m0 + per * warp), wm1 = min(m1, wm0 + per);
    if (wm0 < wm1) {
      // the warp's tokens [wt0, wt1); 32-bit offsets from its first pair (pair r = tokens T0+2r, +1)
      const int64_t wt0 = max(ta, 2 * wm0), wt1 = min(tb, 2 * wm1);
      const int64_t T0 = 2 * wm0;
      const int npairs = (int)(wm1 - wm0);
      const int ra = (int)(wt0 - T0), rb = (int)(wt1 - T0);  // valid relative tokens [ra, rb)
      int c = 0;
      {
        int lo = 0, hi = C;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (__ldg(bounds + mid) <= wt0) lo = mid; else hi = mid;
        }
        c = lo;
      }
      // relative chunk starts: 32-bit differences (a GPU's token range is far below 2^31), low words only
      const uint32_t T0lo = (uint32_t)T0;
      auto next_start = [&](int cc) {
        return (int)(__ldg(reinterpret_cast<const uint32_t*>(bounds + cc)) - T0lo);
      };
      int nbr = next_start(c + 1);  // first token of the next chunk
      hp = hop_sums + (int64_t)(lane & (P - 1)) * C + c;
      const int4* __restrict__ pv = reinterpret_cast<const int4*>(plane) + wm0;

      // one 64-token window: pairs [rfirst, rfirst + 32).  EDGE: it may hold tokens outside
      // [ra, rb) (the warp's first window when ra = 1, the last ones); interior windows carry no
      // per-lane validity logic at all.
      auto window = [&](const int4& x, int rfirst, auto edge_tag) {
        constexpr bool EDGE = decltype(edge_tag)::value;
        ++since;
        bool vA = true, vB = true;
        if constexpr (EDGE) {
          const int tA = 2 * (rfirst + lane);
          vA = tA >= ra && tA < rb;
          vB = tA + 1 >= ra && tA + 1 < rb;
        }
        uint32_t sA[W], sB[W];
        record((uint32_t)x.x, (uint32_t)x.y, vA, sA);
        record((uint32_t)x.z, (uint32_t)x.w, vB, sB);
        const int wlast = EDGE ? min(2 * rfirst + 63, rb - 1) : 2 * rfirst + 63;  // last valid token
        if (nbr <= wlast) {  // chunk boundaries inside the window (warp-uniform)
          const int tA = 2 * (rfirst + lane);
          do {
            const bool inA = tA < nbr, inB = tA + 1 < nbr;  // tokens of chunk c not yet added
            uint32_t pA[W], pB[W];
#pragma unroll
            for (int w = 0; w < W; ++w) {
              pA[w] = inA ? sA[w] : 0u;
              pB[w] = inB ? sB[w] : 0u;
              sA[w] -= pA[w];
              sB[w] -= pB[w];
            }
            add2(pA, pB);
            flush();
            ++c;  // c < C - 1 here: bounds[C] >= the trace end > the window
            ++hp;
            nbr = next_start(c + 1);
          } while (nbr <= wlast);
        }
        add2(sA, sB);
      };
      using Interior = std::integral_constant<bool, false>;
      using Edge = std::integral_constant<bool, true>;

      // pairs [0, full) have both tokens valid when ra = 0; the first window is an edge when ra = 1
      const int full = rb == 2 * npairs ? npairs : npairs - 1;
      int rw = 0, nwin = 0;
      if (ra != 0) {
        const int4 x = lane < npairs ? ldg_stream(pv + lane) : make_int4(0, 0, 0, 0);
        window(x, 0, Edge{});
        rw = 32;
      }
      for (; rw + 32 * U <= full; rw += 32 * U) {  // interior batches: unpredicated loads
        int4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = ldg_stream(pv + rw + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < U; ++u) window(x[u], rw + u * 32, Interior{});
        if ((nwin += U) >= 128) {  // u16 headroom: flush into the same chunk
          flush();
          nwin = 0;
        }
      }
      for (; rw < npairs; rw += 32) {  // the rest, one window at a time (< U + 1 per warp range)
        const int r = rw + lane;
        const int4 x = r < npairs ? ldg_stream(pv + r) : make_int4(0, 0, 0, 0);
        window(x, rw, Edge{});
      }
      flush();
    }

    if constexpr (HIST) {
      __syncthreads();
      for (int e = threadIdx.x; e < 256; e += blockDim.x) {
        const uint32_t* row = kHistRegion ? smw + kHistWords + e * 32 : smw + e * 64 + 32;
        uint32_t sum = 0;
#pragma unroll 8
        for (int r = 0; r < 32; ++r) sum += row[(r + e) & 31];
        if (sum) {
          if (e < E) atomic_add_i64(counts + (int64_t)l * E + e, (int64_t)sum);
          else report_err(err, MP_DATA_EXPERT_RANGE, l, e, sum);
        }
      }
    }
    g += seg;
  }
}

template <int W, bool HIST>
static cudaError_t launch_seg_t(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int E,
                                const int64_t* bounds, int C, const uint32_t* tables, int64_t* counts,
                                int64_t* hop_sums, int64_t* err, cudaStream_t s) {
  auto kern = seg_kernel<W, HIST>;
  const int smem = 256 * 256 + ((HIST && W > 1) ? 256 * 128 : 0) + 128;
  int per_sm = 0;
  cudaError_t e = prepare_kernel((const void*)kern, kSegThreads, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const int nsm = device_sm_count();
  const int64_t total = (t1 - t0) * 8 * (int64_t)L;
  int64_t grid = (int64_t)nsm * max(1, per_sm);
  grid = max((int64_t)1, min(grid, (total + 65535) / 65536));
  kern<<<(unsigned)grid, kSegThreads, smem, s>>>(planes, stride, t0, t1, L, E, bounds, C, tables, counts, hop_sums, err);
  return cudaGetLastError();
}

// K = 8 and max_p <= 31 only (the caller checks).
cudaError_t launch_seg(bool hist, int W, const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int E,
                       const int64_t* bounds, int C, const uint32_t* tables, int64_t* counts, int64_t* hop_sums,
                       int64_t* err, cudaStream_t s) {
  if (hist) {
    if (W == 1) return launch_seg_t<1, true>(planes, stride, t0, t1, L, E, bounds, C, tables, counts, hop_sums, err, s);
    if (W == 2) return launch_seg_t<2, true>(planes, stride, t0, t1, L, E, bounds, C, tables, counts, hop_sums, err, s);
    if (W == 4) return launch_seg_t<4, true>(planes, stride, t0, t1, L, E, bounds, C, tables, counts, hop_sums, err, s);
    return cudaErrorInvalidValue;
  }
  if (W == 1) return launch_seg_t<1, false>(planes, stride, t0, t1, L, E, bounds, C, tables, counts, hop_sums, err, s);
  if (W == 2) return launch_seg_t<2, false>(planes, stride, t0, t1, L, E, bounds, C, tables, counts, hop_sums, err, s);
  if (W == 4) return launch_seg_t<4, false>(planes, stride, t0, t1, L, E, bounds, C, tables, counts, hop_sums, err, s);
  return cudaErrorInvalidValue;
}

}  // namespace mp
