// Segmented gather (MP_ALGO_SEG): per-chunk hop sums whose cost does not depend on the chunk count,
// as a layer-major stream (no per-layer table re-staging per token tile, unlike the token-tiled
// scorer).  K = 8, max_p <= 31.
//
// A CTA walks its byte range plane segment by plane segment like the streaming kernels and stages
// the layer's W-word table replicated per lane slot (conflict-free PRMT-addressed lookups).  The
// segment's tokens are then split into 16 contiguous warp sub-ranges; a warp streams its
// sub-range in windows of 64 tokens (one 16-byte vector = two 8-pick records per lane, four
// windows in flight) and keeps running per-lane sums of the current chunk.  Chunk boundaries are
// detected per window from the chunk bounds (warp-uniform): the tokens before the boundary are
// added, the warp reduce-scatters its running sums and adds them to hop_sums[q][c] (one int64
// atomic per placement), and the sums restart for the next chunk.  The streaming kernels instead
// spread every (layer, chunk) piece over the whole CTA, so short chunks leave most threads idle;
// here a boundary costs one warp reduction wherever it falls.
// Per-token sums of 8 lookups fit u8 lanes (8 * 31 < 256); running sums are u16 lanes widened
// into u32 every 64 windows and at each flush.  With HIST every byte also increments the
// lane-replicated histogram (W = 1: in the table rows' free half, one PRMT per address; W = 2 / 4:
// a separate region of 128-byte rows, PRMT byte extract + IMAD), flushed per segment.
#include "common.cuh"

namespace mp {

constexpr int kSegWarps = kThreads / 32;  // 16
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
__global__ void __launch_bounds__(kThreads, 2)
seg_kernel(const uint8_t* __restrict__ planes, int64_t stride, int64_t t0, int64_t t1, int L, int E,
           const int64_t* __restrict__ bounds, int C, const uint32_t* __restrict__ tables,
           int64_t* __restrict__ counts, int64_t* __restrict__ hop_sums, int64_t* __restrict__ err) {
  constexpr int K = 8;
  constexpr int P = 4 * W;
  // 256 rows x 256 B of tables (W = 1: bytes 128-255 of each row hold the histogram replicas);
  // W > 1 with HIST: + a 256 rows x 128 B histogram region; then a 128-byte trash row
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr bool kHistRegion = HIST && W > 1;
  constexpr int kHistWords = 256 * 256 / 4;  // word offset of the separate histogram region
  uint32_t* smw = reinterpret_cast<uint32_t*>(sm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = smem_addr(sm);
  const uint32_t hbase = base + 128;
  const uint32_t slot = W == 4 ? (uint32_t)((lane & 7) << 4) : W == 2 ? (uint32_t)(lane << 3) : (uint32_t)(lane << 2);
  const uint32_t hslot = (uint32_t)(lane << 2);
  const uint32_t hreg = base + 256 * 256 + hslot;  // W > 1: bin e of this lane at hreg + e * 128
  const uint32_t trash = base + 256 * 256 + (kHistRegion ? 256 * 128 : 0) + hslot;  // masked-out tokens (no branch)
  // histogram address of byte b of `word` (lane replica)
  auto haddr = [&](uint32_t word, int b) -> uint32_t {
    if constexpr (kHistRegion) return prmt(word, 0u, 0x4440u | (uint32_t)b) * 128u + hreg;
    else return hbase + prmt(word, hslot, sel_row(b));
  };

  uint32_t acc16[2 * W], acc32[P];
#pragma unroll
  for (int i = 0; i < 2 * W; ++i) acc16[i] = 0;
#pragma unroll
  for (int i = 0; i < P; ++i) acc32[i] = 0;
  auto widen = [&]() {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      acc32[4 * w + 0] += acc16[2 * w] & 0xffffu;
      acc32[4 * w + 2] += acc16[2 * w] >> 16;
      acc32[4 * w + 1] += acc16[2 * w + 1] & 0xffffu;
      acc32[4 * w + 3] += acc16[2 * w + 1] >> 16;
      acc16[2 * w] = 0;
      acc16[2 * w + 1] = 0;
    }
  };
  auto add_token = [&](const uint32_t (&s)[W]) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      acc16[2 * w] += s[w] & 0x00ff00ffu;
      acc16[2 * w + 1] += (s[w] >> 8) & 0x00ff00ffu;
    }
  };
  auto flush = [&](int c) {  // warp-uniform: running sums of chunk c -> hop_sums[.][c]
    widen();
    int q = 0;
    const uint32_t tot = warp_reduce_scatter<P>(acc32, lane, &q);
    if ((lane & (32 / P - 1)) == 0 && tot) atomic_add_i64(hop_sums + (int64_t)q * C + c, (int64_t)tot);
#pragma unroll
    for (int i = 0; i < P; ++i) acc32[i] = 0;
  };

  Flat f(t0 * K, t1 * K, L);
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
    const int64_t ta = x0 / K, tb = x1 / K;
    const int64_t m0 = ta >> 1, m1 = (tb + 1) >> 1;
    const int64_t per = (m1 - m0 + kSegWarps - 1) / kSegWarps;
    const int64_t wm0 = min(m1, m0 + per * warp), wm1 = min(m1, wm0 + per);
    if (wm0 < wm1) {
      // the warp's tokens [wt0, wt1)
      const int64_t wt0 = max(ta, 2 * wm0), wt1 = min(tb, 2 * wm1);
      int c = 0;
      {
        int lo = 0, hi = C;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (__ldg(bounds + mid) <= wt0) lo = mid; else hi = mid;
        }
        c = lo;
      }
      int64_t nb = __ldg(bounds + c + 1);  // first token of the next chunk
      // 32-bit offsets from the warp's first pair: pair r covers tokens T0 + 2r, T0 + 2r + 1
      const int64_t T0 = 2 * wm0;
      const int npairs = (int)(wm1 - wm0);
      const int ra = (int)(wt0 - T0), rb = (int)(wt1 - T0);  // valid relative tokens [ra, rb)
      auto rel = [&](int64_t t) { return (int)min(t - T0, (int64_t)0x7fffffff); };
      int nbr = rel(nb);
      const int4* __restrict__ pv = reinterpret_cast<const int4*>(plane) + wm0;
      int since = 0;  // windows since the last widen
      for (int rw = 0; rw < npairs; rw += 32 * seg_unroll<W>()) {
        constexpr int kSegU = seg_unroll<W>();
        int4 x[kSegU];
#pragma unroll
        for (int u = 0; u < kSegU; ++u) {
          const int r = rw + u * 32 + lane;
          x[u] = r < npairs ? ldg_stream(pv + r) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kSegU; ++u) {
          const int rfirst = rw + u * 32;
          if (rfirst >= npairs) break;  // warp-uniform
          const int r = rfirst + lane;
          const int tA = 2 * r, tB = tA + 1;
          const bool vA = r < npairs && tA >= ra && tA < rb;
          const bool vB = r < npairs && tB >= ra && tB < rb;
          const uint32_t wd[4] = {(uint32_t)x[u].x, (uint32_t)x[u].y, (uint32_t)x[u].z, (uint32_t)x[u].w};
          uint32_t sA[W], sB[W];
#pragma unroll
          for (int w = 0; w < W; ++w) sA[w] = sB[w] = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t word = wd[k >> 2];
            const uint32_t off = prmt(word, slot, sel_row(k & 3));
            uint32_t t[W];
            seg_lookup<W>(base + off, t);
#pragma unroll
            for (int w = 0; w < W; ++w) sA[w] += t[w];
            if constexpr (HIST) atoms_inc(vA ? haddr(word, k & 3) : trash);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t word = wd[2 + (k >> 2)];
            const uint32_t off = prmt(word, slot, sel_row(k & 3));
            uint32_t t[W];
            seg_lookup<W>(base + off, t);
#pragma unroll
            for (int w = 0; w < W; ++w) sB[w] += t[w];
            if constexpr (HIST) atoms_inc(vB ? haddr(word, k & 3) : trash);
          }
          // last valid token of this window (warp-uniform)
          const int wlast = min(2 * (rfirst + 31) + 1, rb - 1);
          if (nbr > wlast) {  // no boundary in the window (the common case for long chunks)
            if (vA) add_token(sA);
            if (vB) add_token(sB);
          } else {
            bool dA = !vA, dB = !vB;
            while (nbr <= wlast) {  // boundary inside the window: tokens < nb belong to chunk c
              if (!dA && tA < nbr) { add_token(sA); dA = true; }
              if (!dB && tB < nbr) { add_token(sB); dB = true; }
              flush(c);
              since = 0;
              ++c;
              nbr = rel(__ldg(bounds + c + 1));  // c < C - 1 here: bounds[C] >= t1 > the window
            }
            if (!dA) add_token(sA);
            if (!dB) add_token(sB);
          }
          if (++since == 64) {  // u16 lanes: <= 64 windows x 2 tokens x 248 < 2^16
            widen();
            since = 0;
          }
        }
      }
      flush(c);
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
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (e != cudaSuccess) return e;
  const int64_t total = (t1 - t0) * 8 * (int64_t)L;
  int64_t grid = (int64_t)nsm * max(1, per_sm);
  grid = max((int64_t)1, min(grid, (total + 65535) / 65536));
  kern<<<(unsigned)grid, kThreads, smem, s>>>(planes, stride, t0, t1, L, E, bounds, C, tables, counts, hop_sums, err);
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
