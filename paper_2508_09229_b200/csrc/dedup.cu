// Unique-destination scoring (extension A17; BASELINE north_star "each token's top-k destinations
// are deduplicated per server").  Not a SPEC metric: SPEC.md:339 counts every selected expert, and
// the SPEC hop sums are produced alongside, unchanged.
//
// For placement q, token t, layer l with picks e_0..e_{K-1}:
//   S = { server_q(e_k) }                          (servers hosting the picked experts)
//   uniq  = |S \ { server(d_l) }|                   (one message per remote destination server)
//   dedup = sum_{s in S} pe_q[l, s]                 (round-trip hops, one message per server;
//                                                    pe depends on the device only via its server)
// One thread per (token, layer) record; K = 8 records are one aligned 8-byte load.  Layer state in
// shared memory as 256 rows x 256 B: the packed pe word (4 placements) at lane*4 and the packed
// server-id word at 128 + lane*4, both replicated per lane (conflict-free, one PRMT per address).
// First occurrence of a server inside a record is detected by comparing against the record's
// earlier picks (K <= 32), so any server count <= 256 works.
#include "common.cuh"

namespace mp {

constexpr int kDedupMaxK = 32;

// bit 7 of every byte set where a == b (exact per byte, no borrow between lanes); the other bits
// are garbage -- callers mask with 0x80808080 once, after OR-ing several of these together
__device__ __forceinline__ uint32_t bytes_eq7(uint32_t a, uint32_t b) {
  const uint32_t x = a ^ b;
  const uint32_t t = (x & 0x7f7f7f7fu) + 0x7f7f7f7fu;
  return ~(t | x);
}
__device__ __forceinline__ uint32_t bytes_eq(uint32_t a, uint32_t b) { return bytes_eq7(a, b) & 0x80808080u; }

// K = 8 record, all 4 placements at once (byte lanes): SPEC hops and dedup hops widened into u16
// lanes ({q0,q2}, {q1,q3}), unique remote destination servers as u8 lanes (<= 8 per record).
__device__ __forceinline__ void dedup_record8(uint2 v, uint32_t base, uint32_t slot, uint32_t src4,
                                              uint32_t (&hop16)[2], uint32_t& uq8, uint32_t (&dd16)[2]) {
  const uint32_t wv[2] = {v.x, v.y};
  uint32_t sw[8], pw[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t a = base + prmt(wv[k >> 2], slot, sel_row(k & 3));
    pw[k] = lds32(a);
    sw[k] = lds32(a + 128);
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint32_t seen = 0;
#pragma unroll
    for (int j = 0; j < k; ++j) seen |= bytes_eq7(sw[k], sw[j]);
    const uint32_t first = ~seen & 0x80808080u;   // 0x80 where the pick's server is new in the record
    const uint32_t m = pw[k] & ((first >> 7) * 0xffu);
    hop16[0] += pw[k] & 0x00ff00ffu;
    hop16[1] += (pw[k] >> 8) & 0x00ff00ffu;
    dd16[0] += m & 0x00ff00ffu;
    dd16[1] += (m >> 8) & 0x00ff00ffu;
    uq8 += (first & ~bytes_eq(sw[k], src4)) >> 7;  // +1 per lane: new server, not the source
  }
}

constexpr int kDedupThreads = 512;
// One-hot server masks for layers whose server ids are < 32 and costs <= 15, built
// and measured against the pairwise tests: 3.587 vs 3.420 ms at 150 chunks, 3.70 vs 3.56 at 15k,
// 5.03 vs 4.98 at 150k (R1 10M, FatTree 8x4x8; ncu: L1TEX 85 %, 833M shared wavefronts -- the 4
// LDS.128 wavefronts per pick -- and ALU 71 %), so it is off by default (-DMP_DEDUP_ONEHOT=1 builds it).
#ifndef MP_DEDUP_ONEHOT
#define MP_DEDUP_ONEHOT 0
#endif
#ifndef MP_DEDUP_U
#define MP_DEDUP_U 2  // 32-pair windows in flight per warp (K = 8 warp-range path)
#endif

// One record's contributions as u16 lane pairs ({q0, q2}, {q1, q3}): SPEC hops, distinct remote
// destination servers, deduplicated hops.
struct DedupRec {
  uint32_t h[2], u[2], d[2];
};

// Fast K = 8 record (pe bytes <= 31, server ids < 128; slot lane*8 holds {pe word, server word} with
// bit 7 of each server byte flagging the layer's source server).  Per pick k the byte-parallel
// "differs from every earlier pick" test is AND_j ((s_k ^ s_j) | 0x80808080) - 0x01010101 (bit 7 per
// byte, no borrow between bytes); PRMT's sign-replicate mode turns it into a 0x00/0xff byte mask.
// Each pick's loads are consumed at once, so only the 8 server words stay live.
__device__ __forceinline__ void dedup_rec_fast(uint32_t w0, uint32_t w1, uint32_t base, uint32_t slot8, DedupRec& r) {
  uint32_t sw[8];
  uint32_t h8 = 0, d8 = 0, n8 = 0, srcany = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint2 e = lds64(base + prmt(k < 4 ? w0 : w1, slot8, sel_row(k & 3)));
    sw[k] = e.y;
    uint32_t m = 0xffffffffu;
    if (k > 0) {
      uint32_t nw = 0xffffffffu;
#pragma unroll
      for (int j = 0; j < k; ++j) nw &= ((e.y ^ sw[j]) | 0x80808080u) - 0x01010101u;
      m = prmt(nw, 0u, 0xBA98u);  // byte = 0xff iff its bit 7 is set (the server is new)
    }
    h8 += e.x;
    d8 += e.x & m;
    n8 += m & 0x01010101u;
    srcany |= e.y;
  }
  n8 -= (srcany >> 7) & 0x01010101u;  // distinct remote destination servers per placement byte
  r.h[0] = prmt(h8, 0u, 0x7270u);
  r.h[1] = prmt(h8, 0u, 0x7371u);
  r.d[0] = prmt(d8, 0u, 0x7270u);
  r.d[1] = prmt(d8, 0u, 0x7371u);
  r.u[0] = prmt(n8, 0u, 0x7270u);
  r.u[1] = prmt(n8, 0u, 0x7371u);
}

// One-hot K = 8 record (every server id < 32 and pe byte <= 31 in the layer; the variant VERDICT r1
// asked to be built and measured).  Row e: bytes 0-127 hold {onehot_q0 .. onehot_q3} (1 << server of
// expert e under placement q) at slot (lane & 7) * 16 -- one LDS.128 per pick, a quarter-warp per
// wavefront -- and bytes 128-255 the pe word at 128 + lane * 4.  The record's server sets are the OR
// of its 8 masks; distinct remote servers = popc(set & ~source); deduplicated hops =
// sum_b popc(set & plane_b) << b with plane_b = the servers whose cost has bit b (per layer and
// placement, built by the CTA).
struct __align__(16) OnehotLayer {
  uint32_t plane[4][4];  // [q][bit]: costs <= 15 (a layer with a larger cost takes the pairwise path)
  uint32_t src;          // byte q = source server of the layer under placement q
  int nb;                // cost bits in use (<= 4)
};
// The planes stay in shared memory (one broadcast LDS.128 per placement and record): holding the 16
// plane words in registers spilled at the 64-register budget of 2 CTAs per SM.
__device__ __forceinline__ void dedup_rec_onehot(uint32_t w0, uint32_t w1, uint32_t base, uint32_t slot16,
                                                 uint32_t slotpe, const OnehotLayer* ol, uint32_t srcw, DedupRec& r) {
  uint32_t M[4] = {0u, 0u, 0u, 0u}, h8 = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t word = k < 4 ? w0 : w1;
    const uint4 m = lds128(base + prmt(word, slot16, sel_row(k & 3)));
    h8 += lds32(base + prmt(word, slotpe, sel_row(k & 3)));
    M[0] |= m.x;
    M[1] |= m.y;
    M[2] |= m.z;
    M[3] |= m.w;
  }
  uint32_t u[4], d[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    u[q] = __popc(M[q]) - ((M[q] >> ((srcw >> (8 * q)) & 31u)) & 1u);
    const uint4 pl = *reinterpret_cast<const uint4*>(ol->plane[q]);  // zero planes beyond the layer's bits
    d[q] = __popc(M[q] & pl.x) + ((uint32_t)__popc(M[q] & pl.y) << 1) + ((uint32_t)__popc(M[q] & pl.z) << 2) +
           ((uint32_t)__popc(M[q] & pl.w) << 3);
  }
  r.h[0] = prmt(h8, 0u, 0x7270u);
  r.h[1] = prmt(h8, 0u, 0x7371u);
  r.u[0] = u[0] | (u[2] << 16);
  r.u[1] = u[1] | (u[3] << 16);
  r.d[0] = d[0] | (d[2] << 16);
  r.d[1] = d[1] | (d[3] << 16);
}

// MODE 0: general pairwise record (any server id <= 255, pe <= 255); 1: fast pairwise (ids < 128,
// pe <= 31); 2: one-hot masks (ids < 32, pe <= 31)
template <int MODE>
__device__ __forceinline__ void dedup_warp_range(const uint8_t* __restrict__ plane, int64_t wm0, int64_t wm1,
                                                 int64_t r0, int64_t r1, const int64_t* __restrict__ bounds, int C,
                                                 uint32_t base, uint32_t slot, uint32_t slot8, uint32_t src, int lane,
                                                 int64_t* __restrict__ hop_sums, int64_t* __restrict__ uniq_sums,
                                                 int64_t* __restrict__ dedup_sums, const OnehotLayer* s_ol) {
  constexpr int U = MP_DEDUP_U;
  constexpr bool FAST = MODE != 0;
  const uint32_t slot16 = (uint32_t)((lane & 7) << 4), slotpe = 128u + (uint32_t)(lane << 2);
  const int64_t wt0 = max(r0, 2 * wm0), wt1 = min(r1, 2 * wm1);
  int c = 0;
  {
    int lo = 0, hi = C;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(bounds + mid) <= wt0) lo = mid; else hi = mid;
    }
    c = lo;
  }
  const int64_t T0 = 2 * wm0;
  const int npairs = (int)(wm1 - wm0);
  const int ra = (int)(wt0 - T0), rb = (int)(wt1 - T0);  // valid relative tokens [ra, rb)
  const uint32_t T0lo = (uint32_t)T0;                      // 32-bit relative chunk starts
  auto next_start = [&](int cc) { return (int)(__ldg(reinterpret_cast<const uint32_t*>(bounds + cc)) - T0lo); };
  int nbr = next_start(c + 1);
  // lane q < 12 adds value q: 0-3 SPEC hops, 4-7 distinct remote servers, 8-11 deduplicated hops
  // (placement q & 3)
  const int qs = lane < 12 ? lane : 0, qk = qs >> 2, qp = qs & 3;
  int64_t* hp = (qk == 0 ? hop_sums : qk == 1 ? uniq_sums : dedup_sums) + (int64_t)qp * C + c;
  uint32_t h16[2] = {0, 0}, u16[2] = {0, 0}, d16[2] = {0, 0};  // running sums of chunk c, u16 lanes
  int since = 0;  // windows started since the last flush (warp-uniform)
  // warp sums by redux.sync (no shuffle traffic; was a 16-value reduce-scatter); word k16[qp & 1]
  // holds placement qp in its (qp >> 1) half.  Fast records (<= 248 per kind) within 3 windows of
  // the last flush keep the 6 packed words (32 lanes x 4 windows x 2 x 248 < 2^16).
  auto flush = [&]() {
    const uint32_t w[6] = {h16[0], h16[1], u16[0], u16[1], d16[0], d16[1]};
    const int j = 2 * qk + (qp & 1);
    uint32_t t = 0;
    if (FAST && since <= 3) {
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const uint32_t v = __reduce_add_sync(0xffffffffu, w[i]);
        t = i == j ? v : t;
      }
      t = (qp & 2) ? t >> 16 : t & 0xffffu;
    } else {
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        const uint32_t lo = __reduce_add_sync(0xffffffffu, w[i] & 0xffffu);
        const uint32_t hi = __reduce_add_sync(0xffffffffu, w[i] >> 16);
        t = i == j ? ((qp & 2) ? hi : lo) : t;
      }
    }
    h16[0] = h16[1] = u16[0] = u16[1] = d16[0] = d16[1] = 0;
    since = 0;
    if (lane < 12 && t) atomic_add_i64(hp, (int64_t)t);
  };
  auto rec = [&](uint32_t w0, uint32_t w1, DedupRec& r) {
    if constexpr (MODE == 2) {
      dedup_rec_onehot(w0, w1, base, slot16, slotpe, s_ol, src, r);
    } else if constexpr (MODE == 1) {
      dedup_rec_fast(w0, w1, base, slot8, r);
    } else {
      uint32_t hh[2] = {0, 0}, dd[2] = {0, 0}, uq = 0;
      dedup_record8(make_uint2(w0, w1), base, slot, src, hh, uq, dd);
      r.h[0] = hh[0]; r.h[1] = hh[1]; r.d[0] = dd[0]; r.d[1] = dd[1];
      r.u[0] = prmt(uq, 0u, 0x7270u);
      r.u[1] = prmt(uq, 0u, 0x7371u);
    }
  };
  auto mask = [&](DedupRec& r, bool keep) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      r.h[i] = keep ? r.h[i] : 0u;
      r.u[i] = keep ? r.u[i] : 0u;
      r.d[i] = keep ? r.d[i] : 0u;
    }
  };
  auto add2 = [&](const DedupRec& a, const DedupRec& b) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      h16[i] += a.h[i] + b.h[i];
      u16[i] += a.u[i] + b.u[i];
      d16[i] += a.d[i] + b.d[i];
    }
  };
  const uint4* __restrict__ pv = reinterpret_cast<const uint4*>(plane) + wm0;
  auto window = [&](const uint4& x, int rfirst, bool edge) {
    ++since;
    const int tA = 2 * (rfirst + lane);
    DedupRec A, B;
    rec(x.x, x.y, A);
    rec(x.z, x.w, B);
    if (edge) {
      mask(A, tA >= ra && tA < rb);
      mask(B, tA + 1 >= ra && tA + 1 < rb);
    }
    const int wlast = edge ? min(2 * rfirst + 63, rb - 1) : 2 * rfirst + 63;
    while (nbr <= wlast) {  // boundary inside the window (warp-uniform): tokens < nbr are chunk c's
      DedupRec pa = A, pb = B;
      const bool inA = tA < nbr, inB = tA + 1 < nbr;
      mask(pa, inA);
      mask(pb, inB);
      mask(A, !inA);
      mask(B, !inB);
      add2(pa, pb);
      flush();
      ++c;  // c < C - 1 here: bounds[C] >= the trace end > the window
      ++hp;
      nbr = next_start(c + 1);
    }
    add2(A, B);
  };
  // pairs [0, full) have both tokens valid when ra = 0; u16 headroom: 2 records x 2040 per window for
  // the general path, so flush every 16 windows there and every 128 on the fast path (2 x 248)
  constexpr int kFlushWin = FAST ? 128 : 16;
  const int full = rb == 2 * npairs ? npairs : npairs - 1;
  int rw = 0, nwin = 0;
  if (ra != 0) {
    const uint4 x = lane < npairs ? pv[lane] : make_uint4(0, 0, 0, 0);
    window(x, 0, true);
    rw = 32;
    ++nwin;
  }
  for (; rw + 32 * U <= full; rw += 32 * U) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int4 v = ldg_stream(pv + rw + u * 32 + lane);
      x[u] = make_uint4((uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) window(x[u], rw + u * 32, false);
    if ((nwin += U) >= kFlushWin) {
      flush();
      nwin = 0;
    }
  }
  for (; rw < npairs; rw += 32) {
    const int r = rw + lane;
    uint4 x = make_uint4(0, 0, 0, 0);
    if (r < npairs) {
      const int4 v = ldg_stream(pv + r);
      x = make_uint4((uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w);
    }
    window(x, rw, true);
    if (++nwin >= kFlushWin) {
      flush();
      nwin = 0;
    }
  }
  flush();
}

__global__ void __launch_bounds__(kDedupThreads, 2) dedup_kernel(const uint8_t* __restrict__ planes, int64_t stride, int64_t t0,
                                                    int64_t t1, int L, int K, const int64_t* __restrict__ bounds,
                                                    int C, const uint32_t* __restrict__ tables,
                                                    const uint32_t* __restrict__ srv_tables,
                                                    const uint8_t* __restrict__ src_srv, int64_t* __restrict__ hop_sums,
                                                    int64_t* __restrict__ uniq_sums, int64_t* __restrict__ dedup_sums) {
  extern __shared__ __align__(128) uint8_t sm[];  // 256 rows x 256 B
  __shared__ uint32_t s_src;                      // 4 source-server bytes of this layer
  __shared__ OnehotLayer s_ol;                    // one-hot mode: cost bit-planes and source masks
  uint32_t* smw = reinterpret_cast<uint32_t*>(sm);
  const int lane = threadIdx.x & 31;
  const uint32_t base = smem_addr(sm);
  const uint32_t slot = (uint32_t)(lane << 2);
  const uint32_t slot8 = (uint32_t)(lane << 3);
  const int64_t n = t1 - t0;
  const int64_t total = n * (int64_t)L;
  int64_t per = (total + gridDim.x - 1) / gridDim.x;
  int64_t g = min(total, (int64_t)blockIdx.x * per);
  const int64_t g1 = min(total, g + per);
  while (g < g1) {
    const int l = (int)(g / n);
    const int64_t r0 = t0 + (g - (int64_t)l * n);
    const int64_t r1 = min(t0 + n, r0 + (g1 - g));
    const uint8_t* plane = planes + (int64_t)l * stride;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t w = 0;
      for (int q = 0; q < 4; ++q) w |= (uint32_t)src_srv[q * L + l] << (8 * q);
      s_src = w;
    }
    uint32_t wide = 0;  // any pe byte > 31 or server id >= 128 in this layer -> exact general path
    for (int e = threadIdx.x; e < 256; e += blockDim.x)
      wide |= (__ldg(tables + (int64_t)l * 256 + e) & 0xe0e0e0e0u) | (__ldg(srv_tables + (int64_t)l * 256 + e) & 0x80808080u);
    const bool fast = __syncthreads_or(wide != 0 || (threadIdx.x == 0 && (s_src & 0x80808080u))) == 0 && K == 8;
    uint32_t wide32 = 0;  // any server id >= 32 (source included) or cost > 15 -> no one-hot masks
    for (int e = threadIdx.x; e < 256; e += blockDim.x)
      wide32 |= (__ldg(srv_tables + (int64_t)l * 256 + e) & 0xe0e0e0e0u) | (__ldg(tables + (int64_t)l * 256 + e) & 0xf0f0f0f0u);
    const bool onehot = MP_DEDUP_ONEHOT && fast &&
                        __syncthreads_or(wide32 != 0 || (threadIdx.x == 0 && (s_src & 0xe0e0e0e0u))) == 0;
    const uint32_t src = s_src;
    if (onehot) {
      if (threadIdx.x < 16) reinterpret_cast<uint32_t*>(s_ol.plane)[threadIdx.x] = 0u;
      if (threadIdx.x == 0) {
        s_ol.src = src;
        s_ol.nb = 0;
      }
      __syncthreads();
      uint32_t maxp = 0;
      for (int e = threadIdx.x; e < 256; e += blockDim.x) {
        const uint32_t pw = __ldg(tables + (int64_t)l * 256 + e), sw = __ldg(srv_tables + (int64_t)l * 256 + e);
        for (int q = 0; q < 4; ++q) {
          const uint32_t p = (pw >> (8 * q)) & 0xffu, sv = (sw >> (8 * q)) & 31u;
          maxp = max(maxp, p);
          for (int b = 0; b < 4; ++b)
            if ((p >> b) & 1u) atomicOr(&s_ol.plane[q][b], 1u << sv);
        }
      }
      atomicMax(&s_ol.nb, 32 - __clz((int)maxp));
      for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
        const int e = i >> 5, j = i & 31;
        const uint32_t pw = __ldg(tables + (int64_t)l * 256 + e), sw = __ldg(srv_tables + (int64_t)l * 256 + e);
        smw[e * 64 + 32 + j] = pw;  // pe word at 128 + lane * 4
        if (j < 8) {                // one-hot masks at (lane & 7) * 16
#pragma unroll
          for (int q = 0; q < 4; ++q) smw[e * 64 + 4 * j + q] = 1u << ((sw >> (8 * q)) & 31u);
        }
      }
    } else for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
      const int e = i >> 5, j = i & 31;
      const uint32_t pw = __ldg(tables + (int64_t)l * 256 + e), sw = __ldg(srv_tables + (int64_t)l * 256 + e);
      if (fast) {  // {pe, server | source flag} at lane slot j*8
        smw[e * 64 + 2 * j] = pw;
        smw[e * 64 + 2 * j + 1] = sw | bytes_eq(sw, src);
      } else {     // pe at j*4, server at 128 + j*4
        smw[e * 64 + j] = pw;
        smw[e * 64 + 32 + j] = sw;
      }
    }
    __syncthreads();
    if (K == 8) {
      // Warp ranges (as in the segmented gather, csrc/seg.cu): the segment's token pairs are split
      // into 16 contiguous warp ranges; a warp streams 32-pair windows (U in flight), computes each
      // record's contribution separately, keeps running sums of its current chunk and reduces them
      // at every chunk boundary it crosses; interior windows carry no per-lane validity logic.
      const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
      const int64_t m0 = r0 >> 1, m1 = (r1 + 1) >> 1;
      const int64_t perw = (m1 - m0 + nwarps - 1) / nwarps;
      const int64_t wm0 = min(m1, m0 + perw * warp), wm1 = min(m1, wm0 + perw);
      if (wm0 < wm1) {
        if (onehot) dedup_warp_range<2>(plane, wm0, wm1, r0, r1, bounds, C, base, slot, slot8, src, lane,
                                        hop_sums, uniq_sums, dedup_sums, &s_ol);
        else if (fast) dedup_warp_range<1>(plane, wm0, wm1, r0, r1, bounds, C, base, slot, slot8, src, lane,
                                           hop_sums, uniq_sums, dedup_sums, &s_ol);
        else dedup_warp_range<0>(plane, wm0, wm1, r0, r1, bounds, C, base, slot, slot8, src, lane,
                                 hop_sums, uniq_sums, dedup_sums, &s_ol);
      }
      g += r1 - r0;
      continue;
    }
    int c = 0;
    {
      int lo = 0, hi = C;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(bounds + mid) <= r0) lo = mid; else hi = mid;
      }
      c = lo;
    }
    int64_t cend = __ldg(bounds + c + 1);
    for (int64_t t = r0; t < r1;) {
      // chunk piece [t, te): walk forward from the previous chunk, skipping empty ones (K != 8)
      while (cend <= t && c + 1 < C) cend = __ldg(bounds + (++c) + 1);
      const int64_t te = min(r1, cend);
      uint32_t hop[4] = {0, 0, 0, 0}, uq[4] = {0, 0, 0, 0}, dd[4] = {0, 0, 0, 0};
      for (int64_t r = t + threadIdx.x; r < te; r += blockDim.x) {
        uint32_t ids[kDedupMaxK];
        for (int k = 0; k < K; ++k) ids[k] = plane[r * K + k];
        uint32_t srvw[kDedupMaxK];
        for (int k = 0; k < K; ++k) {
          const uint32_t a = base + ((ids[k] << 8) | slot);
          const uint32_t pw = lds32(a);
          const uint32_t sw = lds32(a + 128);
          srvw[k] = sw;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t s = (sw >> (8 * q)) & 0xffu;
            const uint32_t p = (pw >> (8 * q)) & 0xffu;
            hop[q] += p;
            bool first = true;
            for (int j = 0; j < k; ++j) first &= ((srvw[j] >> (8 * q)) & 0xffu) != s;
            if (first) {
              dd[q] += p;
              uq[q] += (s != ((src >> (8 * q)) & 0xffu)) ? 1u : 0u;
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned long long h = warp_sum_u64(hop[q]), u = warp_sum_u64(uq[q]), d = warp_sum_u64(dd[q]);
        if (lane == 0) {
          if (h) atomic_add_i64(hop_sums + (int64_t)q * C + c, (int64_t)h);
          if (u) atomic_add_i64(uniq_sums + (int64_t)q * C + c, (int64_t)u);
          if (d) atomic_add_i64(dedup_sums + (int64_t)q * C + c, (int64_t)d);
        }
      }
      t = te;
    }
    g += r1 - r0;
  }
}

cudaError_t launch_dedup(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K,
                         const int64_t* bounds, int C, const uint32_t* tables, const uint32_t* srv_tables,
                         const uint8_t* src_srv, int64_t* hop_sums, int64_t* uniq_sums, int64_t* dedup_sums,
                         cudaStream_t s) {
  const int smem = 256 * 256;
  int per_sm = 0;
  cudaError_t e = prepare_kernel((const void*)dedup_kernel, kDedupThreads, smem, &per_sm);
  if (e != cudaSuccess) return e;
  const int nsm = device_sm_count();
  const int64_t records = (t1 - t0) * (int64_t)L;
  int64_t grid = (int64_t)nsm * max(1, per_sm);
  grid = max((int64_t)1, min(grid, (records + 4095) / 4096));
  dedup_kernel<<<(unsigned)grid, kDedupThreads, smem, s>>>(planes, stride, t0, t1, L, K, bounds, C, tables, srv_tables, src_srv,
                                                 hop_sums, uniq_sums, dedup_sums);
  return cudaGetLastError();
}

// server-id tables: byte j of tables[(l*256 + e)] = server_of[topo_of[q]][assign[q][l][e]] for q = j
__global__ void pack_srv_kernel(const int32_t* __restrict__ server_of, int T, const int32_t* __restrict__ assign,
                                const int32_t* __restrict__ topo_of, int P, int L, int E, int S,
                                uint32_t* __restrict__ tables, int64_t* err) {
  const int64_t n = (int64_t)L * 256;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(i % 256), l = (int)(i / 256);
    uint32_t w = 0;
    if (e < E) {
      for (int q = 0; q < P; ++q) {
        const int32_t s = assign[((int64_t)q * L + l) * E + e];
        const int32_t tp = topo_of[q];
        if (s < 0 || s >= S || tp < 0 || tp >= T) { report_err(err, MP_DATA_UNPLACED, l, e); continue; }
        const int32_t sv = server_of[(int64_t)tp * S + s];
        if (sv < 0 || sv > 255) { report_err(err, MP_DATA_UNPLACED, l, e); continue; }
        w |= (uint32_t)sv << (8 * q);
      }
    }
    tables[i] = w;
  }
}

cudaError_t launch_pack_srv(const int32_t* server_of, int T, const int32_t* assign, const int32_t* topo_of, int P,
                            int L, int E, int S, uint32_t* tables, int64_t* err, cudaStream_t s) {
  const int64_t n = (int64_t)L * 256;
  pack_srv_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(server_of, T, assign, topo_of, P, L, E, S, tables, err);
  return cudaGetLastError();
}

}  // namespace mp
