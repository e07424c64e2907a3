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
#ifndef MP_DEDUP_U
#define MP_DEDUP_U 2  // 32-pair windows in flight per warp (K = 8 warp-range path)
#endif

// Fast K = 8 record for pe bytes <= 31 and server ids < 128 (checked per layer by the CTA).  Row
// layout of the fast path: slot lane*8 holds {pe word, server word} (one LDS.64 per pick), and bit 7
// of each server byte flags "this is the source server of the layer for that placement".  With the
// server id in bits 0-6, t = ((a ^ b) | 0x80808080) - 0x01010101 has bit 7 of a byte set iff the
// ids differ (each byte of (a^b)|0x80 is >= 0x80, so subtracting 1 never borrows across bytes; the
// flag bit is ignored), so "new server" = AND of t over the earlier picks, read from bit 7 directly
// (PRMT's sign-replicate turns it into the dedup mask); a record's hop and dedup sums fit u8 lanes
// (8 * 31 < 256); the source server is removed once per record (distinct servers - [src in set],
// the latter the OR of the flag bits).
__device__ __forceinline__ uint32_t bytes_ne7(uint32_t a, uint32_t b) {
  return ((a ^ b) | 0x80808080u) - 0x01010101u;
}
__device__ __forceinline__ void dedup_record8_fast(uint2 v, uint32_t base, uint32_t slot8,
                                                   uint32_t (&hop16)[2], uint32_t& uq8, uint32_t (&dd16)[2]) {
  const uint32_t wv[2] = {v.x, v.y};
  uint32_t sw[8], pw[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint2 r = lds64(base + prmt(wv[k >> 2], slot8, sel_row(k & 3)));
    pw[k] = r.x;
    sw[k] = r.y;
  }
  uint32_t h8 = pw[0], d8 = pw[0], n8 = 0x01010101u, srcany = sw[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    uint32_t nw = bytes_ne7(sw[k], sw[0]);
#pragma unroll
    for (int j = 1; j < k; ++j) nw &= bytes_ne7(sw[k], sw[j]);
    const uint32_t f = (nw >> 7) & 0x01010101u;  // 1 in bytes whose server is new in the record
    h8 += pw[k];
    d8 += pw[k] & (f * 0xffu);                    // byte mask by IMAD: keeps the ALU pipe free
    n8 += f;
    srcany |= sw[k];
  }
  uq8 += n8 - ((srcany >> 7) & 0x01010101u);  // distinct remote destination servers per lane
  hop16[0] += h8 & 0x00ff00ffu;
  hop16[1] += (h8 >> 8) & 0x00ff00ffu;
  dd16[0] += d8 & 0x00ff00ffu;
  dd16[1] += (d8 >> 8) & 0x00ff00ffu;
}

__global__ void __launch_bounds__(kDedupThreads, 2) dedup_kernel(const uint8_t* __restrict__ planes, int64_t stride, int64_t t0,
                                                    int64_t t1, int L, int K, const int64_t* __restrict__ bounds,
                                                    int C, const uint32_t* __restrict__ tables,
                                                    const uint32_t* __restrict__ srv_tables,
                                                    const uint8_t* __restrict__ src_srv, int64_t* __restrict__ hop_sums,
                                                    int64_t* __restrict__ uniq_sums, int64_t* __restrict__ dedup_sums) {
  extern __shared__ __align__(128) uint8_t sm[];  // 256 rows x 256 B
  __shared__ uint32_t s_src;                      // 4 source-server bytes of this layer
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
    const uint32_t src = s_src;
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
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
      // into 16 contiguous warp ranges; a warp streams 32-pair windows (4 in flight), computes each
      // record's contribution separately, keeps running sums of its current chunk and reduces them
      // at every chunk boundary it crosses -- so short chunks cost one warp reduction per boundary
      // instead of a pass of the whole CTA over every (layer, chunk) piece.
      const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
      const int64_t m0 = r0 >> 1, m1 = (r1 + 1) >> 1;
      const int64_t perw = (m1 - m0 + nwarps - 1) / nwarps;
      const int64_t wm0 = min(m1, m0 + perw * warp), wm1 = min(m1, wm0 + perw);
      if (wm0 < wm1) {
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
        const int ra = (int)(wt0 - T0), rb = (int)(wt1 - T0);
        auto rel = [&](int64_t x) { return (int)min(x - T0, (int64_t)0x7fffffff); };
        int nbr = rel(__ldg(bounds + c + 1));
        uint32_t h16[2] = {0, 0}, d16[2] = {0, 0}, u8 = 0;          // running, narrow lanes
        uint32_t hop[4] = {0, 0, 0, 0}, uq[4] = {0, 0, 0, 0}, dd[4] = {0, 0, 0, 0};  // running, u32
        int since = 0, recs = 0;
        auto widen = [&]() {
          hop[0] += h16[0] & 0xffffu; hop[2] += h16[0] >> 16; hop[1] += h16[1] & 0xffffu; hop[3] += h16[1] >> 16;
          dd[0] += d16[0] & 0xffffu; dd[2] += d16[0] >> 16; dd[1] += d16[1] & 0xffffu; dd[3] += d16[1] >> 16;
#pragma unroll
          for (int q = 0; q < 4; ++q) uq[q] += (u8 >> (8 * q)) & 0xffu;
          h16[0] = h16[1] = d16[0] = d16[1] = u8 = 0;
        };
        auto flush = [&](int cc) {  // warp-uniform: running sums of chunk cc -> the three outputs
          widen();
          uint32_t v[16] = {hop[0], hop[1], hop[2], hop[3], uq[0], uq[1], uq[2], uq[3],
                            dd[0], dd[1], dd[2], dd[3], 0u, 0u, 0u, 0u};
          int q = 0;
          const uint32_t tot = warp_reduce_scatter<16>(v, lane, &q);
          if ((lane & 1) == 0 && tot && q < 12) {
            int64_t* dst = q < 4 ? hop_sums : q < 8 ? uniq_sums : dedup_sums;
            atomic_add_i64(dst + (int64_t)(q & 3) * C + cc, (int64_t)tot);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) hop[i] = uq[i] = dd[i] = 0;
          recs = 0;
        };
        auto rec = [&](uint2 w, uint32_t (&h_)[2], uint32_t& u_, uint32_t (&d_)[2]) {
          if (fast) dedup_record8_fast(w, base, slot8, h_, u_, d_);
          else dedup_record8(w, base, slot, src, h_, u_, d_);
        };
        auto add_rec = [&](const uint32_t (&h_)[2], uint32_t u_, const uint32_t (&d_)[2]) {
          h16[0] += h_[0]; h16[1] += h_[1]; d16[0] += d_[0]; d16[1] += d_[1]; u8 += u_;
        };
        const uint4* __restrict__ pv = reinterpret_cast<const uint4*>(plane) + wm0;
        for (int rw = 0; rw < npairs; rw += 32 * MP_DEDUP_U) {
          uint4 x[MP_DEDUP_U];
#pragma unroll
          for (int u = 0; u < MP_DEDUP_U; ++u) {
            const int r = rw + u * 32 + lane;
            if (r < npairs) {
              const int4 vv = ldg_stream(pv + r);
              x[u] = make_uint4((uint32_t)vv.x, (uint32_t)vv.y, (uint32_t)vv.z, (uint32_t)vv.w);
            } else {
              x[u] = make_uint4(0, 0, 0, 0);
            }
          }
#pragma unroll
          for (int u = 0; u < MP_DEDUP_U; ++u) {
            const int rfirst = rw + u * 32;
            if (rfirst >= npairs) break;  // warp-uniform
            const int r = rfirst + lane;
            const int tA = 2 * r, tB = tA + 1;
            const bool vA = r < npairs && tA >= ra && tA < rb;
            const bool vB = r < npairs && tB >= ra && tB < rb;
            uint32_t hA[2] = {0, 0}, dA[2] = {0, 0}, uA = 0, hB[2] = {0, 0}, dB[2] = {0, 0}, uB = 0;
            rec(make_uint2(x[u].x, x[u].y), hA, uA, dA);
            rec(make_uint2(x[u].z, x[u].w), hB, uB, dB);
            const int wlast = min(2 * (rfirst + 31) + 1, rb - 1);
            if (nbr > wlast) {
              if (vA) add_rec(hA, uA, dA);
              if (vB) add_rec(hB, uB, dB);
            } else {
              bool doneA = !vA, doneB = !vB;
              while (nbr <= wlast) {  // boundary inside the window: records < nb belong to chunk c
                if (!doneA && tA < nbr) { add_rec(hA, uA, dA); doneA = true; }
                if (!doneB && tB < nbr) { add_rec(hB, uB, dB); doneB = true; }
                flush(c);
                since = 0;
                ++c;  // c < C - 1 here: bounds[C] >= the trace end > the window
                nbr = rel(__ldg(bounds + c + 1));
              }
              if (!doneA) add_rec(hA, uA, dA);
              if (!doneB) add_rec(hB, uB, dB);
            }
            // narrow lanes: u16 hop/dedup sums take 8 records (8 x 8 x 255 < 2^16), u8 unique counts 31
            if (++since == 4) {
              widen();
              since = 0;
              // u32 running sums: a warp's total over 32 lanes x 2^15 records x 2040 stays below 2^32
              if ((recs += 8) >= (1 << 15)) flush(c);
            }
          }
        }
        flush(c);
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
  cudaError_t e = cudaFuncSetAttribute(dedup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dedup_kernel, kDedupThreads, smem);
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
