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
      // chunk piece [t, te): walk forward from the previous chunk, skipping empty ones
      while (cend <= t && c + 1 < C) cend = __ldg(bounds + (++c) + 1);
      const int64_t te = min(r1, cend);
      uint32_t hop[4] = {0, 0, 0, 0}, uq[4] = {0, 0, 0, 0}, dd[4] = {0, 0, 0, 0};
      if (K == 8) {
        // SIMD-within-a-register path over 16-byte vectors (two records each), 4 vectors in flight
        // per thread; lane sums are widened every main-loop iteration (8 records, u16 lanes:
        // 8*8*255 < 2^16) and after every single-record step
        uint32_t h16[2] = {0, 0}, d16[2] = {0, 0}, u8 = 0;
        auto widen = [&]() {
          hop[0] += h16[0] & 0xffffu; hop[2] += h16[0] >> 16; hop[1] += h16[1] & 0xffffu; hop[3] += h16[1] >> 16;
          dd[0] += d16[0] & 0xffffu; dd[2] += d16[0] >> 16; dd[1] += d16[1] & 0xffffu; dd[3] += d16[1] >> 16;
#pragma unroll
          for (int q = 0; q < 4; ++q) uq[q] += (u8 >> (8 * q)) & 0xffu;
          h16[0] = h16[1] = d16[0] = d16[1] = u8 = 0;
        };
        auto rec8 = [&](uint2 w, uint32_t b_, uint32_t s_, uint32_t src_, uint32_t (&h_)[2], uint32_t& u_,
                        uint32_t (&d_)[2]) {
          if (fast) dedup_record8_fast(w, b_, slot8, h_, u_, d_);
          else dedup_record8(w, b_, s_, src_, h_, u_, d_);
        };
        const int64_t va = (t + 1) >> 1, vb = te >> 1;  // full vectors cover records [2va, 2vb)
        const int T = blockDim.x;
        if ((t & 1) && threadIdx.x == 0) {  // lone head record
          rec8(__ldg(reinterpret_cast<const uint2*>(plane + t * 8)), base, slot, src, h16, u8, d16);
          widen();
        }
        if ((te & 1) && te - 1 > t && threadIdx.x == T - 1) {  // lone tail record
          rec8(__ldg(reinterpret_cast<const uint2*>(plane + (te - 1) * 8)), base, slot, src, h16, u8, d16);
          widen();
        }
        const uint4* __restrict__ pv = reinterpret_cast<const uint4*>(plane);
        int64_t v = va + threadIdx.x;
        for (; v + 3 * T < vb; v += 4 * T) {
          uint4 x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int4 r = ldg_stream(pv + v + u * T);
            x[u] = make_uint4((uint32_t)r.x, (uint32_t)r.y, (uint32_t)r.z, (uint32_t)r.w);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            rec8(make_uint2(x[u].x, x[u].y), base, slot, src, h16, u8, d16);
            rec8(make_uint2(x[u].z, x[u].w), base, slot, src, h16, u8, d16);
          }
          widen();
        }
        for (; v < vb; v += T) {
          const int4 r = ldg_stream(pv + v);
          const uint4 x = make_uint4((uint32_t)r.x, (uint32_t)r.y, (uint32_t)r.z, (uint32_t)r.w);
          rec8(make_uint2(x.x, x.y), base, slot, src, h16, u8, d16);
          rec8(make_uint2(x.z, x.w), base, slot, src, h16, u8, d16);
          widen();
        }
      } else
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
