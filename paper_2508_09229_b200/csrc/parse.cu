// Trace ingestion on the device.
//
// Text format: header line, then one token per line
//   chunk_id \t layer0:e,e,...,e \t layer1:... \n      ("layer" prefix optional, K ids per layer)
// The host copies the file bytes to the device once; then
//   1. mp_count_newlines / mp_find_newlines: per-block '\n' counts -> (host prefix sum of a few
//      thousand block counts) -> every line's end offset, written in order;
//   2. mp_parse_trace_text: one thread per line runs a small state machine over its bytes
//      (16-byte aligned vector reads cached in registers), validates the structure, the layer
//      labels, the id range (< E) and the K ids' distinctness, and writes the ids straight into
//      the layer-major planes (neighbouring threads = neighbouring tokens, so each layer's
//      K-byte records are stored coalesced) plus the chunk id per token.
// Errors: err[0] = min over bad lines of (line_index * 16 + code) (caller initialises it to
// INT64_MAX); codes: 1 structure, 2 layer label, 3 id >= E, 4 wrong id count, 5 duplicate id,
// 6 chunk id overflow.  Any K <= E <= 256.
#include "common.cuh"

namespace mp {

constexpr int kNlBlock = 1 << 16;

__global__ void count_nl_kernel(const uint8_t* __restrict__ text, int64_t n, int64_t* __restrict__ counts) {
  __shared__ int s_cnt;
  const int64_t b0 = (int64_t)blockIdx.x * kNlBlock;
  const int64_t b1 = min(n, b0 + kNlBlock);
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  int c = 0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) c += text[i] == '\n';
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = s_cnt;
}

// one warp per block: ordered compaction of '\n' positions with ballot/popc
__global__ void find_nl_kernel(const uint8_t* __restrict__ text, int64_t n, const int64_t* __restrict__ offsets,
                               int64_t* __restrict__ pos) {
  const int64_t b0 = (int64_t)blockIdx.x * kNlBlock;
  const int64_t b1 = min(n, b0 + kNlBlock);
  const int lane = threadIdx.x;
  int64_t out = offsets[blockIdx.x];
  for (int64_t i = b0; i < b1; i += 32) {
    const int64_t j = i + lane;
    const bool nl = j < b1 && text[j] == '\n';
    const uint32_t m = __ballot_sync(0xffffffffu, nl);
    if (nl) pos[out + __popc(m & ((1u << lane) - 1u))] = j;
    out += __popc(m);
  }
}

struct ByteReader {
  const uint8_t* text;
  int64_t blk = -1;
  uint4 v;
  __device__ __forceinline__ uint32_t get(int64_t p) {
    const int64_t b = p >> 4;
    if (b != blk) {
      v = __ldg(reinterpret_cast<const uint4*>(text) + b);
      blk = b;
    }
    const int o = (int)(p & 15);
    const uint32_t w = o < 8 ? (o < 4 ? v.x : v.y) : (o < 12 ? v.z : v.w);
    return (w >> (8 * (o & 3))) & 0xffu;
  }
};

// text must be readable up to the next 16-byte boundary past the last byte (caller pads)
__global__ void __launch_bounds__(256) parse_kernel(const uint8_t* __restrict__ text, const int64_t* __restrict__ ends,
                                                    int64_t first_start, int64_t n_lines, int L, int K, int E,
                                                    uint8_t* __restrict__ planes, int64_t stride,
                                                    int64_t* __restrict__ chunk_ids, int64_t* __restrict__ err) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_lines;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = t == 0 ? first_start : ends[t - 1] + 1;
    int64_t end = ends[t];
    ByteReader rd{text};
    if (end > p && rd.get(end - 1) == '\r') --end;
    int code = 0;
    // chunk id
    uint64_t cid = 0;
    int nd = 0;
    while (p < end) {
      const uint32_t ch = rd.get(p);
      if (ch < '0' || ch > '9') break;
      if (cid > 99999999999999999ull) { code = 6; break; }
      cid = cid * 10 + (ch - '0');
      ++p;
      ++nd;
    }
    if (!code && (nd == 0 || p >= end || rd.get(p) != '\t')) code = 1;
    ++p;
    uint32_t ids[8];
    for (int l = 0; l < L && !code; ++l) {
      uint32_t seen[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // 256-bit set of this record's ids
      uint8_t* out = planes + (int64_t)l * stride + t * K;
      if (p < end && rd.get(p) == 'l') {  // optional "layer" prefix
        const char* lit = "layer";
        for (int i = 0; i < 5 && !code; ++i, ++p)
          if (p >= end || rd.get(p) != (uint32_t)lit[i]) code = 1;
        if (code) break;
      }
      uint32_t lab = 0;
      nd = 0;
      while (p < end) {
        const uint32_t ch = rd.get(p);
        if (ch < '0' || ch > '9') break;
        lab = lab * 10 + (ch - '0');
        if (lab > 1000000u) break;
        ++p;
        ++nd;
      }
      if (nd == 0 || p >= end || rd.get(p) != ':') { code = 1; break; }
      if (lab != (uint32_t)l) { code = 2; break; }
      ++p;
      for (int k = 0; k < K; ++k) {
        uint32_t v = 0;
        nd = 0;
        while (p < end) {
          const uint32_t ch = rd.get(p);
          if (ch < '0' || ch > '9') break;
          v = v * 10 + (ch - '0');
          if (v > 100000u) v = 100000u;
          ++p;
          ++nd;
        }
        if (nd == 0) { code = 4; break; }
        if (v >= (uint32_t)E) { code = 3; break; }
        if (seen[v >> 5] & (1u << (v & 31))) { code = 5; break; }
        seen[v >> 5] |= 1u << (v & 31);
        if (K == 8) ids[k] = v;
        else out[k] = (uint8_t)v;
        const uint32_t ch = p < end ? rd.get(p) : '\n';
        const bool last_k = k == K - 1;
        if (!last_k) {
          if (ch != ',') { code = (ch == '\t' || ch == '\n') ? 4 : 1; break; }
        } else {
          const bool last_l = l == L - 1;
          if (ch == ',') { code = 4; break; }
          if (last_l ? (p != end) : (ch != '\t')) { code = (ch == '\t') ? 1 : 1; break; }
        }
        ++p;
      }
      if (code) break;
      if (K == 8) {  // one coalesced 8-byte store per record
        uint2 w;
        w.x = ids[0] | (ids[1] << 8) | (ids[2] << 16) | (ids[3] << 24);
        w.y = ids[4] | (ids[5] << 8) | (ids[6] << 16) | (ids[7] << 24);
        *reinterpret_cast<uint2*>(out) = w;
      }
    }
    if (code) {
      atomicMin(reinterpret_cast<unsigned long long*>(err), (unsigned long long)(t * 16 + code));
    } else {
      chunk_ids[t] = (int64_t)cid;
    }
  }
}

cudaError_t launch_count_nl(const uint8_t* text, int64_t n, int64_t* counts, cudaStream_t s) {
  const int64_t nb = (n + kNlBlock - 1) / kNlBlock;
  if (nb == 0) return cudaSuccess;
  count_nl_kernel<<<(unsigned)nb, 256, 0, s>>>(text, n, counts);
  return cudaGetLastError();
}

cudaError_t launch_find_nl(const uint8_t* text, int64_t n, const int64_t* offsets, int64_t* pos, cudaStream_t s) {
  const int64_t nb = (n + kNlBlock - 1) / kNlBlock;
  if (nb == 0) return cudaSuccess;
  find_nl_kernel<<<(unsigned)nb, 32, 0, s>>>(text, n, offsets, pos);
  return cudaGetLastError();
}

cudaError_t launch_parse(const uint8_t* text, const int64_t* ends, int64_t first_start, int64_t n_lines, int L, int K,
                         int E, uint8_t* planes, int64_t stride, int64_t* chunk_ids, int64_t* err, cudaStream_t s) {
  if (n_lines <= 0) return cudaSuccess;
  const int nsm = device_sm_count();
  const int64_t want = (n_lines + 255) / 256;
  parse_kernel<<<(unsigned)min(want, (int64_t)nsm * 8), 256, 0, s>>>(text, ends, first_start, n_lines, L, K, E, planes,
                                                                      stride, chunk_ids, err);
  return cudaGetLastError();
}

}  // namespace mp

// ---- text encoder: write_trace on the device (canonical "cid\tlayer<l>:e,..,e\t...\n") ------
namespace mp {

__device__ __forceinline__ int ndigits(uint64_t v) {
  int n = 1;
  while (v >= 10) { v /= 10; ++n; }
  return n;
}

__device__ __forceinline__ int64_t put_uint(uint8_t* out, int64_t p, uint64_t v) {
  const int n = ndigits(v);
  for (int i = n - 1; i >= 0; --i) { out[p + i] = (uint8_t)('0' + v % 10); v /= 10; }
  return p + n;
}

template <bool WRITE>
__global__ void __launch_bounds__(256) format_kernel(const uint8_t* __restrict__ planes, int64_t stride, int64_t t0,
                                                     int64_t n, int L, int K, const int64_t* __restrict__ cids,
                                                     int64_t* __restrict__ lens_or_offsets, uint8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = t0 + i;
    if (!WRITE) {
      int64_t len = ndigits((uint64_t)cids[i]) + 1;  // cid + '\t'
      for (int l = 0; l < L; ++l) {
        len += 5 + ndigits((uint64_t)l) + 1 + (K - 1) + 1;  // "layer" l ':' commas '\t'|'\n'
        const uint8_t* rec = planes + (int64_t)l * stride + t * K;
        for (int k = 0; k < K; ++k) len += ndigits(rec[k]);
      }
      lens_or_offsets[i] = len;
    } else {
      int64_t p = lens_or_offsets[i];
      p = put_uint(out, p, (uint64_t)cids[i]);
      out[p++] = '\t';
      for (int l = 0; l < L; ++l) {
        out[p++] = 'l'; out[p++] = 'a'; out[p++] = 'y'; out[p++] = 'e'; out[p++] = 'r';
        p = put_uint(out, p, (uint64_t)l);
        out[p++] = ':';
        const uint8_t* rec = planes + (int64_t)l * stride + t * K;
        for (int k = 0; k < K; ++k) {
          p = put_uint(out, p, rec[k]);
          if (k + 1 < K) out[p++] = ',';
        }
        out[p++] = (l + 1 < L) ? '\t' : '\n';
      }
    }
  }
}

cudaError_t launch_format(bool write, const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K,
                          const int64_t* cids, int64_t* lens_or_offsets, uint8_t* out, cudaStream_t s) {
  const int64_t n = t1 - t0;
  if (n <= 0) return cudaSuccess;
  const int nsm = device_sm_count();
  const unsigned grid = (unsigned)min((n + 255) / 256, (int64_t)nsm * 16);
  if (write) format_kernel<true><<<grid, 256, 0, s>>>(planes, stride, t0, n, L, K, cids, lens_or_offsets, out);
  else format_kernel<false><<<grid, 256, 0, s>>>(planes, stride, t0, n, L, K, cids, lens_or_offsets, out);
  return cudaGetLastError();
}

}  // namespace mp
