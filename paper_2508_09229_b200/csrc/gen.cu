// Trace synthesis and ingestion checks.
//
// gen: counter-based Zipf(s) top-K sampler (generate_trace).  Each
// (token t, layer l) record is produced by one thread from Philox4x32-10(counter = (t_lo,
// t_hi, l, k/4), key = seed): K successive draws without replacement over the integer rank
// weights w_r = cdf[r+1]-cdf[r].  Draw k maps u_k to x = floor(u_k * W_rem / 2^32) in the
// weight line with the already-chosen rank intervals removed (skip-over walk in ascending rank
// order), then binary-searches the rank (gen8_kernel for K <= 8: register-resident intervals and a
// guide-table search, the same ranks).  Rank -> expert through the layer's permutation.
// No floats, no rejection loop: bounded work and bit-identical to the oracle (oracle/gen.py).
#include "common.cuh"

namespace mp {

__host__ __device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                                                      uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#ifdef __CUDA_ARCH__
  const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
  const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
#else
  const uint64_t p0 = (uint64_t)M0 * c0, p1 = (uint64_t)M1 * c2;
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
  const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
  c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
}

__host__ __device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                        uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c0, c1, c2, c3, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}

template <int KMAX>
__global__ void __launch_bounds__(256) gen_kernel(uint64_t seed, int64_t t0, int64_t n, int L, int K, int E,
                                                  const uint32_t* __restrict__ cdf, const uint8_t* __restrict__ perm,
                                                  uint8_t* __restrict__ planes, int64_t stride) {
  __shared__ uint32_t s_cdf[kMaxE + 1];
  __shared__ uint8_t s_perm[kMaxE];
  const int l = blockIdx.y;
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_cdf[i] = cdf[i];
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_perm[i] = perm[(int64_t)l * E + i];
  __syncthreads();
  const uint32_t total = s_cdf[E];
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  uint8_t* out = planes + (int64_t)l * stride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t t = (uint64_t)(t0 + i);
    uint32_t ch[KMAX];  // chosen ranks, ascending
    int nch = 0;
    uint32_t rem = total;
    uint4 rnd = make_uint4(0, 0, 0, 0);
    uint32_t lo_word = 0, hi_word = 0;  // packed output bytes for K <= 8
    for (int k = 0; k < K; ++k) {
      if ((k & 3) == 0) rnd = philox4x32_10((uint32_t)t, (uint32_t)(t >> 32), (uint32_t)l, (uint32_t)(k >> 2), k0, k1);
      const uint32_t u = (k & 3) == 0 ? rnd.x : (k & 3) == 1 ? rnd.y : (k & 3) == 2 ? rnd.z : rnd.w;
      uint32_t x = (uint32_t)(((uint64_t)u * rem) >> 32);
      for (int j = 0; j < nch; ++j) {
        const uint32_t c = ch[j];
        if (s_cdf[c] <= x) x += s_cdf[c + 1] - s_cdf[c];
        else break;
      }
      int lo = 0, hi = E;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_cdf[mid] <= x) lo = mid; else hi = mid;
      }
      // insert lo into ch (ascending)
      int j = nch;
      while (j > 0 && ch[j - 1] > (uint32_t)lo) { ch[j] = ch[j - 1]; --j; }
      ch[j] = (uint32_t)lo;
      ++nch;
      rem -= s_cdf[lo + 1] - s_cdf[lo];
      const uint32_t e = s_perm[lo];
      if (KMAX <= 8) {
        if (k < 4) lo_word |= e << (8 * k); else hi_word |= e << (8 * (k - 4));
      } else {
        out[i * K + k] = (uint8_t)e;
      }
    }
    if (KMAX <= 8) {
      if (K == 8) {
        *reinterpret_cast<uint2*>(out + i * 8) = make_uint2(lo_word, hi_word);
      } else {
        for (int k = 0; k < K; ++k) out[i * K + k] = (uint8_t)((k < 4 ? lo_word >> (8 * k) : hi_word >> (8 * (k - 4))) & 0xffu);
      }
    }
  }
}

// K <= 8 (every BASELINE shape): the same draws with the state in registers.  The chosen ranks'
// intervals are kept as (start, weight) pairs sorted by start, fully unrolled, so the skip-over walk
// needs no shared-memory loads and nothing spills to local memory; the rank search starts from a
// guide table (guide[b] = the rank containing b * 2^gshift, 4096 buckets of the weight line) and
// walks forward while cdf[r + 1] <= x -- the same rank as the binary search (the largest r with
// cdf[r] <= x), at one or two probes for Zipf weights instead of eight dependent loads.
constexpr int kGuideBits = 12;

__global__ void __launch_bounds__(256) gen8_kernel(uint64_t seed, int64_t t0, int64_t n, int L, int K, int E,
                                                   const uint32_t* __restrict__ cdf, const uint8_t* __restrict__ perm,
                                                   uint8_t* __restrict__ planes, int64_t stride) {
  __shared__ uint32_t s_cdf[kMaxE + 1];
  __shared__ uint8_t s_perm[kMaxE];
  __shared__ uint8_t s_guide[1 << kGuideBits];
  const int l = blockIdx.y;
  for (int i = threadIdx.x; i <= E; i += blockDim.x) s_cdf[i] = cdf[i];
  for (int i = threadIdx.x; i < E; i += blockDim.x) s_perm[i] = perm[(int64_t)l * E + i];
  __syncthreads();
  const uint32_t total = s_cdf[E];
  // bucket b covers weight positions [b << gshift, (b + 1) << gshift); total <= 2^32
  int gshift = 0;
  while (gshift < 32 && ((uint64_t)1 << (gshift + kGuideBits)) < (uint64_t)total) ++gshift;
  for (int b = threadIdx.x; b < (1 << kGuideBits); b += blockDim.x) {
    const uint64_t pos = (uint64_t)b << gshift;
    int lo = 0, hi = E;  // largest r with cdf[r] <= pos (pos beyond the line: the last rank)
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if ((uint64_t)s_cdf[mid] <= pos) lo = mid; else hi = mid;
    }
    s_guide[b] = (uint8_t)lo;
  }
  __syncthreads();
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  uint8_t* out = planes + (int64_t)l * stride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t t = (uint64_t)(t0 + i);
    uint32_t cs[8], cw[8];  // chosen intervals (start, weight), ascending start
    uint32_t rem = total;
    uint32_t word[2] = {0u, 0u};
    uint4 rnd = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= K) break;
      if ((k & 3) == 0) rnd = philox4x32_10((uint32_t)t, (uint32_t)(t >> 32), (uint32_t)l, (uint32_t)(k >> 2), k0, k1);
      const uint32_t u = (k & 3) == 0 ? rnd.x : (k & 3) == 1 ? rnd.y : (k & 3) == 2 ? rnd.z : rnd.w;
      uint32_t x = (uint32_t)(((uint64_t)u * rem) >> 32);
      bool go = true;  // skip-over walk in ascending start order, stopping at the first interval past x
#pragma unroll
      for (int j = 0; j < k; ++j) {
        go = go && cs[j] <= x;
        if (go) x += cw[j];
      }
      int r = s_guide[x >> gshift];
      while (r + 1 < E && s_cdf[r + 1] <= x) ++r;
      const uint32_t st = s_cdf[r], w = s_cdf[r + 1] - st;
      // insert (st, w) at its place in the ascending list (compile-time indices only; starts of
      // drawn ranks are distinct, each having positive weight).  Downward, so cs[j] is still the old
      // value when position j is decided.
#pragma unroll
      for (int j = k; j > 0; --j) {
        const bool shift = cs[j - 1] > st;
        const bool here = !shift && (j == k || cs[j] > st);
        cs[j] = shift ? cs[j - 1] : here ? st : cs[j];
        cw[j] = shift ? cw[j - 1] : here ? w : cw[j];
      }
      const bool first = k == 0 || cs[0] > st;
      cs[0] = first ? st : cs[0];
      cw[0] = first ? w : cw[0];
      rem -= w;
      word[k >> 2] |= (uint32_t)s_perm[r] << (8 * (k & 3));
    }
    if (K == 8) {
      *reinterpret_cast<uint2*>(out + i * 8) = make_uint2(word[0], word[1]);
    } else {
      for (int k = 0; k < K; ++k) out[i * K + k] = (uint8_t)((word[k >> 2] >> (8 * (k & 3))) & 0xffu);
    }
  }
}

cudaError_t launch_gen(uint64_t seed, int64_t t0, int64_t t1, int L, int K, int E, const uint32_t* cdf,
                       const uint8_t* perm, uint8_t* planes, int64_t stride, cudaStream_t s) {
  const int64_t n = t1 - t0;
  if (n <= 0) return cudaSuccess;
  const int nsm = device_sm_count();
  const int64_t want = (n + 255) / 256;
  const unsigned gx = (unsigned)max((int64_t)1, min(want, (int64_t)nsm * 16 / max(1, L) + 1));
  dim3 grid(gx, L);
  if (K <= 8) gen8_kernel<<<grid, 256, 0, s>>>(seed, t0, n, L, K, E, cdf, perm, planes, stride);
  else if (K <= 32) gen_kernel<32><<<grid, 256, 0, s>>>(seed, t0, n, L, K, E, cdf, perm, planes, stride);
  else gen_kernel<kMaxE><<<grid, 256, 0, s>>>(seed, t0, n, L, K, E, cdf, perm, planes, stride);
  return cudaGetLastError();
}

// ---- ActivationTrace invariant check: ids < E, K distinct ids per (t, l) ----
// err = {flag, INT64_MAX - key_min, 0, count} with key = ((t*L + l) * 8 + code) of a violation;
// the host decodes the lowest-token violation from err[1].
__global__ void validate_kernel(const uint8_t* __restrict__ planes, int64_t stride, int64_t t0, int64_t t1,
                                int L, int K, int E, int64_t* __restrict__ err) {
  const int l = blockIdx.y;
  const uint8_t* plane = planes + (int64_t)l * stride;
  for (int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < t1; t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t seen[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int code = 0;
    for (int k = 0; k < K; ++k) {
      const uint32_t e = plane[t * K + k];
      if (e >= (uint32_t)E) { code = MP_DATA_EXPERT_RANGE; break; }
      const uint32_t bit = 1u << (e & 31);
      if (seen[e >> 5] & bit) { code = MP_DATA_DUPLICATE; break; }
      seen[e >> 5] |= bit;
    }
    if (code) {
      unsigned long long* e = reinterpret_cast<unsigned long long*>(err);
      const long long key = ((long long)t * L + l) * 8 + code;
      atomicMax(e, 1ull);
      atomicMax(reinterpret_cast<long long*>(e + 1), (long long)(0x7fffffffffffffffLL - key));
      atomicAdd(e + 3, 1ull);
    }
  }
}

cudaError_t launch_validate(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K, int E,
                            int64_t* err, cudaStream_t s) {
  const int64_t n = t1 - t0;
  if (n <= 0) return cudaSuccess;
  const int nsm = device_sm_count();
  const unsigned gx = (unsigned)max((int64_t)1, min((n + 255) / 256, (int64_t)nsm * 16 / max(1, L) + 1));
  validate_kernel<<<dim3(gx, L), 256, 0, s>>>(planes, stride, t0, t1, L, K, E, err);
  return cudaGetLastError();
}

}  // namespace mp
