// Device kernels of the placement-search loop and of the batched scorer's operands
// (A18): per-expert cost gather, swap perturbation in the cost domain, batch objectives, argmin and
// acceptance, and the Eq. (1) objective value.  Everything a search iteration needs stays on the
// device; the host enqueues the iterations and reads the history once at the end.
//
// Swapping the devices of experts x and y of layer l swaps pe[l][x] and pe[l][y] (pe = p[l, assign]),
// so a candidate's cost row is the incumbent's with its swaps applied: the perturbation writes the
// u8 cost rows the tensor-core contraction reads (mp_contract_tc_u8) and the swap list, and only the
// accepted candidate's swaps are replayed on the int32 assignment.
#include <cfloat>

#include <algorithm>
#include "common.cuh"

namespace mp {
namespace {

// Philox4x32-10 (Salmon et al., SC'11), the generator of csrc/gen.cu, for the swap draws.
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__global__ void pe_gather_kernel(const uint8_t* __restrict__ cost, int T, int L, int S, const int32_t* __restrict__ topo_S,
                                 const int32_t* __restrict__ assign, const int32_t* __restrict__ topo_of, int P, int E,
                                 uint8_t* __restrict__ pe, int64_t ldpe, int64_t* err) {
  const int64_t LE = (int64_t)L * E;
  const int q = blockIdx.y;
  if (q >= P) return;
  const int t = topo_of ? topo_of[q] : 0;
  const int St = (topo_S && t >= 0 && t < T) ? topo_S[t] : S;  // the placement's own device count
  const uint8_t* cq = cost + (int64_t)t * L * S;
  const int32_t* aq = assign + (int64_t)q * LE;
  uint8_t* out = pe + (int64_t)q * ldpe;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ldpe; i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t v = 0;
    if (i < LE) {
      const int l = (int)(i / E);
      const int s = __ldg(aq + i);
      if (s < 0 || s >= St || t < 0 || t >= T) {
        report_err(err, MP_DATA_UNPLACED, q, i);
      } else {
        v = __ldg(cq + (int64_t)l * S + s);
      }
    }
    out[i] = v;
  }
}

// Candidate b = the incumbent's cost row with n_swaps within-layer swaps; draw j of candidate b in
// iteration `iter` is Philox(b, iter, j, 0x53574150 'SWAP') keyed by the seed.  One CTA per candidate:
// the row is copied with 16-byte vectors, then thread 0 applies the swaps in order (a later swap may
// touch an earlier one's experts, so they are sequential) and records them.
__global__ void perturb_pe_kernel(const uint8_t* __restrict__ pe_cur, int L, int E, int B, int n_swaps, uint64_t seed,
                                  int64_t iter, uint8_t* __restrict__ pe_out, int64_t ldpe, int32_t* __restrict__ swaps) {
  const int b = blockIdx.x;
  if (b >= B) return;
  uint8_t* row = pe_out + (int64_t)b * ldpe;
  const int64_t n16 = ldpe / 16;
  const uint4* src = reinterpret_cast<const uint4*>(pe_cur);
  uint4* dst = reinterpret_cast<uint4*>(row);
  for (int64_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    for (int j = 0; j < n_swaps; ++j) {
      const uint4 r = philox(make_uint4((uint32_t)b, (uint32_t)iter, (uint32_t)j, 0x53574150u), key);
      const int l = (int)(((uint64_t)r.x * (uint32_t)L) >> 32);
      const int x = (int)(((uint64_t)r.y * (uint32_t)E) >> 32);
      const int y = (int)(((uint64_t)r.z * (uint32_t)E) >> 32);
      uint8_t* p = row + (int64_t)l * E;
      const uint8_t t = p[x];
      p[x] = p[y];
      p[y] = t;
      int32_t* sw = swaps + ((int64_t)b * n_swaps + j) * 3;
      sw[0] = l;
      sw[1] = x;
      sw[2] = y;
    }
  }
}

// obj[b] from the exact per-chunk hop sums of candidate b: kind 0 = token-weighted mean hops,
// 1 = mean + lam * population std of the per-chunk means, 2 = worst per-chunk mean.  Empty chunks
// are skipped.  One warp per candidate; the total is an exact int64, the mean one
// correctly rounded division (identical to EvalReport.mean_hops_per_token).
__global__ void batch_objective_kernel(const int64_t* __restrict__ sums, const int64_t* __restrict__ tokens, int B,
                                       int C, int kind, double lam, double* __restrict__ obj) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= B) return;
  const int64_t* s = sums + (int64_t)warp * C;
  long long tot = 0, ntok = 0;
  int nk = 0;
  for (int c = lane; c < C; c += 32) {
    const int64_t n = tokens[c];
    if (n > 0) {
      tot += s[c];
      ntok += n;
      ++nk;
    }
  }
  for (int o = 16; o; o >>= 1) {
    tot += __shfl_xor_sync(0xffffffffu, tot, o);
    ntok += __shfl_xor_sync(0xffffffffu, ntok, o);
    nk += __shfl_xor_sync(0xffffffffu, nk, o);
  }
  const double mean = ntok ? (double)tot / (double)ntok : 0.0;
  double v = mean;
  if (kind != 0 && nk > 0) {
    double acc = 0.0, mx = -DBL_MAX, msum = 0.0;
    for (int c = lane; c < C; c += 32)
      if (tokens[c] > 0) msum += (double)s[c] / (double)tokens[c];
    for (int o = 16; o; o >>= 1) msum += __shfl_xor_sync(0xffffffffu, msum, o);
    const double mu = msum / nk;
    for (int c = lane; c < C; c += 32) {
      if (tokens[c] > 0) {
        const double m = (double)s[c] / (double)tokens[c];
        acc += (m - mu) * (m - mu);
        mx = fmax(mx, m);
      }
    }
    for (int o = 16; o; o >>= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    v = kind == 1 ? mean + lam * sqrt(acc / nk) : mx;
  }
  if (lane == 0) obj[warp] = v;
}

// Single CTA: best = argmin obj (lowest index on ties); if obj[best] < *cur_obj the incumbent takes
// candidate best: its swaps are replayed on the int32 assignment and the u8 cost row, *cur_obj is
// updated.  history[iter] = incumbent objective after the step, *best_out = {index or -1}.
__global__ void accept_kernel(const double* __restrict__ obj, int B, const int32_t* __restrict__ swaps, int n_swaps,
                              int E, int32_t* __restrict__ assign, uint8_t* __restrict__ pe_cur, double* cur_obj,
                              double* history, int64_t iter, int64_t* accepted) {
  __shared__ double sv[1024];
  __shared__ int si[1024];
  double v = DBL_MAX;
  int idx = 0x7fffffff;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const double o = obj[i];
    if (o < v || (o == v && i < idx)) {
      v = o;
      idx = i;
    }
  }
  sv[threadIdx.x] = v;
  si[threadIdx.x] = idx;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double o = sv[threadIdx.x + w];
      const int j = si[threadIdx.x + w];
      if (o < sv[threadIdx.x] || (o == sv[threadIdx.x] && j < si[threadIdx.x])) {
        sv[threadIdx.x] = o;
        si[threadIdx.x] = j;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int best = si[0];
    const bool take = best < B && sv[0] < *cur_obj;
    if (take) {
      const int32_t* sw = swaps + (int64_t)best * n_swaps * 3;
      for (int j = 0; j < n_swaps; ++j) {
        const int64_t ox = (int64_t)sw[3 * j] * E + sw[3 * j + 1], oy = (int64_t)sw[3 * j] * E + sw[3 * j + 2];
        const int32_t ta = assign[ox];
        assign[ox] = assign[oy];
        assign[oy] = ta;
        const uint8_t tp = pe_cur[ox];
        pe_cur[ox] = pe_cur[oy];
        pe_cur[oy] = tp;
      }
      *cur_obj = sv[0];
    }
    history[iter] = *cur_obj;
    accepted[iter] = take ? best : -1;
  }
}

// Eq. (1) objective with float frequencies: obj[q] = sum_i f[i] * pe[q][i] (fixed reduction order:
// per-thread strided partial sums, then a shared-memory tree), one CTA per placement.
__global__ void objective_f64_kernel(const double* __restrict__ f, const uint8_t* __restrict__ pe, int64_t ldpe,
                                     int64_t LE, double* __restrict__ out) {
  __shared__ double part[256];
  const uint8_t* row = pe + (int64_t)blockIdx.x * ldpe;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < LE; i += 256) acc += f[i] * (double)row[i];
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = part[0];
}

}  // namespace

cudaError_t launch_pe_gather(const uint8_t* cost, int T, int L, int S, const int32_t* topo_S, const int32_t* assign,
                             const int32_t* topo_of, int P, int E, uint8_t* pe, int64_t ldpe, int64_t* err,
                             cudaStream_t s) {
  const int gx = (int)std::min<int64_t>((ldpe + 255) / 256, 64);
  pe_gather_kernel<<<dim3(gx, P), 256, 0, s>>>(cost, T, L, S, topo_S, assign, topo_of, P, E, pe, ldpe, err);
  return cudaGetLastError();
}

cudaError_t launch_perturb_pe(const uint8_t* pe_cur, int L, int E, int B, int n_swaps, uint64_t seed, int64_t iter,
                              uint8_t* pe_out, int64_t ldpe, int32_t* swaps, cudaStream_t s) {
  perturb_pe_kernel<<<B, 256, 0, s>>>(pe_cur, L, E, B, n_swaps, seed, iter, pe_out, ldpe, swaps);
  return cudaGetLastError();
}

cudaError_t launch_batch_objective(const int64_t* sums, const int64_t* tokens, int B, int C, int kind, double lam,
                                   double* obj, cudaStream_t s) {
  batch_objective_kernel<<<(B + 7) / 8, 256, 0, s>>>(sums, tokens, B, C, kind, lam, obj);
  return cudaGetLastError();
}

cudaError_t launch_accept(const double* obj, int B, const int32_t* swaps, int n_swaps, int E, int32_t* assign,
                          uint8_t* pe_cur, double* cur_obj, double* history, int64_t iter, int64_t* accepted,
                          cudaStream_t s) {
  accept_kernel<<<1, 1024, 0, s>>>(obj, B, swaps, n_swaps, E, assign, pe_cur, cur_obj, history, iter, accepted);
  return cudaGetLastError();
}

cudaError_t launch_objective_f64(const double* f, const uint8_t* pe, int64_t ldpe, int64_t LE, int P, double* out,
                                 cudaStream_t s) {
  objective_f64_kernel<<<P, 256, 0, s>>>(f, pe, ldpe, LE, out);
  return cudaGetLastError();
}

}  // namespace mp
