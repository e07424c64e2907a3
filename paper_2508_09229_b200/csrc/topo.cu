// Small device prologue/epilogue kernels: hop matrix (BFS), device expansion, cost matrix,
// placement tables, ILP coefficients and the communication map.  All are microsecond-scale;
// they exist so the whole path stays device resident (no host round trips between stages).
#include "common.cuh"

namespace mp {

constexpr int kMaxNodes = 8192;
constexpr uint16_t kInf = 0xffffu;

// ---- all_pairs_hops: one CTA per source, level-synchronous BFS in smem ----
__global__ void __launch_bounds__(256) bfs_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                                  int n, const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                                  int n_dst, uint8_t* __restrict__ dist, int64_t* err) {
  __shared__ uint16_t d[kMaxNodes];
  __shared__ int changed;
  const int i = blockIdx.x;
  const int s = src[i];
  for (int v = threadIdx.x; v < n; v += blockDim.x) d[v] = kInf;
  __syncthreads();
  if (threadIdx.x == 0) d[s] = 0;
  __syncthreads();
  for (int level = 0; level < n; ++level) {
    if (threadIdx.x == 0) changed = 0;
    __syncthreads();
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
      if (d[v] != level) continue;
      for (int a = row_ptr[v]; a < row_ptr[v + 1]; ++a) {
        const int u = col[a];
        if (d[u] == kInf) { d[u] = (uint16_t)(level + 1); changed = 1; }
      }
    }
    __syncthreads();
    if (!changed) break;
    __syncthreads();
  }
  for (int j = threadIdx.x; j < n_dst; j += blockDim.x) {
    const uint16_t h = d[dst[j]];
    if (h == kInf) { report_err(err, MP_DATA_UNREACHABLE, s, dst[j]); dist[(int64_t)i * n_dst + j] = 0xff; }
    else if (h > 255) { report_err(err, MP_DATA_HOPS_RANGE, s, dst[j]); dist[(int64_t)i * n_dst + j] = 0xff; }
    else dist[(int64_t)i * n_dst + j] = (uint8_t)h;
  }
}

cudaError_t launch_bfs(const int32_t* row_ptr, const int32_t* col, int n, const int32_t* src, int n_src,
                       const int32_t* dst, int n_dst, uint8_t* dist, int64_t* err, cudaStream_t s) {
  if (n_src <= 0) return cudaSuccess;
  bfs_kernel<<<n_src, 256, 0, s>>>(row_ptr, col, n, src, dst, n_dst, dist, err);
  return cudaGetLastError();
}

// ---- device-level distance matrix ----------------------------------------
__global__ void expand_kernel(const uint8_t* __restrict__ dsrv, int n_srv, const int32_t* __restrict__ server, int S,
                              uint8_t* __restrict__ out) {
  const int64_t n = (int64_t)S * S;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(i / S), b = (int)(i % S);
    out[i] = dsrv[(int64_t)server[a] * n_srv + server[b]];
  }
}

cudaError_t launch_expand(const uint8_t* dsrv, int n_srv, const int32_t* server, int S, uint8_t* out, cudaStream_t s) {
  const int64_t n = (int64_t)S * S;
  if (n == 0) return cudaSuccess;
  expand_kernel<<<(unsigned)min((n + 255) / 256, (int64_t)4096), 256, 0, s>>>(dsrv, n_srv, server, S, out);
  return cudaGetLastError();
}

// ---- cost_matrix: p[l,s] = D[d_l, s] + D[s, c_l] -----------------------
__global__ void cost_kernel(const uint8_t* __restrict__ dsrv, int n_srv, const int32_t* __restrict__ server, int S,
                            const int32_t* __restrict__ disp, const int32_t* __restrict__ coll, int L,
                            uint8_t* __restrict__ p) {
  const int64_t n = (int64_t)L * S;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / S), s = (int)(i % S);
    const int64_t sv = server[s];
    const uint32_t h = (uint32_t)dsrv[(int64_t)server[disp[l]] * n_srv + sv] + (uint32_t)dsrv[sv * n_srv + server[coll[l]]];
    p[i] = (uint8_t)min(h, 255u);  // host checks 2*diameter <= 255 before launching
  }
}

cudaError_t launch_cost(const uint8_t* dsrv, int n_srv, const int32_t* server, int S, const int32_t* disp,
                        const int32_t* coll, int L, uint8_t* p, cudaStream_t s) {
  const int64_t n = (int64_t)L * S;
  if (n == 0) return cudaSuccess;
  cost_kernel<<<(unsigned)min((n + 255) / 256, (int64_t)4096), 256, 0, s>>>(dsrv, n_srv, server, S, disp, coll, L, p);
  return cudaGetLastError();
}

// ---- placement -> packed u8 score tables -------------------------------
__global__ void pack_kernel(const uint8_t* __restrict__ cost, int T, const int32_t* __restrict__ assign,
                            const int32_t* __restrict__ topo_of, int P, int L, int E, int S, uint32_t* __restrict__ tables,
                            int W, int64_t* err) {
  const int64_t n = (int64_t)L * 256 * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % W);
    const int e = (int)((i / W) % 256);
    const int l = (int)(i / ((int64_t)W * 256));
    uint32_t word = 0;
    if (e < E) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int q = 4 * w + j;
        if (q >= P) break;
        const int32_t s = assign[((int64_t)q * L + l) * E + e];
        const int32_t tp = topo_of[q];
        if (s < 0 || s >= S || tp < 0 || tp >= T) { report_err(err, MP_DATA_UNPLACED, l, e); continue; }
        word |= (uint32_t)cost[((int64_t)tp * L + l) * S + s] << (8 * j);
      }
    }
    tables[i] = word;
  }
}

cudaError_t launch_pack(const uint8_t* cost, int T, const int32_t* assign, const int32_t* topo_of, int P, int L, int E,
                        int S, uint32_t* tables, int W, int64_t* err, cudaStream_t s) {
  const int64_t n = (int64_t)L * 256 * W;
  pack_kernel<<<(unsigned)min((n + 255) / 256, (int64_t)4096), 256, 0, s>>>(cost, T, assign, topo_of, P, L, E, S,
                                                                            tables, W, err);
  return cudaGetLastError();
}

// ---- build_instance coefficients -----------------------------------
// numpy order: f = counts / denom ; w = f[:, :, None] * p[:, None, :] ; w_int = rint(w * scale)
__global__ void coeffs_kernel(const int64_t* __restrict__ counts, int64_t denom, const uint8_t* __restrict__ p, int L,
                              int E, int S, double scale, double* __restrict__ w, int64_t* __restrict__ w_int) {
  const int64_t n = (int64_t)L * E * S;
  const double inv_uniform = __ddiv_rn(1.0, (double)E);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i % S);
    const int64_t le = i / S;
    const int l = (int)(le / E);
    const double f = counts ? __ddiv_rn((double)counts[le], (double)denom) : inv_uniform;
    const double v = __dmul_rn(f, (double)p[(int64_t)l * S + s]);
    if (w) w[i] = v;
    if (w_int) {
      // scale > 0: SPEC.md:308 integerisation rint(w * scale); scale == 0: exact count * p
      w_int[i] = scale > 0.0 ? (int64_t)rint(__dmul_rn(v, scale))
                             : (counts ? counts[le] : 1) * (int64_t)p[(int64_t)l * S + s];
    }
  }
}

cudaError_t launch_coeffs(const int64_t* counts, int64_t denom, const uint8_t* p, int L, int E, int S, double scale,
                          double* w, int64_t* w_int, cudaStream_t s) {
  const int64_t n = (int64_t)L * E * S;
  if (n == 0) return cudaSuccess;
  coeffs_kernel<<<(unsigned)min((n + 255) / 256, (int64_t)8192), 256, 0, s>>>(counts, denom, p, L, E, S, scale, w, w_int);
  return cudaGetLastError();
}

// ---- communication_map, accumulated from the per-(l,e) load counts -------
__global__ void comm_kernel(const int64_t* __restrict__ counts, const int32_t* __restrict__ assign,
                            const int32_t* __restrict__ server, const uint8_t* __restrict__ dsrv, int n_srv,
                            const int32_t* __restrict__ disp, const int32_t* __restrict__ coll, int L, int E, int S,
                            int64_t* __restrict__ traffic, int64_t* err) {
  const int64_t n = (int64_t)L * E;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cnt = counts[i];
    if (cnt == 0) continue;
    const int l = (int)(i / E);
    const int32_t dv = assign[i];
    if (dv < 0 || dv >= S) { report_err(err, MP_DATA_UNPLACED, l, i % E); continue; }
    const int64_t a = server[disp[l]], sv = server[dv], b = server[coll[l]];
    const int64_t h1 = dsrv[a * n_srv + sv], h2 = dsrv[sv * n_srv + b];
    if (h1) atomic_add_i64(traffic + a * n_srv + sv, cnt * h1);
    if (h2) atomic_add_i64(traffic + sv * n_srv + b, cnt * h2);
  }
}

cudaError_t launch_comm(const int64_t* counts, const int32_t* assign, const int32_t* server, const uint8_t* dsrv,
                        int n_srv, const int32_t* disp, const int32_t* coll, int L, int E, int S, int64_t* traffic,
                        int64_t* err, cudaStream_t s) {
  const int64_t n = (int64_t)L * E;
  if (n == 0) return cudaSuccess;
  comm_kernel<<<(unsigned)min((n + 255) / 256, (int64_t)4096), 256, 0, s>>>(counts, assign, server, dsrv, n_srv, disp,
                                                                             coll, L, E, S, traffic, err);
  return cudaGetLastError();
}

}  // namespace mp
