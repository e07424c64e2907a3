/* Plain C client of libmoeplace_cuda.so (no Python, no torch): the C-ABI as a reference binding
 * (cgo/JNI/N-API would call exactly these symbols).  Generates a small Zipf-free (uniform) trace
 * on the device, histograms it and scores two placements, and checks the results' invariants.
 *   nvcc -o capi_client examples/capi_client.c -I include -L paper_2508_09229_b200/lib -lmoeplace_cuda
 *   LD_LIBRARY_PATH=paper_2508_09229_b200/lib ./capi_client                                    */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "moeplace_cuda.h"

#define CHECK(x) do { int st_ = (x); if (st_) { fprintf(stderr, "%s -> %s\n", #x, mp_status_string(st_)); return 1; } } while (0)

int main(void) {
  const int L = 4, E = 16, K = 3, C = 5, S = 4;
  const int64_t N = 100003;
  const int64_t stride = ((N * K + 15) / 16) * 16;
  uint32_t cdf[17];
  uint8_t perm[4 * 16], cost[4 * 4];
  int32_t assign[2 * 4 * 16], topo_of[2] = {0, 0};
  int64_t bounds[6];
  for (int r = 0; r <= E; ++r) cdf[r] = (uint32_t)r * 1000u;              /* uniform weights */
  for (int l = 0; l < L; ++l) for (int e = 0; e < E; ++e) perm[l * E + e] = (uint8_t)e;
  for (int l = 0; l < L; ++l) for (int s = 0; s < S; ++s) cost[l * S + s] = (uint8_t)(l + 2 * s);
  for (int q = 0; q < 2; ++q) for (int l = 0; l < L; ++l) for (int e = 0; e < E; ++e)
    assign[(q * L + l) * E + e] = q == 0 ? 0 : e % S;                         /* all on device 0 | spread */
  for (int c = 0; c <= C; ++c) bounds[c] = (c * N + C - 1) / C;

  uint8_t *d_planes, *d_perm, *d_cost; uint32_t *d_cdf, *d_tables; int32_t *d_assign, *d_topo;
  int64_t *d_counts, *d_sums, *d_bounds, *d_err;
  cudaMalloc((void**)&d_planes, L * stride); cudaMalloc((void**)&d_perm, sizeof perm);
  cudaMalloc((void**)&d_cost, sizeof cost); cudaMalloc((void**)&d_cdf, sizeof cdf);
  cudaMalloc((void**)&d_tables, L * 256 * 4); cudaMalloc((void**)&d_assign, sizeof assign);
  cudaMalloc((void**)&d_topo, sizeof topo_of); cudaMalloc((void**)&d_counts, L * E * 8);
  cudaMalloc((void**)&d_sums, 4 * C * 8); cudaMalloc((void**)&d_bounds, sizeof bounds); cudaMalloc((void**)&d_err, 32);
  cudaMemcpy(d_perm, perm, sizeof perm, cudaMemcpyHostToDevice);
  cudaMemcpy(d_cost, cost, sizeof cost, cudaMemcpyHostToDevice);
  cudaMemcpy(d_cdf, cdf, sizeof cdf, cudaMemcpyHostToDevice);
  cudaMemcpy(d_assign, assign, sizeof assign, cudaMemcpyHostToDevice);
  cudaMemcpy(d_topo, topo_of, sizeof topo_of, cudaMemcpyHostToDevice);
  cudaMemcpy(d_bounds, bounds, sizeof bounds, cudaMemcpyHostToDevice);
  cudaMemset(d_counts, 0, L * E * 8); cudaMemset(d_sums, 0, 4 * C * 8); cudaMemset(d_err, 0, 32);

  CHECK(mp_gen_trace(42, 0, N, L, K, E, d_cdf, d_perm, d_planes, stride, NULL));
  CHECK(mp_hist_u8(d_planes, stride, 0, N, L, K, E, d_counts, d_err, NULL));
  CHECK(mp_pack_tables(d_cost, 1, d_assign, d_topo, 2, L, E, S, d_tables, 1, d_err, NULL));
  CHECK(mp_score_u8(d_planes, stride, 0, N, L, K, d_bounds, C, d_tables, 1, 255, d_sums, NULL));
  if (cudaDeviceSynchronize() != cudaSuccess) { fprintf(stderr, "CUDA error\n"); return 1; }

  int64_t counts[4 * 16], sums[4 * 5], err[4];
  cudaMemcpy(counts, d_counts, sizeof counts, cudaMemcpyDeviceToHost);
  cudaMemcpy(sums, d_sums, sizeof sums, cudaMemcpyDeviceToHost);
  cudaMemcpy(err, d_err, sizeof err, cudaMemcpyDeviceToHost);
  int ok = err[0] == 0;
  int64_t expect0 = 0, tot1 = 0;
  for (int l = 0; l < L; ++l) {
    int64_t s = 0;
    for (int e = 0; e < E; ++e) s += counts[l * E + e];
    ok &= s == N * K;                                   /* every pick counted once */
    expect0 += (int64_t)cost[l * S + 0] * N * K;        /* placement 0: every pick costs p[l][0] */
  }
  int64_t got0 = 0;
  for (int c = 0; c < C; ++c) { got0 += sums[0 * C + c]; tot1 += sums[1 * C + c]; }
  for (int l = 0; l < L; ++l) { int64_t t = 0; for (int e = 0; e < E; ++e) t += counts[l * E + e] * cost[l * S + e % S]; tot1 -= t; }
  ok &= got0 == expect0 && tot1 == 0;                  /* placement 1 == sum(counts * pe) */
  printf("capi_client %s: abi %d, hops placement0 %lld (expect %lld)\n", ok ? "ok" : "FAILED", mp_abi_version(),
         (long long)got0, (long long)expect0);
  return ok ? 0 : 1;
}
