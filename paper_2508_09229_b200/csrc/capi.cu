// extern "C" entry points of libmoeplace_cuda.so (declared in include/moeplace_cuda.h).
// Argument validation happens here, synchronously; kernels only see checked shapes.
#include "common.cuh"

namespace mp {
cudaError_t launch_stream(bool hist, int W, int max_p, const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1,
                          int L, int K, int E, const int64_t* bounds, int C, const uint32_t* tables, int64_t* counts,
                          int64_t* hop_sums, int64_t* err, cudaStream_t s, int algo);
int choose_algo(bool hist, int W, int algo, int64_t tokens, int C, int L, int K, int max_p);
int allreduce_supported(int64_t n, int world);
cudaError_t launch_allreduce_i64(int64_t* out, int64_t n, const int64_t* mc, const int64_t* const* peers,
                                 uint32_t* const* pads, int rank, int world, uint32_t epoch, int64_t* err,
                                 cudaStream_t s);
cudaError_t launch_gen(uint64_t seed, int64_t t0, int64_t t1, int L, int K, int E, const uint32_t* cdf,
                       const uint8_t* perm, uint8_t* planes, int64_t stride, cudaStream_t s);
cudaError_t launch_validate(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K, int E,
                            int64_t* err, cudaStream_t s);
cudaError_t launch_bfs(const int32_t* row_ptr, const int32_t* col, int n, const int32_t* src, int n_src,
                       const int32_t* dst, int n_dst, uint8_t* dist, int64_t* err, cudaStream_t s);
cudaError_t launch_expand(const uint8_t* dsrv, int n_srv, const int32_t* server, int S, uint8_t* out, cudaStream_t s);
cudaError_t launch_cost(const uint8_t* dsrv, int n_srv, const int32_t* server, int S, const int32_t* disp,
                        const int32_t* coll, int L, uint8_t* p, cudaStream_t s);
cudaError_t launch_pack(const uint8_t* cost, int T, const int32_t* assign, const int32_t* topo_of, int P, int L, int E,
                        int S, uint32_t* tables, int W, int64_t* err, cudaStream_t s);
cudaError_t launch_coeffs(const int64_t* counts, int64_t denom, const uint8_t* p, int L, int E, int S, double scale,
                          double* w, int64_t* w_int, cudaStream_t s);
cudaError_t launch_comm(const int64_t* counts, const int32_t* assign, const int32_t* server, const uint8_t* dsrv,
                        int n_srv, const int32_t* disp, const int32_t* coll, int L, int E, int S, int64_t* traffic,
                        int64_t* err, cudaStream_t s);
cudaError_t launch_dedup(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K,
                         const int64_t* bounds, int C, const uint32_t* tables, const uint32_t* srv_tables,
                         const uint8_t* src_srv, int64_t* hop_sums, int64_t* uniq_sums, int64_t* dedup_sums,
                         cudaStream_t s);
cudaError_t launch_pack_srv(const int32_t* server_of, int T, const int32_t* assign, const int32_t* topo_of, int P,
                            int L, int E, int S, uint32_t* tables, int64_t* err, cudaStream_t s);
cudaError_t launch_count_nl(const uint8_t* text, int64_t n, int64_t* counts, cudaStream_t s);
cudaError_t launch_find_nl(const uint8_t* text, int64_t n, const int64_t* offsets, int64_t* pos, cudaStream_t s);
cudaError_t launch_parse(const uint8_t* text, const int64_t* ends, int64_t first_start, int64_t n_lines, int L, int K,
                         int E, uint8_t* planes, int64_t stride, int64_t* chunk_ids, int64_t* err, cudaStream_t s);
cudaError_t launch_token_hops(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K,
                              const uint32_t* tables, int max_p, uint32_t* replicated, uint32_t* hops,
                              cudaStream_t s);
cudaError_t launch_hist_chunks(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K, int E,
                               const int64_t* bounds, int C, int64_t* counts, int64_t* err, cudaStream_t s);
cudaError_t launch_contract(const int64_t* counts, int C, const uint8_t* pe, int P, int64_t LE, int64_t* out,
                            cudaStream_t s);
cudaError_t launch_count_digits_u8(const int64_t* counts, int C, int64_t LE, int ndig, int64_t ldd, uint8_t* out,
                                   int64_t* err, cudaStream_t s);
cudaError_t launch_contract_tc(const uint8_t* pe, int P, int64_t ldpe, const uint8_t* digits, int C, int ndig,
                               int64_t LE, int64_t ldd, int64_t* out, int ctas, cudaStream_t s);
cudaError_t launch_pe_gather(const uint8_t* cost, int T, int L, int S, const int32_t* topo_S, const int32_t* assign,
                             const int32_t* topo_of, int P, int E, uint8_t* pe, int64_t ldpe, int64_t* err,
                             cudaStream_t s);
cudaError_t launch_perturb_pe(const uint8_t* pe_cur, int L, int E, int B, int n_swaps, uint64_t seed, int64_t iter,
                              uint8_t* pe_out, int64_t ldpe, int32_t* swaps, cudaStream_t s);
cudaError_t launch_batch_objective(const int64_t* sums, const int64_t* tokens, int B, int C, int kind, double lam,
                                   double* obj, cudaStream_t s);
cudaError_t launch_accept(const double* obj, int B, const int32_t* swaps, int n_swaps, int E, int32_t* assign,
                          uint8_t* pe_cur, double* cur_obj, double* history, int64_t iter, int64_t* accepted,
                          cudaStream_t s);
cudaError_t launch_objective_f64(const double* f, const uint8_t* pe, int64_t ldpe, int64_t LE, int P, double* out,
                                 cudaStream_t s);
cudaError_t launch_tokens_to_planes(const uint8_t* tok, int64_t n, int L, int K, uint8_t* planes, int64_t stride,
                                    int64_t t_out, cudaStream_t s);
cudaError_t launch_format(bool write, const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K,
                          const int64_t* cids, int64_t* lens_or_offsets, uint8_t* out, cudaStream_t s);
}  // namespace mp

namespace {
inline int status(cudaError_t e) { return e == cudaSuccess ? MP_OK : MP_ERR_CUDA; }
inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
// shared trace-shape checks
inline int check_trace(const uint8_t* planes, int64_t stride, int64_t t0, int64_t t1, int L, int K) {
  if (!planes || L <= 0 || K <= 0 || t0 < 0 || t1 < t0) return MP_ERR_ARG;
  if (!aligned16(planes) || (stride & 15) != 0 || stride < t1 * (int64_t)K) return MP_ERR_ARG;
  return MP_OK;
}
}  // namespace

extern "C" {

int mp_abi_version(void) { return MP_ABI_VERSION; }

const char* mp_status_string(int st) {
  switch (st) {
    case MP_OK: return "ok";
    case MP_ERR_ARG: return "invalid argument";
    case MP_ERR_CUDA: return "CUDA launch/runtime failure";
    case MP_ERR_UNSUPPORTED: return "outside the u8 device format (E > 256 or hop cost > 255)";
    case MP_INFEASIBLE: return "infeasible: max flow < L*E";
    default: return "unknown status";
  }
}

int mp_gen_trace(uint64_t seed, int64_t tok_begin, int64_t tok_end, int L, int K, int E, const uint32_t* cdf,
                 const uint8_t* perm, uint8_t* planes, int64_t plane_stride, void* stream) {
  if (E > mp::kMaxE) return MP_ERR_UNSUPPORTED;
  if (E <= 0 || K > E || !cdf || !perm || tok_begin < 0 || L > 65535) return MP_ERR_ARG;
  int r = check_trace(planes, plane_stride, 0, tok_end - tok_begin, L, K);
  if (r) return r;
  return status(mp::launch_gen(seed, tok_begin, tok_end, L, K, E, cdf, perm, planes, plane_stride, S(stream)));
}

int mp_validate_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K, int E,
                   int64_t* err, void* stream) {
  if (E > mp::kMaxE) return MP_ERR_UNSUPPORTED;
  if (E <= 0 || !err) return MP_ERR_ARG;
  int r = check_trace(planes, plane_stride, tok_begin, tok_end, L, K);
  if (r) return r;
  return status(mp::launch_validate(planes, plane_stride, tok_begin, tok_end, L, K, E, err, S(stream)));
}

int mp_hist_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K, int E,
               int64_t* counts, int64_t* err, void* stream) {
  if (E > mp::kMaxE) return MP_ERR_UNSUPPORTED;
  if (E <= 0 || !counts || !err) return MP_ERR_ARG;
  int r = check_trace(planes, plane_stride, tok_begin, tok_end, L, K);
  if (r) return r;
  if (tok_end == tok_begin) return MP_OK;
  return status(mp::launch_stream(true, 0, 0, planes, plane_stride, tok_begin, tok_end, L, K, E, nullptr, 1, nullptr,
                                  counts, nullptr, err, S(stream), MP_ALGO_AUTO));
}

int mp_hist_chunks_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                      int E, const int64_t* chunk_bounds, int C, int64_t* counts, int64_t* err, void* stream) {
  if (E > mp::kMaxE) return MP_ERR_UNSUPPORTED;
  int r = check_trace(planes, plane_stride, tok_begin, tok_end, L, K);
  if (r) return r;
  if (E <= 0 || !counts || !err || !chunk_bounds || C <= 0) return MP_ERR_ARG;
  if (tok_end == tok_begin) return MP_OK;
  return status(mp::launch_hist_chunks(planes, plane_stride, tok_begin, tok_end, L, K, E, chunk_bounds, C, counts, err,
                                       S(stream)));
}

int mp_contract_counts(const int64_t* counts, int C, const uint8_t* pe, int P, int64_t LE, int64_t* out, void* stream) {
  if (!counts || !pe || !out || C <= 0 || P <= 0 || LE <= 0) return MP_ERR_ARG;
  if (C > 65535 * 16) return MP_ERR_UNSUPPORTED;
  return status(mp::launch_contract(counts, C, pe, P, LE, out, S(stream)));
}

int mp_count_digits_u8(const int64_t* counts, int C, int64_t LE, int ndig, int64_t ldd, uint8_t* out, int64_t* err,
                       void* stream) {
  if (!counts || !out || !err || C <= 0 || C > 65535 || LE <= 0 || ldd < LE || (ldd & 15) || !aligned16(out) || (ndig != 1 && ndig != 2 && ndig != 4))
    return MP_ERR_ARG;
  return status(mp::launch_count_digits_u8(counts, C, LE, ndig, ldd, out, err, S(stream)));
}

int mp_contract_tc_u8(const uint8_t* pe, int P, int64_t ldpe, const uint8_t* digits, int C, int ndig, int64_t LE,
                      int64_t ldd, int64_t* out, int ctas, void* stream) {
  if (!pe || !digits || !out || P <= 0 || C <= 0 || LE <= 0 || ctas < -65536) return MP_ERR_ARG;
  if (ndig != 1 && ndig != 2 && ndig != 4) return MP_ERR_ARG;
  if (ldpe < LE || ldd < LE || (ldpe & 15) || (ldd & 15) || !aligned16(pe) || !aligned16(digits)) return MP_ERR_ARG;
  if ((int64_t)C * ndig > (1 << 24)) return MP_ERR_UNSUPPORTED;
  return status(mp::launch_contract_tc(pe, P, ldpe, digits, C, ndig, LE, ldd, out, ctas, S(stream)));
}

int mp_pack_tables(const uint8_t* cost, int T, const int32_t* assign, const int32_t* topo_of, int P, int L, int E,
                   int S_, uint32_t* tables, int W, int64_t* err, void* stream) {
  if (E > mp::kMaxE) return MP_ERR_UNSUPPORTED;
  if (!cost || !assign || !topo_of || !tables || !err || T <= 0 || P <= 0 || L <= 0 || E <= 0 || S_ <= 0) return MP_ERR_ARG;
  if (!(W == 1 || W == 2 || W == 4 || W == 8) || P > 4 * W) return MP_ERR_ARG;
  return status(mp::launch_pack(cost, T, assign, topo_of, P, L, E, S_, tables, W, err, S(stream)));
}

int mp_score_ex_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                   const int64_t* chunk_bounds, int C, const uint32_t* tables, int W, int max_p, int64_t* hop_sums,
                   int algo, void* stream) {
  int r = check_trace(planes, plane_stride, tok_begin, tok_end, L, K);
  if (r) return r;
  if (!chunk_bounds || C <= 0 || !tables || !hop_sums || !(W == 1 || W == 2 || W == 4 || W == 8)) return MP_ERR_ARG;
  if (max_p < 0 || algo < MP_ALGO_AUTO || algo > MP_ALGO_SEG) return MP_ERR_ARG;
  if (max_p > 255 || (algo == MP_ALGO_TOKEN && (int64_t)L * K * max_p > 65535)) return MP_ERR_UNSUPPORTED;
  if (W == 8 && algo != MP_ALGO_AUTO && algo != MP_ALGO_COUNT) return MP_ERR_UNSUPPORTED;  // 32 lanes: count-contract only
  if (algo == MP_ALGO_SEG && (K != 8 || max_p > 31)) return MP_ERR_UNSUPPORTED;
  if (tok_end == tok_begin) return MP_OK;
  return status(mp::launch_stream(false, W, max_p, planes, plane_stride, tok_begin, tok_end, L, K, 256, chunk_bounds,
                                  C, tables, nullptr, hop_sums, nullptr, S(stream), algo));
}

int mp_score_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                const int64_t* chunk_bounds, int C, const uint32_t* tables, int W, int max_p, int64_t* hop_sums,
                void* stream) {
  return mp_score_ex_u8(planes, plane_stride, tok_begin, tok_end, L, K, chunk_bounds, C, tables, W, max_p, hop_sums,
                        MP_ALGO_AUTO, stream);
}

int mp_token_hops_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                     const uint32_t* tables, int max_p, uint32_t* scratch, uint32_t* hops, void* stream) {
  int r = check_trace(planes, plane_stride, tok_begin, tok_end, L, K);
  if (r) return r;
  if (!tables || !hops || !scratch || max_p < 0) return MP_ERR_ARG;
  if ((int64_t)L * K * max_p > 65535 || max_p > 255) return MP_ERR_UNSUPPORTED;
  if (tok_end == tok_begin) return MP_OK;
  return status(mp::launch_token_hops(planes, plane_stride, tok_begin, tok_end, L, K, tables, max_p, scratch, hops,
                                      S(stream)));
}

int mp_hist_score_ex_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                        int E, const int64_t* chunk_bounds, int C, const uint32_t* tables, int W, int max_p,
                        int64_t* counts, int64_t* hop_sums, int64_t* err, int algo, void* stream) {
  if (E > mp::kMaxE) return MP_ERR_UNSUPPORTED;
  int r = check_trace(planes, plane_stride, tok_begin, tok_end, L, K);
  if (r) return r;
  if (E <= 0 || !counts || !err || !chunk_bounds || C <= 0 || !tables || !hop_sums || max_p < 0) return MP_ERR_ARG;
  if (!(W == 1 || W == 2 || W == 4 || W == 8) || algo < MP_ALGO_AUTO || algo > MP_ALGO_SEG) return MP_ERR_ARG;
  if (max_p > 255 || (algo == MP_ALGO_GATHER && W != 1)) return MP_ERR_UNSUPPORTED;
  if (W == 8 && algo != MP_ALGO_AUTO && algo != MP_ALGO_COUNT) return MP_ERR_UNSUPPORTED;  // 32 lanes: count-contract only
  if (algo == MP_ALGO_SEG && (K != 8 || max_p > 31)) return MP_ERR_UNSUPPORTED;
  if (algo == MP_ALGO_TOKEN && (int64_t)L * K * max_p > 65535) return MP_ERR_UNSUPPORTED;
  if (tok_end == tok_begin) return MP_OK;
  return status(mp::launch_stream(true, W, max_p, planes, plane_stride, tok_begin, tok_end, L, K, E, chunk_bounds, C,
                                  tables, counts, hop_sums, err, S(stream), algo));
}

int mp_hist_score_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                     int E, const int64_t* chunk_bounds, int C, const uint32_t* tables, int max_p, int64_t* counts,
                     int64_t* hop_sums, int64_t* err, void* stream) {
  return mp_hist_score_ex_u8(planes, plane_stride, tok_begin, tok_end, L, K, E, chunk_bounds, C, tables, 1, max_p,
                             counts, hop_sums, err, MP_ALGO_AUTO, stream);
}

int mp_allreduce_peers_i64(int64_t* out, int64_t n, const int64_t* mc, const uint64_t* peer_bufs,
                           const uint64_t* peer_pads, int rank, int world, uint32_t epoch, int64_t* err, void* stream) {
  if (!out || n < 0 || !peer_bufs || !peer_pads || !err || world < 1 || world > 64 || rank < 0 || rank >= world)
    return MP_ERR_ARG;
  if (!mp::allreduce_supported(n, world)) return MP_ERR_UNSUPPORTED;  // signal-pad words / vector length
  return status(mp::launch_allreduce_i64(out, n, mc, reinterpret_cast<const int64_t* const*>(peer_bufs),
                                         reinterpret_cast<uint32_t* const*>(peer_pads), rank, world, epoch, err,
                                         S(stream)));
}

int mp_choose_algo(int hist, int W, int64_t tokens, int C, int L, int K, int max_p) {
  return mp::choose_algo(hist != 0, W, MP_ALGO_AUTO, tokens, C, L, K, max_p);
}

int mp_apsp_bfs(const int32_t* row_ptr, const int32_t* col, int n_nodes, const int32_t* src_nodes, int n_src,
                const int32_t* dst_nodes, int n_dst, uint8_t* dist, int64_t* err, void* stream) {
  if (!row_ptr || !col || !src_nodes || !dst_nodes || !dist || !err || n_nodes <= 0 || n_src < 0 || n_dst < 0)
    return MP_ERR_ARG;
  if (n_nodes > 8192) return MP_ERR_UNSUPPORTED;
  return status(mp::launch_bfs(row_ptr, col, n_nodes, src_nodes, n_src, dst_nodes, n_dst, dist, err, S(stream)));
}

int mp_expand_dist(const uint8_t* dsrv, int n_srv, const int32_t* dev_server, int S_, uint8_t* out, void* stream) {
  if (!dsrv || !dev_server || !out || n_srv <= 0 || S_ < 0) return MP_ERR_ARG;
  return status(mp::launch_expand(dsrv, n_srv, dev_server, S_, out, S(stream)));
}

int mp_cost_matrix(const uint8_t* dsrv, int n_srv, const int32_t* dev_server, int S_, const int32_t* dispatch,
                   const int32_t* collect, int L, uint8_t* p, void* stream) {
  if (!dsrv || !dev_server || !dispatch || !collect || !p || n_srv <= 0 || S_ <= 0 || L <= 0) return MP_ERR_ARG;
  return status(mp::launch_cost(dsrv, n_srv, dev_server, S_, dispatch, collect, L, p, S(stream)));
}

int mp_coeffs(const int64_t* counts, int64_t denom, const uint8_t* p, int L, int E, int S_, double scale, double* w,
              int64_t* w_int, void* stream) {
  if (!p || L <= 0 || E <= 0 || S_ <= 0 || (!w && !w_int)) return MP_ERR_ARG;
  if (counts && denom <= 0) return MP_ERR_ARG;
  return status(mp::launch_coeffs(counts, denom, p, L, E, S_, scale, w, w_int, S(stream)));
}

int mp_comm_map(const int64_t* counts, const int32_t* assign, const int32_t* dev_server, const uint8_t* dsrv, int n_srv,
                const int32_t* dispatch, const int32_t* collect, int L, int E, int S_, int64_t* traffic, int64_t* err,
                void* stream) {
  if (!counts || !assign || !dev_server || !dsrv || !dispatch || !collect || !traffic || !err || n_srv <= 0 || L <= 0 ||
      E <= 0 || S_ <= 0)
    return MP_ERR_ARG;
  return status(mp::launch_comm(counts, assign, dev_server, dsrv, n_srv, dispatch, collect, L, E, S_, traffic, err,
                                S(stream)));
}

int mp_score_dedup_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                      const int64_t* chunk_bounds, int C, const uint32_t* tables, const uint32_t* srv_tables,
                      const uint8_t* src_srv, int64_t* hop_sums, int64_t* uniq_sums, int64_t* dedup_sums,
                      void* stream) {
  int r = check_trace(planes, plane_stride, tok_begin, tok_end, L, K);
  if (r) return r;
  if (K > 32) return MP_ERR_UNSUPPORTED;
  if (!chunk_bounds || C <= 0 || !tables || !srv_tables || !src_srv || !hop_sums || !uniq_sums || !dedup_sums)
    return MP_ERR_ARG;
  if (tok_end == tok_begin) return MP_OK;
  return status(mp::launch_dedup(planes, plane_stride, tok_begin, tok_end, L, K, chunk_bounds, C, tables, srv_tables,
                                 src_srv, hop_sums, uniq_sums, dedup_sums, S(stream)));
}

int mp_pack_server_tables(const int32_t* server_of, int T, const int32_t* assign, const int32_t* topo_of, int P, int L,
                          int E, int S_, uint32_t* srv_tables, int64_t* err, void* stream) {
  if (E > mp::kMaxE) return MP_ERR_UNSUPPORTED;
  if (!server_of || !assign || !topo_of || !srv_tables || !err || T <= 0 || P <= 0 || P > 4 || L <= 0 || E <= 0 || S_ <= 0)
    return MP_ERR_ARG;
  return status(mp::launch_pack_srv(server_of, T, assign, topo_of, P, L, E, S_, srv_tables, err, S(stream)));
}

int mp_count_newlines(const uint8_t* text, int64_t n, int64_t* counts, void* stream) {
  if (!text || n < 0 || !counts) return MP_ERR_ARG;
  return status(mp::launch_count_nl(text, n, counts, S(stream)));
}

int mp_find_newlines(const uint8_t* text, int64_t n, const int64_t* offsets, int64_t* positions, void* stream) {
  if (!text || n < 0 || !offsets || !positions) return MP_ERR_ARG;
  return status(mp::launch_find_nl(text, n, offsets, positions, S(stream)));
}

int mp_parse_trace_text(const uint8_t* text, const int64_t* ends, int64_t first_start, int64_t n_lines, int L, int K,
                        int E, uint8_t* planes, int64_t plane_stride, int64_t* chunk_ids, int64_t* err, void* stream) {
  if (E > mp::kMaxE) return MP_ERR_UNSUPPORTED;
  if (!text || !ends || n_lines < 0 || first_start < 0 || !chunk_ids || !err || E <= 0) return MP_ERR_ARG;
  int r = check_trace(planes, plane_stride, 0, n_lines, L, K);
  if (r) return r;
  return status(mp::launch_parse(text, ends, first_start, n_lines, L, K, E, planes, plane_stride, chunk_ids, err,
                                 S(stream)));
}

int mp_format_lengths(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                      const int64_t* cids, int64_t* lengths, void* stream) {
  int r = check_trace(planes, plane_stride, tok_begin, tok_end, L, K);
  if (r) return r;
  if (!cids || !lengths) return MP_ERR_ARG;
  return status(mp::launch_format(false, planes, plane_stride, tok_begin, tok_end, L, K, cids, lengths, nullptr,
                                  S(stream)));
}

int mp_format_trace_text(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                         const int64_t* cids, const int64_t* offsets, uint8_t* out, void* stream) {
  int r = check_trace(planes, plane_stride, tok_begin, tok_end, L, K);
  if (r) return r;
  if (!cids || !offsets || !out) return MP_ERR_ARG;
  return status(mp::launch_format(true, planes, plane_stride, tok_begin, tok_end, L, K, cids,
                                  const_cast<int64_t*>(offsets), out, S(stream)));
}

int mp_copy_planes_h2d(void* dst, int64_t dst_stride, const void* src, int64_t src_stride, int64_t width, int rows,
                       void* stream) {
  if (!dst || !src || width < 0 || rows < 0 || dst_stride < width || src_stride < width) return MP_ERR_ARG;
  if (width == 0 || rows == 0) return MP_OK;
  return status(cudaMemcpy2DAsync(dst, (size_t)dst_stride, src, (size_t)src_stride, (size_t)width, (size_t)rows,
                                  cudaMemcpyHostToDevice, S(stream)));
}

int mp_tokens_to_planes_u8(const uint8_t* tokens, int64_t n, int L, int K, uint8_t* planes, int64_t plane_stride,
                           int64_t tok_out, void* stream) {
  if (!tokens || !planes || n < 0 || L <= 0 || K <= 0 || tok_out < 0) return MP_ERR_ARG;
  if (!aligned16(planes) || (plane_stride & 15) != 0 || plane_stride < (tok_out + n) * (int64_t)K) return MP_ERR_ARG;
  return status(mp::launch_tokens_to_planes(tokens, n, L, K, planes, plane_stride, tok_out, S(stream)));
}

int mp_pe_gather_u8(const uint8_t* cost, int T, int L, int n_dev, const int32_t* topo_S, const int32_t* assign,
                    const int32_t* topo_of, int P, int E, uint8_t* pe, int64_t ldpe, int64_t* err, void* stream) {
  if (!cost || !assign || !pe || !err || T <= 0 || L <= 0 || n_dev <= 0 || P <= 0 || E <= 0 || P > 65535)
    return MP_ERR_ARG;
  if (ldpe < (int64_t)L * E) return MP_ERR_ARG;
  return status(mp::launch_pe_gather(cost, T, L, n_dev, topo_S, assign, topo_of, P, E, pe, ldpe, err, S(stream)));
}

int mp_perturb_pe_u8(const uint8_t* pe_cur, int L, int E, int B, int n_swaps, uint64_t seed, int64_t iter,
                     uint8_t* pe_out, int64_t ldpe, int32_t* swaps, void* stream) {
  if (!pe_cur || !pe_out || !swaps || L <= 0 || E <= 0 || B <= 0 || n_swaps < 1 || iter < 0) return MP_ERR_ARG;
  if (ldpe < (int64_t)L * E || (ldpe & 15) || !aligned16(pe_cur) || !aligned16(pe_out)) return MP_ERR_ARG;
  return status(mp::launch_perturb_pe(pe_cur, L, E, B, n_swaps, seed, iter, pe_out, ldpe, swaps, S(stream)));
}

int mp_batch_objective(const int64_t* sums, const int64_t* tokens, int B, int C, int kind, double lam, double* obj,
                       void* stream) {
  if (!sums || !tokens || !obj || B <= 0 || C <= 0 || kind < 0 || kind > 2) return MP_ERR_ARG;
  return status(mp::launch_batch_objective(sums, tokens, B, C, kind, lam, obj, S(stream)));
}

int mp_search_accept(const double* obj, int B, const int32_t* swaps, int n_swaps, int E, int32_t* assign,
                     uint8_t* pe_cur, double* cur_obj, double* history, int64_t iter, int64_t* accepted, void* stream) {
  if (!obj || !swaps || !assign || !pe_cur || !cur_obj || !history || !accepted || B <= 0 || n_swaps < 1 || E <= 0 ||
      iter < 0)
    return MP_ERR_ARG;
  return status(mp::launch_accept(obj, B, swaps, n_swaps, E, assign, pe_cur, cur_obj, history, iter, accepted,
                                  S(stream)));
}

int mp_objective_f64(const double* f, const uint8_t* pe, int64_t ldpe, int64_t LE, int P, double* out, void* stream) {
  if (!f || !pe || !out || LE <= 0 || ldpe < LE || P <= 0) return MP_ERR_ARG;
  return status(mp::launch_objective_f64(f, pe, ldpe, LE, P, out, S(stream)));
}

}  // extern "C"
