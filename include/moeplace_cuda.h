/*
 * moeplace_cuda.h — C-ABI of the B200 (sm_100a) engine behind the `moeplace` hot path.
 *
 * The reference (arXiv 2508.09229, `moeplace` 0.1.0) is a pure-Python package whose hot-path
 * operations are specified in /root/reference/SPEC.md; it ships no native code and no FFI.
 * Each entry point below therefore replaces the CPU body of one SPEC operation; the Python
 * package `paper_2508_09229_b200` (re-exported as `moeplace`) binds them with ctypes
 * (see INTEGRATION.md).  Cited lines are SPEC.md:N.
 *
 * Conventions (all functions):
 *   - Plain pointers and sizes only.  Device pointers are CUDA global-memory addresses; the
 *     caller owns every buffer (inputs, outputs, scratch).  The library never allocates or
 *     frees device memory; its only global state is a mutex-guarded cache of per-device launch
 *     facts (SM count, each kernel's resident CTAs, its shared-memory attribute), filled on a
 *     device's first launch, and a 4 KB pinned host-mapped table of {span, non-empty chunks} per
 *     chunk-bounds array seen by the count-contract launchers (filled by a one-block kernel on the
 *     caller's stream, read without a wait; it picks a kernel shape, never changes a result).
 *     Safe to call concurrently on different streams.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every
 *     function only ENQUEUES work; nothing synchronises the host.
 *   - Integer outputs are ACCUMULATED (`+=`): the caller zeroes them.  This makes sharded
 *     (multi-GPU, token-range) calls compose by plain addition.
 *   - Return value: MP_OK, or an MP_ERR_* code describing a synchronous argument/launch
 *     failure (the Python layer maps MP_ERR_ARG/MP_ERR_UNSUPPORTED to ConfigError,
 *     MP_ERR_CUDA to RuntimeError).  Data errors found by a kernel are written to a caller
 *     owned device `err` block (int64[4] = {code, layer, value, count}; code 0 = clean).  Every
 *     entry point that takes `err` requires it (NULL -> MP_ERR_ARG); argument checks run before
 *     any CUDA call, so a rejected call never touches the device.
 *
 * Trace layout ("layer planes"): uint8 planes[L][plane_stride]; byte t*K+k of plane l is the
 * k-th expert selected by token t in MoE layer l.  plane_stride and the
 * base address must be multiples of 16.  Expert IDs are one byte, so E <= 256.
 */
#ifndef MOEPLACE_CUDA_H
#define MOEPLACE_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MP_ABI_VERSION 1

#define MP_OK 0
#define MP_ERR_ARG 1          /* invalid argument (shape, range, alignment)        */
#define MP_ERR_CUDA 2         /* CUDA launch/runtime failure                       */
#define MP_ERR_UNSUPPORTED 3  /* outside the u8 device format (E > 256, p > 255)    */

/* device err-block codes (err[0]) */
#define MP_DATA_OK 0
#define MP_DATA_EXPERT_RANGE 1   /* expert id >= E            err = {1, layer, id, count}          */
#define MP_DATA_DUPLICATE 2      /* repeated id in one record err = {2, layer, token, count}       */
#define MP_DATA_UNREACHABLE 3    /* BFS: disconnected graph   err = {3, src, dst, count}           */
#define MP_DATA_UNPLACED 4       /* assign outside [0, S)     err = {4, layer, expert, count}      */
#define MP_DATA_HOPS_RANGE 5     /* hop count > 255           err = {5, src, dst, count}           */

/* ---- library identity ------------------------------------------------------------------- */
int mp_abi_version(void);
const char* mp_status_string(int status);

/* ---- trace synthesis: generate_trace ------------------------------
 * Counter-based Zipf(s) sampler: token t, layer l draws K distinct ranks without replacement
 * with probability proportional to the integer weights cdf[r+1]-cdf[r] (successive sampling),
 * maps rank -> expert through perm[l][rank].  Randomness is Philox4x32-10 keyed by `seed`
 * with counter (t_lo, t_hi, l, k/4), so any token range regenerates bit-identically on any
 * device or shard.  Writes planes[l][(t - tok_begin)*K + k] for t in [tok_begin, tok_end).
 *   cdf: device uint32[E+1], cdf[0]=0, strictly increasing, cdf[E] < 2^31
 *   perm: device uint8[L][E] (a permutation of 0..E-1 per layer)                             */
int mp_gen_trace(uint64_t seed, int64_t tok_begin, int64_t tok_end, int L, int K, int E,
                 const uint32_t* cdf, const uint8_t* perm, uint8_t* planes, int64_t plane_stride,
                 void* stream);

/* ---- ingestion check: ActivationTrace invariants ----------------------------
 * For tokens [tok_begin, tok_end): every id < E and the K ids of each (token, layer) record
 * are distinct.  First violation (lowest token) lands in err.                                */
int mp_validate_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end,
                   int L, int K, int E, int64_t* err, void* stream);

/* ---- text ingestion: parse_trace on the device ----------------------
 * mp_count_newlines: counts[b] = #'\n' in text[b*65536, (b+1)*65536), b < ceil(n/65536).
 * mp_find_newlines: positions of every '\n', in order; offsets[b] = exclusive prefix of counts.
 * mp_parse_trace_text: line t (0-based, after the header) spans [first_start or ends[t-1]+1,
 *   ends[t]); parses "cid\t[layer]0:e,..,e\t...", writes planes[l][t*K + k] and chunk_ids[t].
 *   err[0] (caller sets INT64_MAX) = min over bad lines of t*16 + code (1 structure, 2 layer
 *   label, 3 id >= E, 4 id count, 5 duplicate id, 6 chunk id overflow).  The text buffer must
 *   be readable (padded) up to the 16-byte boundary after its last byte.                     */
int mp_count_newlines(const uint8_t* text, int64_t n, int64_t* counts, void* stream);
int mp_find_newlines(const uint8_t* text, int64_t n, const int64_t* offsets, int64_t* positions, void* stream);
int mp_parse_trace_text(const uint8_t* text, const int64_t* ends, int64_t first_start, int64_t n_lines, int L, int K,
                        int E, uint8_t* planes, int64_t plane_stride, int64_t* chunk_ids, int64_t* err, void* stream);

/* ---- text encoder: write_trace on the device ---------------------------
 * mp_format_lengths: lengths[i] = byte length of token (tok_begin+i)'s canonical line
 *   "cid\tlayer0:e,..,e\t...\n" (cids: device int64 [n], one chunk id per token, >= 0).
 * mp_format_trace_text: writes each line at out[offsets[i]] (offsets = exclusive prefix sum of
 *   lengths, so the lines are contiguous and in token order).                                  */
int mp_format_lengths(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                      const int64_t* cids, int64_t* lengths, void* stream);
int mp_format_trace_text(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                         const int64_t* cids, const int64_t* offsets, uint8_t* out, void* stream);

/* ---- load statistics: estimate_frequencies ------------------------
 * counts[l*E + e] += #{(t,k) : t in [tok_begin,tok_end), planes[l][t*K+k] == e}.
 * Ids >= E are not counted; they raise MP_DATA_EXPERT_RANGE in err.                          */
int mp_hist_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end,
               int L, int K, int E, int64_t* counts, int64_t* err, void* stream);

/* ---- factorized evaluator (SPEC.md:383 linearity) -------------------------------
 * mp_hist_chunks_u8: per-chunk histogram, counts[(c*L + l)*E + e] += #{(t,k): t in chunk c, ...}
 *   (int64 [C][L][E]; same bounds contract as mp_score_u8).
 * mp_contract_counts: out[q*C + c] += sum_i counts[c*LE + i] * pe[q*LE + i] (int64, exact; each
 *   count must be < 2^31), pe = uint8 [P][LE] per-expert round-trip costs (LE = L*E).
 * Together they give exactly mp_score_u8's per-chunk hop sums for any number of placements.    */
int mp_hist_chunks_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                      int E, const int64_t* chunk_bounds, int C, int64_t* counts, int64_t* err, void* stream);
int mp_contract_counts(const int64_t* counts, int C, const uint8_t* pe, int P, int64_t LE, int64_t* out, void* stream);
/* Tensor-core form of the same contraction (5th-generation tensor cores, tcgen05 kind::i8; no library GEMM):
 * mp_count_digits_u8: out uint8 [C*ndig][ldd], out[(c*ndig + a)*ldd + i] = byte a of counts[c*LE + i]
 *   (ndig in {1, 2, 4}; columns [LE, ldd) zero).  A count < 0 or >= 2^(8*ndig) is written as 0 and
 *   raises MP_DATA_EXPERT_RANGE in err = {1, chunk, index, count}.
 * mp_contract_tc_u8: out[q*C + c] += sum_{i<LE} pe[q*ldpe + i] * counts[c][i], exactly (int64), from
 *   the digit operand above: ONE u8 x u8 GEMM with int32 accumulators in TMEM (TMA-fed, 128-byte
 *   swizzled K-major tiles), stream-K over every (128-row pe tile, 128-byte k-block) unit with runs
 *   of <= 32768 K per accumulation so every int32 partial is exact, the digits recombined in the
 *   epilogue and added with coalesced int64 atomics.  ldpe, ldd: multiples of 16; pe, digits:
 *   16-byte aligned.  ctas = 0: automatic (single CTAs, one epilogue each); ctas > 0: that many
 *   single CTAs per 512-row digit tile; ctas < 0: -ctas CTA pairs per digit tile
 *   (tcgen05.mma.cta_group::2 on 256-row tiles, each CTA loading half of the digit tile).  Together with
 *   mp_hist_chunks_u8 this is the factorized evaluator for any number of placements.              */
int mp_count_digits_u8(const int64_t* counts, int C, int64_t LE, int ndig, int64_t ldd, uint8_t* out, int64_t* err,
                       void* stream);
int mp_contract_tc_u8(const uint8_t* pe, int P, int64_t ldpe, const uint8_t* digits, int C, int ndig, int64_t LE,
                      int64_t ldd, int64_t* out, int ctas, void* stream);

/* ---- placement tables: Placement -> per-expert round-trip hops ---------
 * tables[((l*256 + e)*W + w)] is a u32 whose byte j is pe_q[l][e] = cost[topo_of[q]][l][assign[q][l][e]]
 * for placement q = 4*w + j (q < P; unused lanes and e >= E are 0).  W = 1, 2, 4 or 8 (P <= 4W;
 * W = 8 -- 32 placements per pass -- runs the count-contract algorithm only).
 *   cost: device uint8[T][L][S]; assign: device int32[P][L][E]; topo_of: device int32[P]      */
int mp_pack_tables(const uint8_t* cost, int T, const int32_t* assign, const int32_t* topo_of, int P,
                   int L, int E, int S, uint32_t* tables, int W, int64_t* err, void* stream);

/* ---- traffic evaluator: token_hops / evaluate -----------------
 * For placement q and chunk c:
 *   hop_sums[q*C + c] += sum_{t in chunk c, t in [tok_begin,tok_end)} sum_l sum_k pe_q[l][planes[l][t*K+k]]
 * chunk_bounds: device int64[C+1], ascending token indices; chunk c = [bounds[c], bounds[c+1]);
 * the caller guarantees bounds[0] <= tok_begin and bounds[C] >= tok_end.
 * max_p: an upper bound on every table byte (selects the u8-lane widening interval).
 * hop_sums is int64[4W][C].                                                                  */
int mp_score_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end,
                int L, int K, const int64_t* chunk_bounds, int C, const uint32_t* tables, int W,
                int max_p, int64_t* hop_sums, void* stream);

/* ---- per-token hops for every token: token_hops over the whole trace -----
 * hops[q*n + i] = sum_l sum_k pe_q[l][planes[l][(tok_begin+i)*K + k]] for q < 4 (W = 1 tables),
 * n = tok_end - tok_begin, uint32 output (fully written).  Requires L*K*max_p <= 65535.
 * scratch: device uint32 [L][256][32] (the lane-replicated tables, 32 KB per layer).           */
int mp_token_hops_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                     const uint32_t* tables, int max_p, uint32_t* scratch, uint32_t* hops, void* stream);

/* ---- fused statistics + traffic pass (one read of the trace) -----------------------------
 * mp_hist_u8 and mp_score_u8 over the same token range in one kernel (W = 1 tables).          */
int mp_hist_score_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end,
                     int L, int K, int E, const int64_t* chunk_bounds, int C, const uint32_t* tables,
                     int max_p, int64_t* counts, int64_t* hop_sums, int64_t* err, void* stream);

/* ---- explicit algorithm choice for the hop sums -------------------------------------------
 * Both algorithms produce bit-identical hop_sums (and counts):
 *   MP_ALGO_GATHER: every expert byte looks up its placement costs in a shared-memory table and
 *     per-token-layer sums are accumulated in u8 lanes (one LDS per lookup);
 *   MP_ALGO_COUNT:  count-contract -- the kernel only histograms; at each (layer, chunk) piece it
 *     contracts the piece's bin totals with the tables (hop sum = sum_e n[e]*pe[e]),
 *     so the per-byte cost does not depend on the number of placements;
 *   MP_ALGO_TOKEN:  token-tiled -- a CTA keeps per-token sums of a 4096-token tile in registers
 *     across all L layers and reduces them per chunk (segmented warp scan); its cost does not
 *     depend on the chunk count C, where GATHER / COUNT pay per (layer, chunk) piece and slow
 *     down sharply for short chunks.  Requires L*K*max_p <= 65535 (else MP_ERR_UNSUPPORTED);
 *     with a histogram it is mp_hist_u8 + the token pass;
 *   MP_ALGO_AUTO:   the faster one for the shape, by average tokens per chunk (measured
 *     crossovers, mp_choose_algo): when SEG applies (K = 8, max_p <= 31) SEG below 5000 / 3000 /
 *     1500 (with a histogram, W = 1 / 2 / 4) and 40000 / 6000 / 2400 (score-only) tokens per
 *     chunk, TOKEN below 50 (score-only W = 1); otherwise TOKEN below MP_TOKEN_CHUNK_TOKENS (W = 1 with
 *     a histogram; half of it for W = 2, 700 for W = 4; score-only 4096 / 1600 / 800) when the
 *     limit above holds; else GATHER for score-only W = 1 and COUNT otherwise.  This is what
 *     mp_score_u8 / mp_hist_score_u8 use.
 *   MP_ALGO_SEG:    segmented gather -- a layer-major stream in which each warp owns a contiguous
 *     token range and reduces its running sums at every chunk boundary it crosses (a warp
 *     redux.sync per boundary, no per-piece CTA work), so it is C-independent like TOKEN while
 *     reading each layer's table once per CTA segment.  K = 8 and max_p <= 31 only (else
 *     MP_ERR_UNSUPPORTED); the histogram is fused for every W.
 * mp_hist_score_ex_u8 takes W = 1, 2, 4 or 8 (GATHER supports W = 1 only, and W = 8 COUNT / AUTO
 * only -> MP_ERR_UNSUPPORTED).                                                                     */
#define MP_ALGO_AUTO 0
#define MP_ALGO_GATHER 1
#define MP_ALGO_COUNT 2
#define MP_ALGO_TOKEN 3
#define MP_ALGO_SEG 4
#define MP_TOKEN_CHUNK_TOKENS 2560
int mp_score_ex_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end,
                   int L, int K, const int64_t* chunk_bounds, int C, const uint32_t* tables, int W,
                   int max_p, int64_t* hop_sums, int algo, void* stream);
int mp_hist_score_ex_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end,
                        int L, int K, int E, const int64_t* chunk_bounds, int C, const uint32_t* tables, int W,
                        int max_p, int64_t* counts, int64_t* hop_sums, int64_t* err, int algo, void* stream);
/* ---- cross-GPU sum of the packed result vector ---------------------------------
 * mp_allreduce_peers_i64: out[i] = sum over the world of every rank's copy of a symmetric int64
 * buffer (torch.distributed._symmetric_memory), through NVLink/NVSwitch peer memory instead of a
 * separate NCCL collective.  peer_bufs / peer_pads: DEVICE arrays of the world's buffer and
 * signal-pad addresses (the buffer to sum, e.g. one half of a double-buffered allocation); mc: its
 * multicast address (NVLS: one multimem.ld_reduce per element, summed in the switch) or NULL (P2P
 * loads); out: this rank's private result.  Every rank calls it with the same n and an epoch larger
 * than any earlier call's; a rank must not rewrite the summed buffer before the NEXT call has
 * returned (double-buffer the inputs by epoch parity).  Signal-pad words [1024, 2048) are used;
 * n <= 2^21 / world (else MP_ERR_UNSUPPORTED).  A peer that does not arrive within ~2 s of clock
 * sets err = {MP_DATA_UNREACHABLE, rank, slice} instead of hanging.                          */
int mp_allreduce_peers_i64(int64_t* out, int64_t n, const int64_t* mc, const uint64_t* peer_bufs,
                           const uint64_t* peer_pads, int rank, int world, uint32_t epoch, int64_t* err, void* stream);

/* The algorithm MP_ALGO_AUTO resolves to for a call over `tokens` tokens in C chunks (hist != 0: the
 * fused histogram + score pass).  Host-only, no device work. */
int mp_choose_algo(int hist, int W, int64_t tokens, int C, int L, int K, int max_p);

/* ---- unique-destination scoring (extension A17; not a SPEC metric) ------------------------
 * For up to 4 placements (W = 1 tables) and per chunk c:
 *   hop_sums[q*C+c]   += SPEC hops (identical to mp_score_u8)
 *   uniq_sums[q*C+c]  += sum over (t,l) of |{server_q(e_k)} \ {src_srv[q*L+l]}|
 *   dedup_sums[q*C+c] += sum over (t,l) of sum over distinct servers s of the picks of pe_q[l][s]
 * srv_tables: uint32 [L][256], byte q = server id (< 256) hosting expert e under placement q
 * (built by mp_pack_server_tables); src_srv: device uint8 [4][L], the dispatch server per layer.
 * K <= 32.                                                                                   */
int mp_score_dedup_u8(const uint8_t* planes, int64_t plane_stride, int64_t tok_begin, int64_t tok_end, int L, int K,
                      const int64_t* chunk_bounds, int C, const uint32_t* tables, const uint32_t* srv_tables,
                      const uint8_t* src_srv, int64_t* hop_sums, int64_t* uniq_sums, int64_t* dedup_sums,
                      void* stream);
/* srv_tables for mp_score_dedup_u8: server_of: device int32 [T][S] (device -> server per topology). */
int mp_pack_server_tables(const int32_t* server_of, int T, const int32_t* assign, const int32_t* topo_of, int P,
                          int L, int E, int S, uint32_t* srv_tables, int64_t* err, void* stream);

/* ---- topology: all_pairs_hops -------------------------------------
 * Unit-weight BFS over the undirected switch/server graph in CSR form (row_ptr[n_nodes+1],
 * col[nnz]) from every node in src_nodes; dist[i*n_dst + j] = hops(src_nodes[i], dst_nodes[j]).
 * Unreachable pairs raise MP_DATA_UNREACHABLE; hop counts > 255 raise MP_DATA_HOPS_RANGE.
 * n_nodes <= 8192.                                                                            */
int mp_apsp_bfs(const int32_t* row_ptr, const int32_t* col, int n_nodes, const int32_t* src_nodes,
                int n_src, const int32_t* dst_nodes, int n_dst, uint8_t* dist, int64_t* err, void* stream);

/* device-level expansion: out[a*S + b] = dsrv[server[a]*n_srv + server[b]]   */
int mp_expand_dist(const uint8_t* dsrv, int n_srv, const int32_t* dev_server, int S, uint8_t* out,
                   void* stream);

/* ---- cost_matrix: p[l*S + s] = D[d_l][s] + D[s][c_l] ---------------------
 * D given at server level: D[a][b] = dsrv[server[a]*n_srv + server[b]].                        */
int mp_cost_matrix(const uint8_t* dsrv, int n_srv, const int32_t* dev_server, int S,
                   const int32_t* dispatch, const int32_t* collect, int L, uint8_t* p, void* stream);

/* ---- build_instance coefficients ---------------------------
 * f[l][e] = counts[l*E+e] / denom (float64; counts == NULL means uniform f = 1/E), then
 *   w[l][e][s] = f[l][e] * p[l][s]              (float64, nullable output)
 *   w_int[l][e][s] = rint(w[l][e][s] * scale)   (int64 round-half-even, nullable output)
 * in exactly numpy's operation order, so results are bit-identical to the host formula.
 * scale == 0 selects exact integer costs w_int = counts[l][e] * p[l][s] (1 * p when uniform):
 * the same argmin (f is a positive multiple of counts) without the 1e9 rounding.   */
int mp_coeffs(const int64_t* counts, int64_t denom, const uint8_t* p, int L, int E, int S, double scale,
              double* w, int64_t* w_int, void* stream);

/* ---- communication_map ------------------------------------------------
 * traffic[a*n_srv + b] += sum over (l,e) of counts[l*E+e] * D(d_l, s) at (server d_l, server s)
 * and counts[l*E+e] * D(s, c_l) at (server s, server c_l), with s = assign[l*E+e].
 * (Un-normalised and un-symmetrised; the host divides by N and symmetrises.)                 */
int mp_comm_map(const int64_t* counts, const int32_t* assign, const int32_t* dev_server, const uint8_t* dsrv,
                int n_srv, const int32_t* dispatch, const int32_t* collect, int L, int E, int S,
                int64_t* traffic, int64_t* err, void* stream);

/* ---- host -> device staging of a token slice of layer planes (end-to-end path) ---------------
 * Copies `rows` plane rows of `width` bytes from pinned host memory (pitch src_stride) into device
 * memory (pitch dst_stride) with one 2-D async copy on `stream`.  Used to stream a host-resident
 * trace through double-buffered device slices while the kernels run on the previous slice.   */
int mp_copy_planes_h2d(void* dst, int64_t dst_stride, const void* src, int64_t src_stride, int64_t width, int rows,
                       void* stream);

/* ---- batched-scoring operands and the device search loop (A18) --------------------
 * mp_pe_gather_u8: pe[q*ldpe + l*E + e] = cost[topo_of[q]][l][assign[q][l][e]] (topo_of NULL = 0),
 *   columns [L*E, ldpe) zero; an assignment outside [0, topo_S[t]) (topo_S NULL: [0, n_dev)) raises
 *   MP_DATA_UNPLACED err = {4, placement, l*E + e, count}.  cost uint8 [T][L][n_dev] (topologies
 *   zero-padded to the widest), topo_S int32 [T], assign int32 [P][L][E], topo_of int32 [P].
 * mp_perturb_pe_u8: candidate b = pe_cur with n_swaps within-layer swaps (layer l, experts x, y drawn by
 *   Philox4x32-10 keyed by `seed`, counter (b, iter, j, 'SWAP')) -> pe_out[b*ldpe ..], the swaps
 *   (l, x, y) -> swaps int32 [B][n_swaps][3].  Swapping two experts' devices swaps their pe bytes.
 * mp_batch_objective: obj[b] from int64 per-chunk hop sums [B][C] and tokens [C]: kind 0 = mean hops
 *   per token (exact total / tokens), 1 = mean + lam * population std of the per-chunk means, 2 =
 *   the worst per-chunk mean; empty chunks skipped.
 * mp_search_accept: best = argmin obj (lowest index on ties); if obj[best] < *cur_obj, replay its swaps
 *   on assign int32 [L][E] and pe_cur, *cur_obj = obj[best]; history[iter] = *cur_obj and
 *   accepted[iter] = best or -1 (all device pointers: the loop never synchronises the host).
 * mp_objective_f64: out[q] = sum_i f[i] * pe[q*ldpe + i] (float64 f [LE], fixed reduction order) --
 *   objective_value for float frequencies; with integer counts the exact form is
 *   mp_contract_counts with C = 1.                                                                */
int mp_pe_gather_u8(const uint8_t* cost, int T, int L, int n_dev, const int32_t* topo_S, const int32_t* assign,
                    const int32_t* topo_of, int P, int E, uint8_t* pe, int64_t ldpe, int64_t* err, void* stream);
int mp_perturb_pe_u8(const uint8_t* pe_cur, int L, int E, int B, int n_swaps, uint64_t seed, int64_t iter,
                     uint8_t* pe_out, int64_t ldpe, int32_t* swaps, void* stream);
int mp_batch_objective(const int64_t* sums, const int64_t* tokens, int B, int C, int kind, double lam, double* obj,
                       void* stream);
int mp_search_accept(const double* obj, int B, const int32_t* swaps, int n_swaps, int E, int32_t* assign,
                     uint8_t* pe_cur, double* cur_obj, double* history, int64_t iter, int64_t* accepted, void* stream);
int mp_objective_f64(const double* f, const uint8_t* pe, int64_t ldpe, int64_t LE, int P, double* out, void* stream);

/* ---- token-major ingestion (an ActivationTrace is per token) --------------------
 * planes[l][(tok_out + i)*K + k] = tokens[(i*L + l)*K + k] for i < n: the device transpose of a
 * token-major uint8 [n][L][K] slice (router output, or a host array streamed slice by slice) into
 * the layer planes.  `tokens` is a device pointer; K = 8 with an 8-byte aligned `tokens` takes the
 * tiled u64 transpose.                                                                            */
int mp_tokens_to_planes_u8(const uint8_t* tokens, int64_t n, int L, int K, uint8_t* planes, int64_t plane_stride,
                           int64_t tok_out, void* stream);

/* ---- solve_exact: min-cost flow on the class-compressed FlowNetwork ------
 * HOST function (the ILP solve stays on the host).  Costs w_int[l][e][s] are int64 >= 0 in
 * host memory.  When p (host uint8[L][S]) is given, w_int must depend on s only through
 * p[l][s] (true for build_instance output) and the network is class-compressed:
 * item(l,e) -> class(l, p value) -> slot(l,s) -> server(s) -> sink, which has the same optimum
 * as the full network.  p == NULL uses the full item(l,e) -> slot(l,s) arc set of SPEC.md:264-268.
 * Successive shortest paths with potentials.  assign_out: host int32[L][E] (device ids).
 * Returns MP_OK, MP_ERR_ARG, or 4 (= infeasible: max flow < L*E; *flow_out says how much). */
#define MP_INFEASIBLE 4
int mp_solve_mcf(const int64_t* w_int, const uint8_t* p, int L, int E, int S, int c_layer, int c_exp,
                 int32_t* assign_out, int64_t* objective_out, int64_t* flow_out);

#ifdef __cplusplus
}
#endif
#endif /* MOEPLACE_CUDA_H */
