/* ecoserve_ops.h -- op-level entry points of the same CUDA kernels the phases
 * run, for kernel-by-kernel parity tests and microbenchmarks. All pointers are
 * device pointers on the current device; every call is asynchronous on
 * `stream` (a cudaStream_t, NULL = legacy default stream) and returns
 * ECOSERVE_ERR_CUDA on a launch error, ECOSERVE_ERR_INVALID_ARG on bad sizes.
 * Nothing is allocated except where noted (workspace arguments are caller
 * memory). */
#ifndef ECOSERVE_OPS_H_
#define ECOSERVE_OPS_H_
#include <stdint.h>
#include "ecoserve.h"
#ifdef __cplusplus
extern "C" {
#endif

/* D = A B^T on tcgen05 (Table 2 projections). A [m][k], B [n][k] bf16
 * row-major, k % 64 == 0 is not required (TMA zero-fills). out_mode 0: out f32
 * [m][n]; 1: out bf16 [m][n]. bn in {64, 128, 256}: one CTA per 128 x bn tile;
 * bn = 2: the CTA-pair (cta_group::2) kernel with 256 x 256 tiles. */
ecoserve_status ecoserve_op_gemm(const void* A, const void* B, int32_t m, int32_t n, int32_t k, int32_t out_mode,
                                 void* out, int32_t bn, void* stream);

/* Decode-shaped ("swap-AB") GEMM: out f32 [n][m] = (W [m][k]) (X [n][k])^T with
 * weights as the 128-row MMA M side, tokens as N, K split `splits` ways into the
 * caller's workspace f32 [splits][n][m], then a fixed-order reduction. */
ecoserve_status ecoserve_op_gemm_swap(const void* W, const void* X, int32_t m, int32_t n, int32_t k, int32_t splits,
                                      float* workspace, float* out, int32_t bn, void* stream);

/* The decode-phase form of the same GEMM: in-kernel split-K reduction (the last
 * CTA of each tile sums the f32 partials of all splits in split order) and an
 * in-kernel epilogue writing out bf16 [n][m]. part: f32 [splits][n][m];
 * counters: int32 [ceil(m/128) * ceil(n/bn)], zero on entry, zero on return. */
ecoserve_status ecoserve_op_gemm_swap_bf16(const void* W, const void* X, int32_t m, int32_t n, int32_t k,
                                           int32_t splits, float* part, int32_t* counters, void* out, int32_t bn,
                                           void* stream);

/* The engine's decode GEMM: out f32 [n][m] = X W^T with r (1 or 2) 128-row weight
 * tiles per CTA sharing one activation tile; splits == 1: written by the GEMM
 * epilogue; splits > 1: f32 partials in `ws` [splits][n][m] + fixed-order reduction. */
ecoserve_status ecoserve_op_gemm_decode(const void* W, const void* X, int32_t m, int32_t n, int32_t k, int32_t r,
                                        int32_t splits, float* ws, float* out, int32_t bn, void* stream);

/* The same decode GEMM with the balanced split-K (the engine's O / down / QKV
 * projections when their weight tiles are fewer than the SMs; Table 2 P:232-236,
 * SURVEY 8(a) rows a13, a15): the ceil(m/128) x ceil(k/64) sequence of (weight tile,
 * K block) units is cut into equal chunks of *chunk units, one CTA per chunk, so every
 * SM streams the same number of weight blocks; each CTA writes the f32 partial of every
 * tile its chunk touches into slot (cta - first cta of the tile) of ws, and the reduction
 * sums each tile's slots in K order. n <= bn (one token tile). ws: f32
 * [max_slots][n][m] (device, caller-owned). *chunk (host) receives the chunk length
 * used (0: no balanced split exists for these sizes -> ECOSERVE_ERR_INVALID_ARG). */
ecoserve_status ecoserve_op_gemm_decode_balanced(const void* W, const void* X, int32_t m, int32_t n, int32_t k,
                                                 int32_t max_slots, float* ws, float* out, int32_t bn,
                                                 int32_t* chunk, void* stream);

/* Decode GEMM with the K split over the CTAs of a thread-block cluster and the split
 * reduction in distributed shared memory (no partials in HBM): out f32 [n][m] =
 * X W^T, partials summed in split order. splits 2..4 (clamped so every split owns a
 * K block; ECOSERVE_ERR_INVALID_ARG outside), bn 64 or 128. */
ecoserve_status ecoserve_op_gemm_cluster(const void* W, const void* X, int32_t m, int32_t n, int32_t k,
                                         int32_t splits, float* out, int32_t bn, void* stream);

/* Greedy LM head (rows a12/a16): tokens[i] = argmax_v (X [n][k] W[v][k]^T), lowest
 * v on ties, logits never materialised. workspace: f32 [n][ceil(V/128)] and
 * i32 [n][ceil(V/128)]. */
ecoserve_status ecoserve_op_lm_argmax(const void* W, const void* X, int32_t V, int32_t n, int32_t k, float* ws_val,
                                      int32_t* ws_idx, int32_t* tokens, void* stream);

/* out bf16 [n][H] = rmsnorm(x f32 [rows[i] or i][H]) * gamma (A4). */
ecoserve_status ecoserve_op_rmsnorm(const float* x, const int32_t* rows, const void* gamma, void* out, int32_t n,
                                    int32_t H, float eps, void* stream);

/* Causal varlen prefill attention over a paged pool laid out as in ecoserve.h
 * for a single layer (n_layers = 1): q bf16 [T][M][D] (RoPE applied), out bf16
 * [T][M*D]. block_tables int32 [n_seq][bt_ld] (physical block of each 64-token
 * logical block). ctx_off_host (host int32 [n_seq], or NULL = zeros): chunked
 * prefill -- sequence s's q rows are the chunk at positions ctx_off[s] + i, attending
 * to pool keys 0 .. ctx_off[s] + i (the earlier chunks' K / V already in the pool). */
ecoserve_status ecoserve_op_attention_prefill(const void* q, const void* pool, int64_t num_blocks, int32_t n_heads,
                                              int32_t n_kv, int32_t head_dim, const int32_t* cu_seqlens_host,
                                              int32_t n_seq, const int32_t* block_tables, int32_t bt_ld, void* out,
                                              void* stream, const int32_t* ctx_off_host);

/* The same prefill attention on tcgen05 (head_dim 128 only): 128-query tiles, S and
 * P V accumulated in TMEM, K / V loaded by TMA from the pool. */
ecoserve_status ecoserve_op_attention_prefill_tc(const void* q, const void* pool, int64_t num_blocks,
                                                 int32_t n_heads, int32_t n_kv, const int32_t* cu_seqlens_host,
                                                 int32_t n_seq, const int32_t* block_tables, int32_t bt_ld, void* out,
                                                 void* stream, const int32_t* ctx_off_host);

/* Split-K decode attention over the same pool: q bf16 [B][M][D], ctx_lens int32
 * [B] (device), out bf16 [B][M*D]. n_splits x blocks_per_split must cover the
 * longest context; workspace f32 [B][M][n_splits][D + 2]. use_tma (head_dim 128):
 * stage K / V by TMA (the engine's path) instead of cp.async. */
ecoserve_status ecoserve_op_attention_decode(const void* q, const void* pool, int32_t n_heads, int32_t n_kv,
                                             int32_t head_dim, const int32_t* ctx_lens, int32_t B,
                                             const int32_t* block_tables, int32_t bt_ld, int32_t n_splits,
                                             int32_t blocks_per_split, float* workspace, void* out, void* stream,
                                             int32_t use_tma);

/* The persistent stream-K decode attention (head_dim 128, n_heads / n_kv <= 4; the
 * engine uses it with ECOSERVE_ATTN_SK=1 when the work is large enough): sequences in longest-first order,
 * their (kv head, 64-token block) units split evenly over 2 CTAs per SM, items cut
 * between CTAs combined by their last contributor. ctx_host: host int32 [B];
 * block_tables: device int32 [B][bt_ld] into a single-layer pool; workspace: device f32
 * >= B * n_heads * 64 * (head_dim + 2); counters: device int32 [B * n_kv], zero (left
 * zero); meta: device int32 scratch >= 2B + 1. Synchronous. ECOSERVE_ERR_UNSUPPORTED
 * when the work is too small or the group too wide for this kernel. */
ecoserve_status ecoserve_op_attention_decode_sk(const void* q, const void* pool, int32_t n_heads, int32_t n_kv,
                                                int32_t head_dim, const int32_t* ctx_host, int32_t B,
                                                const int32_t* block_tables, int32_t bt_ld, float* workspace,
                                                int32_t* counters, int32_t* meta, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
