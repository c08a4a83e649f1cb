// Internal launchers of the sm_100a kernels (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace eco {

typedef __nv_bfloat16 bf16;

// ------------------------------------------------------------------ GEMM
// D[m, n] = sum_k A[m, k] * B[n, k]; A [m_rows, K], B [n_rows, K] bf16 row-major.
// "rows"/"cols" below are the logical output (token, feature) coordinates:
//   non-swapped modes: m = token, n = feature   (prefill projections)
//   swapped modes    : m = feature, n = token   (decode skinny GEMMs, LM head)
enum EpiMode : int {
  EPI_F32 = 0,          // out f32 [m][ldo]
  EPI_BF16 = 1,         // out bf16 [m][ldo]
  EPI_RESID = 2,        // resid f32 [m][ldr] += acc
  EPI_SILU = 3,         // out bf16 [m][ldo] at n/2: silu(acc[2j]) * acc[2j+1]
  EPI_QKV = 4,          // RoPE on pair-interleaved q/k heads, q -> q_out, k/v -> paged pool
  EPI_SWAP_F32 = 5,     // out f32 [split][n][ldo] (ldo = padded m), partial sums of a K split
  EPI_SWAP_ARGMAX = 6,  // per token n, per 128-row m tile: (max, lowest argmax) -> am_val/am_idx [n][am_ld]
  // swapped (decode) epilogues applied in-kernel; with splits > 1 every split writes
  // its f32 partial to `part` and the last-arriving CTA of a tile (per-tile counter)
  // sums the partials in split order (deterministic) and applies the epilogue
  EPI_SWAP_BF16 = 7,    // out bf16 [n][ldo] at m
  EPI_SWAP_RESID = 8,   // resid f32 [n][ldr] at m += acc
  EPI_SWAP_SILU = 9,    // out bf16 [n][ldo] at m/2: silu(acc[m even]) * acc[m + 1]
  EPI_SWAP_QKV = 10,    // RoPE on pair-interleaved q/k rows (lanes 2j, 2j+1), KV to the pool
  EPI_SWAP_STORE = 11,  // resid f32 [n][ldr] at m = acc (TP ranks > 0: partial sum before the all-reduce)
};

struct GemmEpi {
  int mode;
  void* out;
  int64_t ldo;
  float* resid;
  int64_t ldr;
  // QKV epilogue
  const int* pos;          // [rows] position of each token
  const int* slot;         // [rows] physical slot = block * 64 + offset
  const float* rope_cos;   // [max_pos][D/2]
  const float* rope_sin;
  bf16* q_out;             // [rows][n_heads][D]
  bf16* k_cache;           // layer base of K (block 0, kv head 0)
  bf16* v_cache;
  int64_t blk_stride;      // elements between consecutive physical blocks
  int n_heads, n_kv, head_dim;
  // argmax epilogue
  float* am_val;
  int* am_idx;
  int am_ld;
  // split-K workspace of the in-kernel reduction (swapped modes 7..10)
  float* part;             // [splits][n_rows][m_rows] f32
  int* counters;           // [m_tiles * n_tiles], zero on entry, left zero on exit
  // which operand does not depend on the previous kernel on the stream (0 none,
  // 1 A, 2 B): it is prefetched into the first smem stages before the PDL wait
  int indep;
  // optional per-CTA phase timestamps (%globaltimer, ns), [grid][16]; null in the engine
  unsigned long long* trace;
  // pair GEMM tile order: token panels per band (0 = default 16)
  int band;
  // L2 prefetch of the NEXT decode GEMM's first stages (null = none): once this CTA's
  // producer has issued its last load it prefetches, into L2, the first pf_kb weight
  // K blocks of the work unit the same blockIdx runs in the next GEMM (tensor map in
  // global memory; geometry m_rows / K / splits / token tiles of that GEMM)
  const CUtensorMap* pf_map;
  int pf_m_rows, pf_K, pf_splits, pf_n_tiles, pf_kb;
  // TP push (N2): when set, the f32 epilogues (EPI_F32, EPI_SWAP_STORE) also store every
  // output element here -- the peer GPU's receive plane over NVLink, same layout as
  // out / resid -- and the epilogue threads end with fence.sys
  float* out2;
  // Prefill deferred RMSNorm (non-swapped epilogues): EPI_RESID with nrm_h also writes
  // nrm_h = bf16(x_new * nrm_gamma) [rows][nrm_ldh] and the row's sum of x_new^2 over its
  // N tile into nrm_ss_out[nt][row] (row stride nrm_ss_ld); EPI_QKV / EPI_SILU with
  // nrm_ss_in scale every output by rsqrt(sum over nrm_ss_n tiles * nrm_inv_h + nrm_eps).
  bf16* nrm_h;
  int64_t nrm_ldh;
  const bf16* nrm_gamma;
  float* nrm_ss_out;
  const float* nrm_ss_in;
  int nrm_ss_ld, nrm_ss_n;
  float nrm_inv_h, nrm_eps;
  // Concurrent decode GEMMs (the gate/up second wave beside the down projection's first K
  // part): flag_set -- CTA 0 stores flag_epoch there once its PDL wait returned (its inputs,
  // and so the inputs of later kernels that read the same buffers, are complete);
  // flag_wait -- the GEMM does not wait for the previous kernel: its producer waits until
  // *flag_wait >= flag_epoch instead, the epilogue writes without waiting, and thread 0
  // of every CTA waits for the previous kernel at the very end (so kernels launched after
  // this one still wait, through it, for the one before it).
  int* flag_set;
  const int* flag_wait;
  int flag_epoch;
  // decode (indep == 1): after the first smem stages, prefetch up to this many more of the
  // CTA's weight K blocks into L2 before the PDL wait (0 = none)
  int l2_pf_kb;
  // deferred RMSNorm (decode flow path): the GEMM input was bf16(x * gamma), so the QKV
  // epilogues (EPI_SWAP_QKV, RED_QKV) multiply token n's outputs by rvec[n] = 1/rms(x_n)
  const float* rvec;
  // balanced split-K of a decode projection (EPI_SWAP_F32 partials, one token tile,
  // sk_L > 0): the m_tiles x sk_kbt sequence of (weight tile, K block) units is cut into
  // equal chunks of sk_L units and CTA c streams chunk c, so every SM streams the same
  // number of K blocks (a uniform split leaves tiles x splits CTAs, e.g. 128 of 148 SMs,
  // busy). Its piece of tile t goes to partial slot c - (t * sk_kbt) / sk_L; tile t has
  // sk_slots(t) slots, summed in slot (= K) order by the reductions.
  int sk_L, sk_kbt;
  // bulk-store epilogues: 1 = copy the staged token rows out with one async bulk copy per
  // row (cp.async.bulk) instead of 16-byte st.global from the 4 epilogue warps
  // (ECOSERVE_EPI_BULK=1; measured slower in the decode step, so off by default)
  int bulk_copy;
};

// Partial slots of weight tile `tile` under the balanced split (see GemmEpi::sk_L).
__host__ __device__ __forceinline__ int sk_slots(int tile, int kbt, int L) {
  return ((tile + 1) * kbt - 1) / L - (tile * kbt) / L + 1;
}
// Balanced chunk length for m_tiles weight tiles of kbt K blocks on num_sms SMs, at
// most max_slots partial slots per tile; 0 when a uniform split is at least as balanced.
int gemm_sk_chunk(int m_tiles, int kbt, int num_sms, int max_slots);

// Split count for a decode GEMM: minimises waves x K-blocks per CTA (+ a per-split reduction cost).
int gemm_choose_splits(int m_rows, int n_rows, int K, int bn, int num_sms, int max_splits);
// Split count of the engine's decode GEMMs: no split once the weight tiles cover 3/4 of
// the SMs, else the s in 1..4 with the fewest K blocks on the busiest CTA (waves x K blocks
// per split + a reduction cost) -- the 8B choices of the measured sweep
// (tools/gemm_decode_sweep.py), and 3 instead of 4 for the 70B/TP=2 QKV (40 tiles).
int gemm_decode_splits(int m_rows, int K, int num_sms);

// Creates a 2D bf16 tensor map (rows x cols, row-major, 128B swizzle, box 64 x box_rows).
int make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int box_rows);
// Plain (unswizzled) 2D map for TMA stores / reductions from row-major smem tiles:
// f32 (f32 != 0) or bf16 [rows][cols], box box_cols x box_rows.
int make_tmap_2d_plain(CUtensorMap* map, const void* ptr, int f32, int64_t rows, int64_t cols, int box_cols,
                       int box_rows);
// General bf16 tensor map, 128B swizzle: dims[0] innermost; strides_bytes[i] of dim i+1.
int make_tmap_bf16_nd(CUtensorMap* map, const void* ptr, int rank, const int64_t* dims, const int64_t* strides_bytes,
                      const int* box);

// Launch; tile width bn in {64, 128, 256}; splits > 1 only with EPI_SWAP_F32.
cudaError_t gemm_launch(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K, int bn,
                        int splits, const GemmEpi& epi, int num_sms, cudaStream_t stream);
// r = 128-row A tiles per work unit (1 or 2; 2 needs an A tensor map with a 256-row box
// and a swapped epilogue without the in-kernel split reduction).
cudaError_t gemm_launch_r(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K, int bn,
                          int r, int splits, const GemmEpi& epi, int num_sms, cudaStream_t stream);
int gemm_smem_bytes(int bn);
// Swap-AB decode GEMM with K split over the CTAs of a thread-block cluster (splits 2..4,
// bn 64 / 128) and the split reduction done in distributed shared memory; swapped
// in-kernel epilogues (modes >= EPI_SWAP_BF16). splits must equal gemm_effective_splits.
cudaError_t gemm_cluster_launch(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K,
                                int bn, int splits, const GemmEpi& epi, cudaStream_t stream);
// How many clusters of `splits` CTAs of that kernel can be resident at once (0 if unsupported).
int gemm_cluster_max_active(int bn, int splits);

// ------------------------------------------------------------------ decode layer chain
// One persistent kernel (one CTA per SM) runs the post-attention GEMMs of a decode layer
// -- O, gate/up, down and the next layer's QKV -- with a grid-wide barrier between them
// instead of kernel boundaries. Every GEMM is partitioned stream-K: CTA c owns an equal
// contiguous range of the flattened (tile, K-block) iterations; the CTAs sharing a tile
// add their f32 partials with L2 atomics (into x for the residual modes, else into a
// zeroed tile buffer) and the last one to arrive (counter) applies the epilogue -- the
// sum order of a split tile is therefore not fixed (fp32 rounding may differ run to
// run); the epilogues carry the rest of the layer:
//   CE_RESID_SS  x += acc; hb = bf16(x * gamma) (the next RMSNorm's input before its
//                1/rms); ssp[m-tile][tok] = sum of x^2 over the tile's 128 features
//   CE_SILU_R    acc *= r_tok (r = rsqrt(sum_t ssp[t][tok] / H + eps)): the RMSNorm
//                scale applied after the GEMM; out = silu(gate) * up
//   CE_QKV_R     acc *= r_tok; RoPE on the pair-interleaved q / k rows; q, paged K / V
// The producer streams a GEMM's weights into free smem stages before the barrier and
// waits only before its activation loads.
enum ChainEpi : int { CE_RESID_SS = 0, CE_SILU_R = 1, CE_QKV_R = 2 };
struct ChainStep {
  const CUtensorMap* wmap;  // weights [m_rows][K], 128-row box (device memory)
  const CUtensorMap* xmap;  // activations [tok][K], 128-row box (device memory)
  int m_rows, K, mode;
  float* x;                 // CE_RESID_SS: residual [tok][m_rows] f32
  const bf16* gamma;        //   next RMSNorm weight [m_rows]
  bf16* hb;                 //   bf16(x * gamma) [tok][m_rows]
  float* ssp_out;           //   [m_rows / 128][ss_ld]
  const float* ssp_in;      // CE_SILU_R / CE_QKV_R: [ssp_tiles][ss_ld] of the previous step
  int ssp_tiles, H;
  float eps;
  GemmEpi e;                // SILU_R: e.out bf16 [tok][e.ldo]; QKV_R: RoPE / q / pool geometry
  int* counters;            // per-tile arrivals of this step (zero on entry, left zero)
};
struct ChainCall {
  int n_tok, ss_ld;               // tokens (<= 512); row stride of the ssp buffers
  const int* pos;                 // [n_tok] (CE_QKV_R)
  const int* slot;                // [n_tok] (CE_QKV_R)
  float* ws;                      // split tiles' f32 sums [tiles][128 tok][128] (zero on entry, left zero)
  unsigned long long* bar;        // grid-barrier counter, monotonic across launches
  unsigned long long bar_base;    // its value when this launch starts
  int* err;                       // set to 1 if a grid barrier timed out (CTAs not co-resident)
  unsigned long long* trace;      // optional %globaltimer marks [grid][32 steps][4] (null: off)
};
// grid = num_sms CTAs; the counter advances by n_steps * grid per launch
cudaError_t decode_chain_launch(const ChainStep* d_steps, int n_steps, const ChainCall& c, int num_sms,
                                cudaStream_t stream);
// CTA-pair (cta_group::2) 256 x 256-tile variant for the non-swapped (prefill) epilogues.
// mapA box 128 rows (A), mapB box 128 rows (half of the 256 B rows of a tile).
cudaError_t gemm2_launch(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K,
                         const GemmEpi& epi, int num_sms, cudaStream_t stream);
// The number of K splits gemm_launch actually runs for a requested count (every
// split owns >= 1 K block); the reduction must use the same number.
int gemm_effective_splits(int K, int splits);

// ------------------------------------------------------------------ attention
// Prefill causal varlen attention over the paged pool (mma.sync, FA2-style online softmax).
struct PrefillAttnArgs {
  const bf16* q;            // [T][M][D]
  const bf16* k_cache;      // layer base
  const bf16* v_cache;
  int64_t blk_stride;
  const int* cu_seqlens;    // [n_seq + 1]
  const int* block_tables;  // [n_seq][bt_ld]
  int bt_ld;
  const int* tiles;         // [n_tiles][2]: (seq, q_start) for 128-row q tiles
  int n_tiles;
  bf16* out;                // [T][M*D]
  int n_heads, n_kv;
  float scale_log2;         // log2(e) / sqrt(D)
  const int* ctx_off;       // optional [n_seq]: cached tokens before this chunk (chunked prefill)
};
cudaError_t attn_prefill_launch(const PrefillAttnArgs& a, int head_dim, cudaStream_t s);

// Prefill causal attention on tcgen05 (head_dim 128): 128-query tiles, K/V by TMA from the
// block-major pool. qmap: 3D map over q [q_rows][n_heads][128]; kvmap: 2D map over the pool
// as rows of 128 elements (rows = num_blocks * L * 2 * Mkv * 64).
int make_attn_tc_maps(CUtensorMap* qmap, CUtensorMap* kvmap, const void* q, int64_t q_rows, int n_heads,
                      const void* pool, int64_t pool_rows);
// ctx_off (optional [n_seq]): tokens of each sequence already in the pool before this
// chunk; its q rows sit at positions ctx_off + i and attend to pool keys 0..position.
// timing probe (tools/attn_bench): when set, CTA (trace_tile, 0) of the next launches
// records clock64 stamps per KV block into trace[20][64] (see attention_tc.cu)
void attn_tc_set_trace(long long* trace, int trace_tile);
cudaError_t attn_prefill_tc_launch(const CUtensorMap* qmap, const CUtensorMap* kvmap, const int* cu_seqlens,
                                   const int* block_tables, int bt_ld, const int* tiles, int n_tiles, bf16* out,
                                   int n_heads, int n_kv, int layer, int n_layers, cudaStream_t s,
                                   const int* ctx_off = nullptr, int mean_keys = 0);
// (mean_keys: keys attended per query token, averaged over the batch -- selects the
// 128-key kernel for long prompts unless ECOSERVE_ATTN_T128 forces a choice)

// Decode split-K paged attention + combine.
struct DecodeAttnArgs {
  const bf16* q;            // [B][M][D]
  const bf16* k_cache;
  const bf16* v_cache;
  int64_t blk_stride;
  const int* ctx_lens;      // [B] tokens incl. the current one
  const int* block_tables;  // [B][bt_ld]
  int bt_ld;
  int B, n_heads, n_kv;
  int n_splits, blocks_per_split;
  float* part_o;            // [B][M][n_splits][D]
  float* part_ml;           // [B][M][n_splits][2] (max (log2 domain), sum)
  bf16* out;                // [B][M*D]
  float scale_log2;
  const int* order;         // optional [B]: sequences longest-context first (null = 0..B-1)
  // optional (head_dim 128): TMA map over the pool as rows of 128 elements (see
  // make_attn_tc_maps) -> K / V blocks staged by TMA instead of cp.async; layer / n_layers
  // locate the layer in the block-major pool
  const CUtensorMap* kvmap;
  int layer, n_layers;
  // optional (TMA path): the QKV projection's split-K f32 partials [qkv_splits][B][qkv_ld]
  // instead of q -- each CTA sums its q heads and its kv head's new k / v row in split
  // order, applies RoPE (pair-interleaved prepared rows, tables rope_cos / rope_sin at
  // pos[b]) and writes the new K / V into the pool at slot[b] itself (the split that owns
  // the last block), replacing the separate reduction kernel (a13)
  const float* qkv_part = nullptr;
  int qkv_splits = 0, qkv_ld = 0;
  const int* pos = nullptr;
  const int* slot = nullptr;
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  // optional (TMA path, head_dim 128, G <= 4): persistent stream-K decode attention. The
  // (rank, kv head, 64-token block) units in LPT rank order are split evenly over
  // sk_grid CTAs; items cut between CTAs are combined by their last contributor.
  const int* sk_prefix = nullptr;  // [B + 1] blocks before each LPT rank (rank r = sequence order[r])
  int* sk_cnt = nullptr;           // [B * n_kv] arrival counters, zero at rest
  int sk_grid = 0, sk_maxp = 0;    // CTAs; parts per item bound (workspace stride)
};
cudaError_t attn_decode_launch(const DecodeAttnArgs& a, int head_dim, cudaStream_t s);
// the stream-K kernel applies (and is enabled: ECOSERVE_ATTN_SK=1, or force for the op-level
// entry point): returns its grid (0 = use the per-item kernel)
int attn_decode_sk_grid(int total_units, int max_item_blocks, int min_item_blocks, int n_heads, int n_kv,
                        int head_dim, int num_sms, int* maxp, bool force = false);

// ------------------------------------------------------------------ TP=2 fused all-reduce (N2)
struct TpAllreduceArgs {
  const float* recv0;      // rank 0's projection output [splits][rows][H] f32 (this GPU's receive plane)
  const float* recv1;      // rank 1's
  int splits;              // split-K partials per rank, summed in split order (prefill: 1)
  float* x;                // residual [rows][H] f32, updated in place: x = (x + recv0) + recv1
  const bf16* gamma;       // next RMSNorm weight, or null (x only)
  bf16* h;                 // rmsnorm(x) * gamma [rows][H]
  float eps;
  int rows, H, epoch;
  int* peer_flag;          // the peer's flag (P2P): set to epoch once this rank's pushes are done
  const int* my_flag;      // set by the peer
  int* err;                // set to 1 when the peer's flag did not arrive within timeout_ns
  unsigned long long timeout_ns;
};
cudaError_t tp_allreduce_norm_launch(const TpAllreduceArgs& a, int num_sms, cudaStream_t s);
// decode variant: sums this rank's split partials per row and pushes the row itself
struct TpRowsArgs {
  const float* part;       // this rank's partials [splits][plane] (row stride ldp)
  int splits;
  int64_t plane, ldp;
  float* x;
  const bf16* gamma;
  bf16* h;
  float eps;
  int rows, H, rank, epoch;
  float* peer_recv;        // the peer's receive rows of this epoch's parity [rows][H] (P2P)
  int* peer_flags;         // the peer's row flags of this parity [rows] (P2P)
  const float* my_recv;    // this rank's receive rows, written by the peer
  const int* my_flags;
  int* err;                // as TpAllreduceArgs
  unsigned long long timeout_ns;
  int sk_L, sk_kbt;        // balanced split (GemmEpi::sk_L): per-tile slot counts instead of splits
};
cudaError_t tp_push_rows_launch(const TpRowsArgs& a, int num_sms, cudaStream_t s);

// ------------------------------------------------------------------ decode flow
// One persistent kernel per decoder layer runs the O projection, gate/up (+SiLU) and
// down projection of a decode step (rows a9-a11 / a15) as a dataflow: every GEMM's
// K blocks are spread evenly over all CTAs (split tiles summed by their last arriving
// contributor in fixed order), and each CTA's activation loads wait on per-tile
// readiness flags of the producing GEMM instead of a kernel boundary, while its weight
// loads run ahead. RMSNorm is deferred: the O / down reducers write x (f32), h =
// bf16(x * gamma_next) and per-tile sums of squares; the consumer (gate/up epilogue,
// next QKV reduction) multiplies by 1/rms. See decode_flow.cu.
struct FlowArgs {
  int B;                   // tokens (<= BN)
  int H, F, MD;            // hidden, FFN width, heads * head_dim
  int epoch;               // flags of this launch read as ready when >= epoch
  float eps, inv_h;
  float* x;                // [>=B][H] f32 residual, updated in place
  bf16* h;                 // [>=B][H] gate/up input: bf16(x * gamma_o) after O
  bf16* h_out;             // [>=B][H] bf16(x * gamma_d) after down (next QKV / LM head input)
  bf16* act;               // [>=B][F] silu(g) * u
  const bf16* gamma_o;     // ffn_norm of this layer
  const bf16* gamma_d;     // next layer's attn_norm, or the final norm
  float* ss_o;             // [H/128][128] per-tile sums of x^2 after O
  float* ss_d;             // [H/128][128] after down
  float* rvec;             // [128] 1/rms(x) after down (read by the next QKV epilogue)
  int* flags_o;            // [H/128]
  int* flags_gu;           // [2F/128]
  int* cnt;                // [6][cnt_ld] per-tile arrival (g) and reduced (3 + g) counters, zero at rest
  int cnt_ld;
  int* done_d;             // completed down tiles, zero at rest
  float* slots;            // [3][grid][2][BN * 128] f32 partial tiles
  int* err;                // set on a dependency-wait timeout (CTAs not co-resident)
  unsigned long long* trace;  // debug: [grid][16] %globaltimer marks, or null
};
// BN (64 or 128) >= B. maps: weights (128-row boxes) of O, gate/up, down; activations
// ao / h / act as B operands with BN-row boxes.
// x_map: f32 x [rows][H], box 128 x 32 (TMA reduce-add of split partials); act_map: bf16
// act [rows][F], box 64 x 32 (TMA store of the gate/up output). Both unswizzled.
cudaError_t decode_flow_launch(const CUtensorMap* w_o, const CUtensorMap* w_gu, const CUtensorMap* w_d,
                               const CUtensorMap* b_o, const CUtensorMap* b_gu, const CUtensorMap* b_d,
                               const CUtensorMap* x_map, const CUtensorMap* act_map, const FlowArgs& a, int bn,
                               int num_sms, cudaStream_t s);
int64_t decode_flow_slot_floats(int num_sms);  // size of FlowArgs::slots

// ------------------------------------------------------------------ decode gate/up, stream-K
// (decode_gu.cu) act = silu(gate) * up of W_gu [m_rows = 2F][K = H] x h [B][H], every
// CTA streaming the same number of weight K blocks; a tile split between two CTAs is
// finished by the head's owner from the tail's partial (flags[t] >= epoch) -- a
// two-term sum, bitwise deterministic.
struct GuSkArgs {
  int m_rows, K, B, epoch;
  int* flags;              // [m_rows / 128], epoch of the tail partial's store
  int* err;                // set on a flag-wait timeout (CTAs not co-resident)
  unsigned long long* trace;  // debug: [grid][16] %globaltimer marks, or null
};
bool gu_sk_applicable(int m_rows, int K, int B, int num_sms);
// w_map: W_gu (128-row boxes, SW128), x_map: h as B operand (bn-row box), act_map: bf16
// act [rows][F] box 64 x 32 (plain), part_map: f32 partials [m_rows][128] box 128 x 32.
cudaError_t gu_sk_launch(const CUtensorMap* w_map, const CUtensorMap* x_map, const CUtensorMap* act_map,
                         const CUtensorMap* part_map, const GuSkArgs& a, int bn, int num_sms, cudaStream_t s);

// ------------------------------------------------------------------ small kernels
// x[t] = E[clamp(ids[t], 0, V-1)] (fp32)
cudaError_t embed_launch(const int* ids, const bf16* E, float* x, int n, int H, int V, cudaStream_t s);
cudaError_t rmsnorm_launch(const float* x, int64_t ldx, const int* rows, const bf16* gamma, bf16* out, int n, int H,
                           float eps, cudaStream_t s);
// dst[r] = src_sel[r][row[r]] (row copy of `cols` bf16), sel in {0,1,2} -> s0/s1/s2.
cudaError_t row_gather_launch(const bf16* s0, const bf16* s1, const bf16* s2, const int* sel, const int* row, bf16* dst,
                              int nrows, int cols, cudaStream_t s);
// x[row] += sum_s part[s][row] (split order); out[row] = bf16(rmsnorm(x[row]) * gamma). part plane = rows x H.
cudaError_t splitk_resid_rmsnorm_launch(const float* part, int splits, int rows, float* x, const bf16* gamma,
                                        bf16* out, int H, float eps, cudaStream_t s, int sk_L = 0, int sk_kbt = 0);
// tokens[i] = argmax over the [n][parts] (val, idx) partials; NaN wins, and a NaN row
// yields ECO_TOKEN_NAN (reading A6) instead of a token id.
constexpr int ECO_TOKEN_NAN = -2;
cudaError_t argmax_reduce_launch(const float* val, const int* idx, int n, int parts, int ld, int* tokens,
                                 cudaStream_t s);
// Decode epilogues (after a split-K swap GEMM): sum partial[split][row][col] in fixed split order
// (epi.sk_L > 0: the balanced split's sk_slots(col / 128) slots), then
enum RedMode : int { RED_BF16 = 0, RED_RESID = 1, RED_SILU = 2, RED_QKV = 3, RED_F32 = 4 };
cudaError_t splitk_reduce_launch(int mode, const float* part, int splits, int rows, int cols, int64_t ld_part,
                                 const GemmEpi& epi, cudaStream_t s);

}  // namespace eco
