// Op-level entry points of include/ecoserve_ops.h: thin wrappers that run the
// same kernels the phase executors use, for kernel-by-kernel parity tests.
#include <string.h>

#include <vector>

#include "../../include/ecoserve_ops.h"
#include "kernels.h"

#include <algorithm>
#include <vector>

using namespace eco;

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

#define OPCK(expr)                                   \
  do {                                               \
    if ((expr) != cudaSuccess) return ECOSERVE_ERR_CUDA; \
  } while (0)

extern "C" {

ecoserve_status ecoserve_op_gemm(const void* A, const void* B, int32_t m, int32_t n, int32_t k, int32_t out_mode,
                                 void* out, int32_t bn, void* stream) {
  if (!A || !B || !out || m < 1 || n < 1 || k < 1 || k % 8 || (out_mode != 0 && out_mode != 1)) return ECOSERVE_ERR_INVALID_ARG;
  if (bn != 2 && bn != 64 && bn != 128 && bn != 256) return ECOSERVE_ERR_INVALID_ARG;
  CUtensorMap ma, mb;
  if (make_tmap_bf16(&ma, A, m, k, 128) || make_tmap_bf16(&mb, B, n, k, bn == 2 ? 128 : bn)) return ECOSERVE_ERR_CUDA;
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  e.mode = out_mode == 0 ? EPI_F32 : EPI_BF16;
  e.out = out;
  e.ldo = n;
  if (out_mode == 1 && n % 8) return ECOSERVE_ERR_INVALID_ARG;
  if (out_mode == 0 && n % 4) return ECOSERVE_ERR_INVALID_ARG;
  if (bn == 2)
    OPCK(gemm2_launch(&ma, &mb, m, n, k, e, num_sms(), (cudaStream_t)stream));
  else
    OPCK(gemm_launch(&ma, &mb, m, n, k, bn, 1, e, num_sms(), (cudaStream_t)stream));
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_op_gemm_swap(const void* W, const void* X, int32_t m, int32_t n, int32_t k, int32_t splits,
                                      float* workspace, float* out, int32_t bn, void* stream) {
  if (!W || !X || !workspace || !out || m < 1 || n < 1 || k < 1 || k % 8 || m % 2 || splits < 1)
    return ECOSERVE_ERR_INVALID_ARG;
  if (bn != 64 && bn != 128 && bn != 256) return ECOSERVE_ERR_INVALID_ARG;
  CUtensorMap ma, mb;
  if (make_tmap_bf16(&ma, W, m, k, 128) || make_tmap_bf16(&mb, X, n, k, bn)) return ECOSERVE_ERR_CUDA;
  const int eff = gemm_effective_splits(k, splits);
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  e.mode = EPI_SWAP_F32;
  e.out = workspace;
  e.ldo = m;
  OPCK(gemm_launch(&ma, &mb, m, n, k, bn, eff, e, num_sms(), (cudaStream_t)stream));
  GemmEpi r;
  memset(&r, 0, sizeof(r));
  r.out = out;
  r.ldo = m;
  OPCK(splitk_reduce_launch(RED_F32, workspace, eff, n, m, m, r, (cudaStream_t)stream));
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_op_gemm_swap_bf16(const void* W, const void* X, int32_t m, int32_t n, int32_t k,
                                           int32_t splits, float* part, int32_t* counters, void* out, int32_t bn,
                                           void* stream) {
  if (!W || !X || !out || m < 1 || n < 1 || k < 1 || k % 8 || splits < 1 || (splits > 1 && (!part || !counters)))
    return ECOSERVE_ERR_INVALID_ARG;
  if (bn != 64 && bn != 128 && bn != 256) return ECOSERVE_ERR_INVALID_ARG;
  CUtensorMap ma, mb;
  if (make_tmap_bf16(&ma, W, m, k, 128) || make_tmap_bf16(&mb, X, n, k, bn)) return ECOSERVE_ERR_CUDA;
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  e.mode = EPI_SWAP_BF16;
  e.out = out;
  e.ldo = m;
  e.part = part;
  e.counters = counters;
  OPCK(gemm_launch(&ma, &mb, m, n, k, bn, gemm_effective_splits(k, splits), e, num_sms(), (cudaStream_t)stream));
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_op_gemm_cluster(const void* W, const void* X, int32_t m, int32_t n, int32_t k,
                                         int32_t splits, float* out, int32_t bn, void* stream) {
  if (!W || !X || !out || m < 1 || n < 1 || k < 1 || k % 8 || m % 2 || (bn != 64 && bn != 128))
    return ECOSERVE_ERR_INVALID_ARG;
  const int eff = gemm_effective_splits(k, splits);
  if (eff < 2 || eff > 4) return ECOSERVE_ERR_INVALID_ARG;
  CUtensorMap ma, mb;
  if (make_tmap_bf16(&ma, W, m, k, 128) || make_tmap_bf16(&mb, X, n, k, bn)) return ECOSERVE_ERR_CUDA;
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  e.mode = EPI_SWAP_STORE;
  e.resid = out;
  e.ldr = m;
  OPCK(gemm_cluster_launch(&ma, &mb, m, n, k, bn, eff, e, (cudaStream_t)stream));
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_op_gemm_decode(const void* W, const void* X, int32_t m, int32_t n, int32_t k, int32_t r,
                                        int32_t splits, float* ws, float* out, int32_t bn, void* stream) {
  if (!W || !X || !out || m < 1 || n < 1 || k < 1 || k % 8 || m % 2 || splits < 1 || r < 1 || r > 3 ||
      (splits > 1 && !ws))
    return ECOSERVE_ERR_INVALID_ARG;
  if (bn != 64 && bn != 128) return ECOSERVE_ERR_INVALID_ARG;
  CUtensorMap ma, mb;
  if (make_tmap_bf16(&ma, W, m, k, r == 2 ? 256 : 128) || make_tmap_bf16(&mb, X, n, k, bn)) return ECOSERVE_ERR_CUDA;
  const int eff = gemm_effective_splits(k, splits);
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  if (eff == 1) {
    e.mode = EPI_SWAP_STORE;
    e.resid = out;
    e.ldr = m;
    OPCK(gemm_launch_r(&ma, &mb, m, n, k, bn, r, 1, e, num_sms(), (cudaStream_t)stream));
    return ECOSERVE_OK;
  }
  e.mode = EPI_SWAP_F32;
  e.out = ws;
  e.ldo = m;
  OPCK(gemm_launch_r(&ma, &mb, m, n, k, bn, r, eff, e, num_sms(), (cudaStream_t)stream));
  GemmEpi red;
  memset(&red, 0, sizeof(red));
  red.out = out;
  red.ldo = m;
  OPCK(splitk_reduce_launch(RED_F32, ws, eff, n, m, m, red, (cudaStream_t)stream));
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_op_gemm_decode_balanced(const void* W, const void* X, int32_t m, int32_t n, int32_t k,
                                                 int32_t max_slots, float* ws, float* out, int32_t bn,
                                                 int32_t* chunk, void* stream) {
  if (!W || !X || !ws || !out || !chunk || m < 1 || n < 1 || k < 1 || k % 8 || m % 4 || max_slots < 1 ||
      (bn != 64 && bn != 128) || n > bn)
    return ECOSERVE_ERR_INVALID_ARG;
  const int kbt = (k + 63) / 64;
  const int L = gemm_sk_chunk((m + 127) / 128, kbt, num_sms(), max_slots);
  *chunk = L;
  if (L <= 0) return ECOSERVE_ERR_INVALID_ARG;
  CUtensorMap ma, mb;
  if (make_tmap_bf16(&ma, W, m, k, 128) || make_tmap_bf16(&mb, X, n, k, bn)) return ECOSERVE_ERR_CUDA;
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  e.mode = EPI_SWAP_F32;
  e.out = ws;
  e.ldo = m;
  e.sk_L = L;
  e.sk_kbt = kbt;
  OPCK(gemm_launch_r(&ma, &mb, m, n, k, bn, 1, 1, e, num_sms(), (cudaStream_t)stream));
  GemmEpi red;
  memset(&red, 0, sizeof(red));
  red.out = out;
  red.ldo = m;
  red.sk_L = L;
  red.sk_kbt = kbt;
  OPCK(splitk_reduce_launch(RED_F32, ws, 1, n, m, m, red, (cudaStream_t)stream));
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_op_lm_argmax(const void* W, const void* X, int32_t V, int32_t n, int32_t k, float* ws_val,
                                      int32_t* ws_idx, int32_t* tokens, void* stream) {
  if (!W || !X || !ws_val || !ws_idx || !tokens || V < 1 || n < 1 || k < 1 || k % 8) return ECOSERVE_ERR_INVALID_ARG;
  const int bn = n <= 64 ? 64 : n <= 128 ? 128 : 256;
  CUtensorMap ma, mb;
  if (make_tmap_bf16(&ma, W, V, k, 128) || make_tmap_bf16(&mb, X, n, k, bn)) return ECOSERVE_ERR_CUDA;
  const int parts = (V + 127) / 128;
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  e.mode = EPI_SWAP_ARGMAX;
  e.am_val = ws_val;
  e.am_idx = ws_idx;
  e.am_ld = parts;
  OPCK(gemm_launch(&ma, &mb, V, n, k, bn, 1, e, num_sms(), (cudaStream_t)stream));
  OPCK(argmax_reduce_launch(ws_val, ws_idx, n, parts, parts, tokens, (cudaStream_t)stream));
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_op_rmsnorm(const float* x, const int32_t* rows, const void* gamma, void* out, int32_t n,
                                    int32_t H, float eps, void* stream) {
  if (!x || !gamma || !out || n < 0 || H < 4 || H % 4) return ECOSERVE_ERR_INVALID_ARG;
  OPCK(rmsnorm_launch(x, H, rows, (const bf16*)gamma, (bf16*)out, n, H, eps, (cudaStream_t)stream));
  return ECOSERVE_OK;
}

// chunk offsets (optional) -> device, appended after the tiles: returns the device pointer or null
static int* append_offsets(int* d, size_t at, const int32_t* ctx_off_host, int n_seq, cudaStream_t st,
                           cudaError_t* err) {
  if (!ctx_off_host) return nullptr;
  *err = cudaMemcpyAsync(d + at, ctx_off_host, sizeof(int) * n_seq, cudaMemcpyHostToDevice, st);
  return d + at;
}

ecoserve_status ecoserve_op_attention_prefill(const void* q, const void* pool, int64_t num_blocks, int32_t n_heads,
                                              int32_t n_kv, int32_t head_dim, const int32_t* cu_seqlens_host,
                                              int32_t n_seq, const int32_t* block_tables, int32_t bt_ld, void* out,
                                              void* stream, const int32_t* ctx_off_host) {
  if (!q || !pool || !cu_seqlens_host || !block_tables || !out || n_seq < 1 || n_heads % n_kv || num_blocks < 1)
    return ECOSERVE_ERR_INVALID_ARG;
  std::vector<int> tiles;
  for (int s = 0; s < n_seq; ++s) {
    const int len = cu_seqlens_host[s + 1] - cu_seqlens_host[s];
    const int off = ctx_off_host ? ctx_off_host[s] : 0;
    if (len < 1 || off < 0 || (off + len + 63) / 64 > bt_ld) return ECOSERVE_ERR_INVALID_ARG;
    for (int qs = 0; qs < len; qs += 64) { tiles.push_back(s); tiles.push_back(qs); }
  }
  int* d = nullptr;
  const size_t bytes = sizeof(int) * (tiles.size() + 2 * n_seq + 1);
  OPCK(cudaMallocAsync((void**)&d, bytes, (cudaStream_t)stream));
  OPCK(cudaMemcpyAsync(d, cu_seqlens_host, sizeof(int) * (n_seq + 1), cudaMemcpyHostToDevice, (cudaStream_t)stream));
  OPCK(cudaMemcpyAsync(d + n_seq + 1, tiles.data(), sizeof(int) * tiles.size(), cudaMemcpyHostToDevice,
                       (cudaStream_t)stream));
  cudaError_t oe = cudaSuccess;
  int* d_off = append_offsets(d, n_seq + 1 + tiles.size(), ctx_off_host, n_seq, (cudaStream_t)stream, &oe);
  OPCK(oe);
  PrefillAttnArgs a;
  a.q = (const bf16*)q;
  a.k_cache = (const bf16*)pool;
  a.v_cache = (const bf16*)pool + (int64_t)n_kv * 64 * head_dim;
  a.blk_stride = 2LL * n_kv * 64 * head_dim;
  a.cu_seqlens = d;
  a.block_tables = block_tables;
  a.bt_ld = bt_ld;
  a.tiles = d + n_seq + 1;
  a.n_tiles = (int)tiles.size() / 2;
  a.out = (bf16*)out;
  a.n_heads = n_heads;
  a.n_kv = n_kv;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)head_dim));
  a.ctx_off = d_off;
  const cudaError_t e = attn_prefill_launch(a, head_dim, (cudaStream_t)stream);
  cudaFreeAsync(d, (cudaStream_t)stream);
  return e == cudaSuccess ? ECOSERVE_OK : ECOSERVE_ERR_CUDA;
}

ecoserve_status ecoserve_op_attention_prefill_tc(const void* q, const void* pool, int64_t num_blocks,
                                                 int32_t n_heads, int32_t n_kv, const int32_t* cu_seqlens_host,
                                                 int32_t n_seq, const int32_t* block_tables, int32_t bt_ld, void* out,
                                                 void* stream, const int32_t* ctx_off_host) {
  if (!q || !pool || !cu_seqlens_host || !block_tables || !out || n_seq < 1 || n_heads % n_kv || num_blocks < 1)
    return ECOSERVE_ERR_INVALID_ARG;
  std::vector<int> tiles;
  double keys = 0;  // keys attended, summed over the queries (the engine's kernel choice)
  for (int s = 0; s < n_seq; ++s) {
    const int len = cu_seqlens_host[s + 1] - cu_seqlens_host[s];
    const int off = ctx_off_host ? ctx_off_host[s] : 0;
    if (len < 1 || off < 0 || (off + len + 63) / 64 > bt_ld) return ECOSERVE_ERR_INVALID_ARG;
    for (int qs = 0; qs < len; qs += 128) { tiles.push_back(s); tiles.push_back(qs); }
    keys += (double)len * off + 0.5 * len * (len + 1.0);
  }
  const int mean_keys = (int)(keys / std::max(1, cu_seqlens_host[n_seq]));
  CUtensorMap qm, km;
  if (make_attn_tc_maps(&qm, &km, q, cu_seqlens_host[n_seq], n_heads, pool, num_blocks * 2 * n_kv * 64))
    return ECOSERVE_ERR_CUDA;
  int* d = nullptr;
  const size_t bytes = sizeof(int) * (tiles.size() + 2 * n_seq + 1);
  OPCK(cudaMallocAsync((void**)&d, bytes, (cudaStream_t)stream));
  OPCK(cudaMemcpyAsync(d, cu_seqlens_host, sizeof(int) * (n_seq + 1), cudaMemcpyHostToDevice, (cudaStream_t)stream));
  OPCK(cudaMemcpyAsync(d + n_seq + 1, tiles.data(), sizeof(int) * tiles.size(), cudaMemcpyHostToDevice,
                       (cudaStream_t)stream));
  cudaError_t oe = cudaSuccess;
  int* d_off = append_offsets(d, n_seq + 1 + tiles.size(), ctx_off_host, n_seq, (cudaStream_t)stream, &oe);
  OPCK(oe);
  const cudaError_t e = attn_prefill_tc_launch(&qm, &km, d, block_tables, bt_ld, d + n_seq + 1,
                                               (int)tiles.size() / 2, (bf16*)out, n_heads, n_kv, 0, 1,
                                               (cudaStream_t)stream, d_off, mean_keys);
  cudaFreeAsync(d, (cudaStream_t)stream);
  return e == cudaSuccess ? ECOSERVE_OK : ECOSERVE_ERR_CUDA;
}

ecoserve_status ecoserve_op_attention_decode(const void* q, const void* pool, int32_t n_heads, int32_t n_kv,
                                             int32_t head_dim, const int32_t* ctx_lens, int32_t B,
                                             const int32_t* block_tables, int32_t bt_ld, int32_t n_splits,
                                             int32_t blocks_per_split, float* workspace, void* out, void* stream, int32_t use_tma) {
  if (!q || !pool || !ctx_lens || !block_tables || !out || B < 1 || n_heads % n_kv || n_splits < 1 ||
      blocks_per_split < 1 || (n_splits > 1 && !workspace))
    return ECOSERVE_ERR_INVALID_ARG;
  DecodeAttnArgs a;
  a.q = (const bf16*)q;
  a.k_cache = (const bf16*)pool;
  a.v_cache = (const bf16*)pool + (int64_t)n_kv * 64 * head_dim;
  a.blk_stride = 2LL * n_kv * 64 * head_dim;
  a.ctx_lens = ctx_lens;
  a.block_tables = block_tables;
  a.bt_ld = bt_ld;
  a.B = B;
  a.n_heads = n_heads;
  a.n_kv = n_kv;
  a.n_splits = n_splits;
  a.blocks_per_split = blocks_per_split;
  a.part_o = workspace;
  a.part_ml = workspace ? workspace + (int64_t)B * n_heads * n_splits * head_dim : nullptr;
  a.out = (bf16*)out;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)head_dim));
  a.order = nullptr;
  a.kvmap = nullptr;
  a.layer = 0;
  a.n_layers = 1;
  CUtensorMap kvm;
  if (head_dim == 128 && use_tma) {  // the engine's TMA staging path (single-layer pool)
    const int64_t dims[2] = {128, (int64_t)1 << 30};  // rows: an upper bound, accesses stay in the pool
    const int64_t strides[1] = {256};
    const int box[2] = {64, 64};
    if (make_tmap_bf16_nd(&kvm, pool, 2, dims, strides, box)) return ECOSERVE_ERR_CUDA;
    a.kvmap = &kvm;
  }
  OPCK(attn_decode_launch(a, head_dim, (cudaStream_t)stream));
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_op_attention_decode_sk(const void* q, const void* pool, int32_t n_heads, int32_t n_kv,
                                                int32_t head_dim, const int32_t* ctx_host, int32_t B,
                                                const int32_t* block_tables, int32_t bt_ld, float* workspace,
                                                int32_t* counters, int32_t* meta, void* out, void* stream) {
  if (!q || !pool || !ctx_host || !block_tables || !out || !workspace || !counters || !meta || B < 1 ||
      n_heads % n_kv || head_dim != 128)
    return ECOSERVE_ERR_INVALID_ARG;
  // LPT order and the block prefix over it, as the engine builds them
  std::vector<int32_t> h((size_t)2 * B + 1);
  int32_t* ord = h.data();
  int32_t* skp = ord + B;
  for (int k = 0; k < B; ++k) ord[k] = k;
  std::stable_sort(ord, ord + B, [ctx_host](int x, int y) { return ctx_host[x] > ctx_host[y]; });
  int max_nb = 0, min_nb = 1 << 30;
  skp[0] = 0;
  for (int r = 0; r < B; ++r) {
    const int nb = (ctx_host[ord[r]] + 63) / 64;
    skp[r + 1] = skp[r] + nb;
    max_nb = std::max(max_nb, nb);
    min_nb = std::min(min_nb, nb);
  }
  int dev = 0, sms = 148, maxp = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = attn_decode_sk_grid(skp[B] * n_kv, max_nb, min_nb, n_heads, n_kv, head_dim, sms, &maxp, true);
  if (grid <= 0) return ECOSERVE_ERR_UNSUPPORTED;
  OPCK(cudaMemcpyAsync(meta, h.data(), sizeof(int32_t) * h.size(), cudaMemcpyHostToDevice, (cudaStream_t)stream));
  OPCK(cudaStreamSynchronize((cudaStream_t)stream));  // (h is a local)
  // ctx_lens on the device: the caller's block tables are, the lengths are only on the host
  int32_t* d_ctx = nullptr;
  OPCK(cudaMalloc(&d_ctx, sizeof(int32_t) * B));
  OPCK(cudaMemcpy(d_ctx, ctx_host, sizeof(int32_t) * B, cudaMemcpyHostToDevice));
  DecodeAttnArgs a;
  a.q = (const bf16*)q;
  a.k_cache = (const bf16*)pool;
  a.v_cache = (const bf16*)pool + (int64_t)n_kv * 64 * head_dim;
  a.blk_stride = 2LL * n_kv * 64 * head_dim;
  a.ctx_lens = d_ctx;
  a.block_tables = block_tables;
  a.bt_ld = bt_ld;
  a.B = B;
  a.n_heads = n_heads;
  a.n_kv = n_kv;
  a.n_splits = 1;
  a.blocks_per_split = max_nb;
  a.part_o = workspace;
  a.part_ml = nullptr;
  a.out = (bf16*)out;
  a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)head_dim));
  a.order = meta;
  a.layer = 0;
  a.n_layers = 1;
  a.sk_prefix = meta + B;
  a.sk_cnt = counters;
  a.sk_grid = grid;
  a.sk_maxp = maxp;
  CUtensorMap kvm;
  const int64_t dims[2] = {128, (int64_t)1 << 30};
  const int64_t strides[1] = {256};
  const int box[2] = {64, 64};
  if (make_tmap_bf16_nd(&kvm, pool, 2, dims, strides, box)) {
    cudaFree(d_ctx);
    return ECOSERVE_ERR_CUDA;
  }
  a.kvmap = &kvm;
  const cudaError_t e = attn_decode_launch(a, head_dim, (cudaStream_t)stream);
  cudaStreamSynchronize((cudaStream_t)stream);
  cudaFree(d_ctx);
  OPCK(e);
  return ECOSERVE_OK;
}

}  // extern "C"
