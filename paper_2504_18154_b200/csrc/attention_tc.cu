// Prefill causal varlen attention on the 5th-generation tensor cores (SURVEY 8(a)
// row a8; Eq. 2). One CTA = one 128-query tile of one
// sequence x one q head, head_dim 128, K/V streamed 64 tokens (= one paged-pool
// block) at a time by TMA straight out of the pool through the block table.
//
//   warp 0     TMA producer: Q tile once, then K / V blocks into a 3-stage ring
//   warp 1     TMEM owner + single-thread MMA issuer:
//                S_j = Q K_j^T      (M=128, N=64,  K=128; A, B K-major)   -> TMEM S[j%2]
//                O_j = P_j V_j      (M=128, N=128, K=64;  B = V MN-major) -> TMEM O[j%2]
//   warps 2-5  softmax: thread r owns query row r (TMEM lane r). Per block it loads
//              its S row, applies the causal mask and the exp2 online softmax,
//              writes P (bf16) as a K-major 128B-swizzled smem tile for the next
//              MMA, and folds O_{j-1} into fp32 registers with the running
//              rescale (the MMA writes each block's P V into a fresh TMEM
//              buffer, so no TMEM read-modify-write is needed).
// S and O are double buffered in TMEM (2 x 64 + 2 x 128 of 512 columns), so the
// tensor core computes S_{j+1} and O_j while the softmax warps work on block j.
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace eco {

namespace {
constexpr int TQ = 128;   // queries per tile
constexpr int TK = 64;    // keys per block (= KV block of the pool)
constexpr int HD = 128;   // head dim
constexpr int KV_STAGES = 3;
constexpr int Q_BYTES = TQ * HD * 2;          // 32 KB: 2 panels [128][64]
constexpr int K_BYTES = TK * HD * 2;          // 16 KB: 2 panels [64][64]
constexpr int V_BYTES = TK * HD * 2;          // 16 KB: 2 panels [64 keys][64 d]
constexpr int P_BYTES = TQ * TK * 2;          // 16 KB: 1 panel [128][64]
constexpr int SMEM = Q_BYTES + KV_STAGES * (K_BYTES + V_BYTES) + 2 * P_BYTES + 1024 + 512;
constexpr int S_COL = 0, O_COL = 128;         // TMEM columns: S[2] at 0 / 64, O[2] at 128 / 256

// instruction descriptor, bf16 x bf16 -> f32, A K-major, B K-major (b_mn = 0) or MN-major (1)
__host__ __device__ constexpr uint32_t idesc(int M, int N, int b_mn) {
  return umma_idesc_bf16(M, N) | ((uint32_t)b_mn << 16);
}

// smem descriptor of an MN-major operand staged with 128B swizzle: 64-element wide
// MN panels `lbo` bytes apart, 8-row K groups 1024 B apart (SBO)
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace

struct TcAttnParams {
  const int* cu_seqlens;
  const int* block_tables;
  int bt_ld;
  const int* tiles;        // [n_tiles][2] (seq, q_start), 128-query tiles
  bf16* out;               // [T][M*128]
  int n_heads, n_kv, layer, n_layers;
  float scale_log2;
};

__global__ void __launch_bounds__(192, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kvmap,
                           TcAttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sKV = sQ + Q_BYTES;                               // stage s: K at s*(K+V), V after it
  uint8_t* sP = sKV + KV_STAGES * (K_BYTES + V_BYTES);       // [2][P_BYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * P_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + KV_STAGES;
  uint64_t* s_full = kv_empty + KV_STAGES;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 2;
  uint64_t* o_full = p_empty + 2;
  uint64_t* o_empty = o_full + 2;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(o_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = blockIdx.x, h = blockIdx.y;
  const int G = p.n_heads / p.n_kv, kvh = h / G;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < KV_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 4);
      mbar_init(&p_full[s], 4);
      mbar_init(&p_empty[s], 1);
      mbar_init(&o_full[s], 1);
      mbar_init(&o_empty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&qmap);
    tma_prefetch(&kvmap);
  }
  if (warp == 1) tmem_alloc(tmem_ptr, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  pdl_trigger();
  pdl_wait();

  const int seq = p.tiles[2 * tile], q_start = p.tiles[2 * tile + 1];
  const int tok0 = p.cu_seqlens[seq];
  const int len = p.cu_seqlens[seq + 1] - tok0;
  const int n_kv = (min(q_start + TQ, len) + TK - 1) / TK;  // causal: keys < q_start + 128
  const int* bt = p.block_tables + (int64_t)seq * p.bt_ld;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, Q_BYTES);
      for (int pn = 0; pn < 2; ++pn) tma_load_3d(sQ + pn * (TQ * 128), &qmap, q_full, pn * 64, h, tok0 + q_start);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % KV_STAGES;
        if (j >= KV_STAGES) mbar_wait(&kv_empty[s], ((j / KV_STAGES) - 1) & 1);
        uint8_t* sk = sKV + s * (K_BYTES + V_BYTES);
        uint8_t* sv = sk + K_BYTES;
        // pool rows: ((block * L + layer) * 2 + kv) * Mkv * 64 + kvh * 64 + token
        const int64_t base = ((int64_t)bt[j] * p.n_layers + p.layer) * 2;
        const int krow = (int)((base * p.n_kv + kvh) * TK);
        const int vrow = (int)(((base + 1) * p.n_kv + kvh) * TK);
        mbar_arrive_expect_tx(&kv_full[s], K_BYTES + V_BYTES);
        for (int pn = 0; pn < 2; ++pn) {
          tma_load_2d(sk + pn * (TK * 128), &kvmap, &kv_full[s], pn * 64, krow);
          tma_load_2d(sv + pn * (TK * 128), &kvmap, &kv_full[s], pn * 64, vrow);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = idesc(TQ, TK, 0);
      constexpr uint32_t id_o = idesc(TQ, HD, 1);
      const uint32_t aq = smem_u32(sQ);
      auto issue_s = [&](int j) {
        const int s = j % KV_STAGES;
        mbar_wait(&kv_full[s], (j / KV_STAGES) & 1);
        tc_fence_after();
        const uint32_t ak = smem_u32(sKV + s * (K_BYTES + V_BYTES));
        const uint32_t d = tmem + S_COL + (j & 1) * TK;
#pragma unroll
        for (int pn = 0; pn < 2; ++pn) {
          const uint64_t da = umma_desc_sw128(aq + pn * (TQ * 128)), db = umma_desc_sw128(ak + pn * (TK * 128));
#pragma unroll
          for (int k = 0; k < 4; ++k) tc_mma_f16(d, da + 2 * k, db + 2 * k, id_s, (pn | k) ? 1u : 0u);
        }
        tc_commit(&s_full[j & 1]);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      if (n_kv > 0) issue_s(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) {
          if (j + 1 >= 2) mbar_wait(&s_empty[(j + 1) & 1], (((j + 1) >> 1) - 1) & 1);
          tc_fence_after();
          issue_s(j + 1);
        }
        // O_j = P_j V_j into a fresh TMEM buffer
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        if (j >= 2) mbar_wait(&o_empty[j & 1], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const int s = j % KV_STAGES;
        const uint32_t ap = smem_u32(sP + (j & 1) * P_BYTES);
        const uint32_t av = smem_u32(sKV + s * (K_BYTES + V_BYTES) + K_BYTES);
        const uint32_t d = tmem + O_COL + (j & 1) * HD;
        const uint64_t da = umma_desc_sw128(ap);
#pragma unroll
        for (int k = 0; k < TK / 16; ++k)  // 16 keys per MMA: +32 B along P rows, +2 x 1024 B along V rows
          tc_mma_f16(d, da + 2 * k, desc_mn_sw128(av + k * 2048, TK * 128), id_o, k ? 1u : 0u);
        tc_commit(&o_full[j & 1]);
        tc_commit(&kv_empty[s]);
        tc_commit(&p_empty[j & 1]);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int q = warp & 3;
    const int r = q * 32 + lane;              // query row = TMEM lane
    const int qpos = q_start + r;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    float o[HD];
#pragma unroll
    for (int i = 0; i < HD; ++i) o[i] = 0.f;
    float m_run = -INFINITY, l_run = 0.f, corr_prev = 1.f;
    auto fold_o = [&](int jb, float corr) {   // o = o * corr + O_jb
      mbar_wait(&o_full[jb & 1], (jb >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(lane_base + O_COL + (jb & 1) * HD + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) o[c0 + i] = o[c0 + i] * corr + __uint_as_float(v[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[jb & 1]);
    };
    for (int j = 0; j < n_kv; ++j) {
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      float sv[TK];
#pragma unroll
      for (int c0 = 0; c0 < TK; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(lane_base + S_COL + (j & 1) * TK + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c0 + i] = __uint_as_float(v[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[j & 1]);
      const bool diag = j * TK + TK - 1 > q_start;
      float mx = m_run;
#pragma unroll
      for (int c = 0; c < TK; ++c) {
        float x = sv[c] * p.scale_log2;
        if (diag && j * TK + c > qpos) x = -INFINITY;
        sv[c] = x;
        mx = fmaxf(mx, x);
      }
      const float corr = (m_run == -INFINITY) ? 0.f : exp2f(m_run - mx);
      float rs = 0.f;
      uint32_t pk[TK / 2];
#pragma unroll
      for (int c = 0; c < TK; c += 2) {
        const float a = (mx == -INFINITY) ? 0.f : exp2f(sv[c] - mx);
        const float b = (mx == -INFINITY) ? 0.f : exp2f(sv[c + 1] - mx);
        rs += a + b;
        pk[c / 2] = pack_bf16x2(a, b);
      }
      l_run = l_run * corr + rs;
      m_run = mx;
      // P row -> K-major 128B-swizzled smem tile (row r: 128 B, 16-byte chunk c at c ^ (r % 8))
      if (j >= 2) mbar_wait(&p_empty[j & 1], ((j >> 1) - 1) & 1);
      uint8_t* prow = sP + (j & 1) * P_BYTES + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) << 4)) =
            make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j & 1]);
      if (j > 0) fold_o(j - 1, corr_prev);
      corr_prev = corr;
    }
    if (n_kv > 0) fold_o(n_kv - 1, corr_prev);
    if (qpos < len) {
      const float inv = 1.f / l_run;
      bf16* dst = p.out + (int64_t)(tok0 + qpos) * p.n_heads * HD + h * HD;
#pragma unroll
      for (int i = 0; i < HD; i += 8)
        *reinterpret_cast<uint4*>(dst + i) =
            make_uint4(pack_bf16x2(o[i] * inv, o[i + 1] * inv), pack_bf16x2(o[i + 2] * inv, o[i + 3] * inv),
                       pack_bf16x2(o[i + 4] * inv, o[i + 5] * inv), pack_bf16x2(o[i + 6] * inv, o[i + 7] * inv));
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem, 512);
  }
}

// q: [q_rows][n_heads][128] bf16 (TMA 3D map over the whole buffer); pool: the instance's
// block-major pool (2D map over rows of 128 elements).
int make_attn_tc_maps(CUtensorMap* qmap, CUtensorMap* kvmap, const void* q, int64_t q_rows, int n_heads,
                      const void* pool, int64_t pool_rows) {
  const int64_t qd[3] = {HD, n_heads, q_rows};
  const int64_t qs[2] = {HD * 2, (int64_t)n_heads * HD * 2};
  const int qb[3] = {64, 1, TQ};
  if (make_tmap_bf16_nd(qmap, q, 3, qd, qs, qb)) return -1;
  const int64_t kd[2] = {HD, pool_rows};
  const int64_t ks[1] = {HD * 2};
  const int kb[2] = {64, TK};
  return make_tmap_bf16_nd(kvmap, pool, 2, kd, ks, kb);
}

cudaError_t attn_prefill_tc_launch(const CUtensorMap* qmap, const CUtensorMap* kvmap, const int* cu_seqlens,
                                   const int* block_tables, int bt_ld, const int* tiles, int n_tiles, bf16* out,
                                   int n_heads, int n_kv, int layer, int n_layers, cudaStream_t s) {
  cudaError_t e = ensure_smem(attn_prefill_tc_kernel, SMEM);
  if (e != cudaSuccess) return e;
  if (n_tiles == 0) return cudaSuccess;
  TcAttnParams p;
  p.cu_seqlens = cu_seqlens;
  p.block_tables = block_tables;
  p.bt_ld = bt_ld;
  p.tiles = tiles;
  p.out = out;
  p.n_heads = n_heads;
  p.n_kv = n_kv;
  p.layer = layer;
  p.n_layers = n_layers;
  p.scale_log2 = (float)(1.4426950408889634 / sqrt((double)HD));
  return launch_k(attn_prefill_tc_kernel, dim3(n_tiles, n_heads), dim3(192), SMEM, s, *qmap, *kvmap, p);
}

}  // namespace eco
