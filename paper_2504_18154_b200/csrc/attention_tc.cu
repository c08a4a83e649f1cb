// Prefill causal varlen attention on the 5th-generation tensor cores (SURVEY 8(a)
// row a8; Eq. 2). One CTA = one 128-query tile of one sequence x
// HP (= 2 when the GQA group is even) q heads of the same kv head, head_dim 128; K/V
// stream 64 tokens (= one paged-pool block) at a time by TMA straight out of the pool
// through the block table (4-stage ring), shared by the HP heads.
//
//   warp 0          TMA producer: the HP Q tiles once, then K / V blocks
//   warp 1          TMEM owner + single-thread MMA issuer, per block j and head e:
//                     S_e[j%2] = Q_e K_j^T     (M=128, N=64, K=128; A, B K-major, smem)
//                     O_e     += P_e[j%2] V_j  (M=128, N=128, K=64; A = P from TMEM,
//                                               B = V MN-major from smem)
//                   issue order per block: PV(j, e) then S(j+2, e) -- S is double
//                   buffered, so the scores of the next block are always ready when
//                   the softmax warps finish the current one.
//   warps 2..       4 softmax warps per head; thread r owns query row r (TMEM lane). Per
//                   block: load the S row, causal mask, exp2 online softmax with a lazily
//                   updated running max (O in TMEM is rescaled only when the max grows by
//                   more than 2^8 -- the stale max keeps P <= 256, exact after the final
//                   1/l), P (bf16 pairs) written back over its own S columns (tcgen05.st)
//                   as the A operand of the PV MMA.
// TMEM per head e: S[0] / S[1] at columns e*256 + {0, 64}, O at e*256 + [128, 256).
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace eco {

namespace {
constexpr int TQ = 128;   // queries per tile
constexpr int TK = 64;    // keys per block (= KV block of the pool)
constexpr int HD = 128;   // head dim
constexpr int KV_STAGES = 4;
constexpr int Q_BYTES = TQ * HD * 2;          // 32 KB per head: 2 panels [128][64]
constexpr int K_BYTES = TK * HD * 2;          // 16 KB: 2 panels [64][64]
constexpr int V_BYTES = TK * HD * 2;          // 16 KB: 2 panels [64 keys][64 d]
constexpr float RESCALE_LOG2 = 8.f;           // rescale O when the row max grows by > 2^8

template <int HP>
struct AttnCfg {
  static constexpr int THREADS = 64 + 128 * HP;
  static constexpr int SMEM = HP * Q_BYTES + KV_STAGES * (K_BYTES + V_BYTES) + 1024 + 512;
  static constexpr int TMEM_COLS = HP == 2 ? 512 : 256;
};

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

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ float fast_ex2(float x) {  // MUFU.EX2, flush-to-zero; 2^-inf = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA pipe (Cody-Waite: x = n + f, n = round(x) via the 1.5 * 2^23 magic
// addend, f in [-0.5, 0.5]; degree-3 fit of 2^f, max relative error 7.5e-5 -- below the
// bf16 rounding P gets anyway). Moves part of the softmax exponentials off the MUFU
// (16 / clk / SM, tools/umma_probe.cu). x >= -126 keeps the result a non-negative float
// (masked -inf scores give ~1e-38).
__device__ __forceinline__ float poly_ex2(float x) {
  x = fmaxf(x, -126.f);
  const float xr = __fadd_rn(x, 12582912.f);
  const float f = x - __fsub_rn(xr, 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05517146f, f, 0.24261115f), f, 0.69326103f), f, 0.99992806f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(xr) << 23));
}
// O[tmem] (+)= A[tmem] * B[smem desc]: A (M x 16 bf16 per step, K-major) read from TMEM,
// 16 bf16 = 8 columns per K step
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
}  // namespace

struct TcAttnParams {
  const int* cu_seqlens;
  const int* block_tables;
  int bt_ld;
  const int* tiles;        // [n_tiles][2] (seq, q_start), 128-query tiles
  bf16* out;               // [T][M*128]
  int n_heads, n_kv, layer, n_layers;
  float scale_log2;
  int pv_wait;             // experiment switch: wait for PV(j) before S(j+2) reuses its buffer
  const int* ctx_off;      // optional [n_seq]: cached tokens before this chunk (chunked prefill)
  long long* trace;        // timing probe: [20][64] clock64 stamps of CTA (trace_tile, 0), or null
  int trace_tile;
};

template <int HP>
__global__ void __launch_bounds__(AttnCfg<HP>::THREADS, 1)
    attn_prefill_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kvmap,
                           TcAttnParams p) {
  using C = AttnCfg<HP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                                          // [HP][Q_BYTES]
  uint8_t* sKV = sQ + HP * Q_BYTES;                          // stage s: K at s*(K+V), V after it
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + KV_STAGES * (K_BYTES + V_BYTES));
  uint64_t* q_full = bars;
  uint64_t* kv_full = q_full + 1;
  uint64_t* kv_empty = kv_full + KV_STAGES;
  uint64_t* s_full = kv_empty + KV_STAGES;   // [HP][2]
  uint64_t* p_full = s_full + 2 * HP;        // [HP][2]
  // o_done[e][b]: PV(j, e) complete for blocks j = b (mod 2). Two barriers alternating by
  // block parity: a consumer lagging by several blocks can then never mistake a later
  // phase for the one it waits on (PV(j + 2) needs P_{j+2}, which it has not produced)
  uint64_t* o_done = p_full + 2 * HP;        // [HP][2]
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(o_done + 2 * HP);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = blockIdx.x, h0 = blockIdx.y * HP;
  const int G = p.n_heads / p.n_kv, kvh = h0 / G;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < KV_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int e = 0; e < HP; ++e) {
      for (int b = 0; b < 2; ++b) {
        mbar_init(&o_done[2 * e + b], 1);
        mbar_init(&s_full[2 * e + b], 1);
        mbar_init(&p_full[2 * e + b], 4);
      }
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&qmap);
    tma_prefetch(&kvmap);
  }
  if (warp == 1) tmem_alloc(tmem_ptr, C::TMEM_COLS);
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  pdl_trigger();
  pdl_wait();

  const int seq = p.tiles[2 * tile], q_start = p.tiles[2 * tile + 1];
  const int tok0 = p.cu_seqlens[seq];
  const int len = p.cu_seqlens[seq + 1] - tok0;
  const int off = p.ctx_off ? p.ctx_off[seq] : 0;  // chunked prefill: cached tokens before the chunk
  const int n_kv = (off + min(q_start + TQ, len) + TK - 1) / TK;  // causal: keys < off + q_start + 128
  const int* bt = p.block_tables + (int64_t)seq * p.bt_ld;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, HP * Q_BYTES);
      for (int e = 0; e < HP; ++e)
        for (int pn = 0; pn < 2; ++pn)
          tma_load_3d(sQ + e * Q_BYTES + pn * (TQ * 128), &qmap, q_full, pn * 64, h0 + e, tok0 + q_start);
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
      // S_e[j % 2] = Q_e K_j^T (the caller has waited for K_j)
      auto mma_s = [&](int j, int e) {
        const uint32_t ak = smem_u32(sKV + (j % KV_STAGES) * (K_BYTES + V_BYTES));
        const uint32_t aq = smem_u32(sQ + e * Q_BYTES);
        const uint32_t d = tmem + e * 256 + (j & 1) * 64;
#pragma unroll
        for (int pn = 0; pn < 2; ++pn) {
          const uint64_t da = umma_desc_sw128(aq + pn * (TQ * 128)), db = umma_desc_sw128(ak + pn * (TK * 128));
#pragma unroll
          for (int k = 0; k < 4; ++k) tc_mma_f16(d, da + 2 * k, db + 2 * k, id_s, (pn | k) ? 1u : 0u);
        }
        tc_commit(&s_full[2 * e + (j & 1)]);
      };
      auto wait_k = [&](int j) {
        mbar_wait(&kv_full[j % KV_STAGES], (j / KV_STAGES) & 1);
        tc_fence_after();
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      for (int j = 0; j < 2 && j < n_kv; ++j) {
        wait_k(j);
        for (int e = 0; e < HP; ++e) mma_s(j, e);
      }
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % KV_STAGES;
        const uint32_t av = smem_u32(sKV + s * (K_BYTES + V_BYTES) + K_BYTES);
        const bool next = j + 2 < n_kv;
        if (next) wait_k(j + 2);
#pragma unroll
        for (int e = 0; e < HP; ++e) {
          mbar_wait(&p_full[2 * e + (j & 1)], (j >> 1) & 1);
          tc_fence_after();
          const uint32_t ap = tmem + e * 256 + (j & 1) * 64;  // P_j over S_j's first 32 columns
          const uint32_t d = tmem + e * 256 + 128;
#pragma unroll
          for (int k = 0; k < TK / 16; ++k)  // 16 keys per MMA: +8 TMEM columns of P, +2 x 1024 B along V rows
            tc_mma_ts(d, ap + 8 * k, desc_mn_sw128(av + k * 2048, TK * 128), id_o, (j > 0 || k > 0) ? 1u : 0u);
          tc_commit(&o_done[2 * e + (j & 1)]);
          if (e == HP - 1) tc_commit(&kv_empty[s]);
          // S(j+2) overwrites buffer j % 2, which PV(j) reads P_j from: wait for PV(j)
          if (next) {
            if (p.pv_wait) {
              mbar_wait(&o_done[2 * e + (j & 1)], (j >> 1) & 1);
              tc_fence_after();
            }
            mma_s(j + 2, e);
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int e = (warp - 2) >> 2;
    const int q = warp & 3;                   // TMEM lane quarter accessible to this warp
    const int r = q * 32 + lane;              // query row = TMEM lane
    const int qpos = off + q_start + r;       // position of this query row
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + e * 256;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const uint32_t sb = lane_base + (j & 1) * 64;
      mbar_wait(&s_full[2 * e + (j & 1)], (j >> 1) & 1);
      tc_fence_after();
      float sv[TK];
      {
        uint32_t v0[32], v1[32];
        tmem_ld32(sb, v0);
        tmem_ld32(sb + 32, v1);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          sv[i] = __uint_as_float(v0[i]);
          sv[32 + i] = __uint_as_float(v1[i]);
        }
      }
      // causal mask on the diagonal blocks; the row max in raw score units (scale > 0),
      // as an 8-way tree to keep the dependent chain short
      if (j * TK + TK - 1 > off + q_start) {
#pragma unroll
        for (int c = 0; c < TK; ++c)
          if (j * TK + c > qpos) sv[c] = -INFINITY;
      }
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = sv[i];
#pragma unroll
      for (int c = 8; c < TK; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], sv[c]);
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * p.scale_log2;
      const float m_new = fmaxf(m_run, mx);
      if (j == 0) {
        m_run = m_new;
      } else {
        const bool need = m_new > m_run + RESCALE_LOG2;
        if (__any_sync(0xffffffffu, need)) {
          // O (TMEM) *= exp2(m_run - m_new) for the rows whose max grew past the threshold;
          // PV_{j-1} must have landed, PV_j is not issued before this warp's P_j arrives
          const float corr = need ? exp2f(m_run - m_new) : 1.f;
          if (need) m_run = m_new;
          l_run *= corr;
          mbar_wait(&o_done[2 * e + ((j - 1) & 1)], ((j - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c0 = 0; c0 < HD; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(lane_base + 128 + c0, v);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st32(lane_base + 128 + c0, v);
          }
        }
      }
      // P = 2^(s * scale - m_run); key 0 is never masked, so m_run is finite for every row
      float rs8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rs8[i] = 0.f;
      uint32_t pk[TK / 2];
      const float neg_m = -m_run;
#pragma unroll
      for (int c = 0; c < TK; c += 2) {
        const float a = fast_ex2(fmaf(sv[c], p.scale_log2, neg_m));
        const float b = fast_ex2(fmaf(sv[c + 1], p.scale_log2, neg_m));
        rs8[(c >> 1) & 7] += a + b;
        pk[c / 2] = pack_bf16x2(a, b);
      }
      l_run += ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
      // P (bf16 pairs along the keys) over the first 32 columns of this S buffer
      tmem_st32(sb, pk);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * e + (j & 1)]);
    }
    if (n_kv > 0) {
      mbar_wait(&o_done[2 * e + ((n_kv - 1) & 1)], ((n_kv - 1) >> 1) & 1);
      tc_fence_after();
    }
    // tcgen05.ld is warp-collective: every lane loads, rows past the sequence do not store
    const float inv = 1.f / l_run;
    const int lrow = q_start + r;             // row of the chunk
    bf16* dst = p.out + (int64_t)(tok0 + lrow) * p.n_heads * HD + (h0 + e) * HD;
#pragma unroll
    for (int c0 = 0; c0 < HD; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(lane_base + 128 + c0, v);
      tc_wait_ld();
      if (lrow < len) {
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(dst + c0 + i) = make_uint4(
              pack_bf16x2(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv),
              pack_bf16x2(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv),
              pack_bf16x2(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv),
              pack_bf16x2(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv));
      }
    }
  }
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------------------
// 128-key variant: one q head per CTA, K / V consumed 128 keys (two pool blocks) per step.
// tools/umma_probe.cu measured why this pays: a tcgen05.mma of N = 64 occupies the pipe
// ~48 cycles against 32 for its work (N >= 128 runs at the 4096 MAC/cycle rate), and a
// commit + wait round trip on the issuer's own MMAs costs ~350 idle cycles. Here every
// MMA has N = 128 (S = Q K^T over 128 keys; O += P V with 128 head dims), and the issuer
// never waits on its own MMAs: S and P are both double buffered in TMEM and disjoint,
//   TMEM: S[0] [0,128)  S[1] [128,256)  O [256,384)  P[0] [384,448)  P[1] [448,512)
// so S(j+2) overwrites only scores the softmax has finished reading, and the softmax
// writes P(j) into P[j%2] only after PV(j-2) has consumed it.
//   warp 0   TMA producer: Q (2 panels), then per key tile j the K tile (both 64-key
//            pool blocks into one 32 KB [128 keys][128 dims] stage, so the S MMA's B
//            operand is one descriptor) and the two V blocks (16 KB stages: a PV MMA
//            covers 16 keys, never straddling blocks)
//   warp 1   TMEM owner + MMA issuer: S(0), S(1); per j: PV(j), S(j+2)
//   warps 2-5 softmax, thread r = query row r (TMEM lane)
// A missing second block of the last tile (odd block count) is loaded from the
// sequence's first block: finite values under keys the causal mask removes.
namespace t128 {
constexpr int TKT = 128;                       // keys per step
constexpr int K_STAGES = 3;                    // 32 KB K tiles
constexpr int V_STAGES = 6;                    // 16 KB V blocks (3 tiles)
constexpr int KT_BYTES = TKT * HD * 2;         // 32 KB: 2 panels [128 keys][64 dims]
constexpr int SMEM = Q_BYTES + K_STAGES * KT_BYTES + V_STAGES * V_BYTES + 1024 + 512;
constexpr int THREADS = 192;                   // producer, issuer, 4 softmax warps
constexpr uint32_t S_COL = 0, O_COL = 256, P_COL = 384;
}  // namespace t128

template <int POLY>
__global__ void __launch_bounds__(t128::THREADS, 1)
    attn_prefill_t128_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kvmap,
                             TcAttnParams p) {
  using namespace t128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                              // [Q_BYTES]
  uint8_t* sK = sQ + Q_BYTES;                    // [K_STAGES][KT_BYTES]
  uint8_t* sV = sK + K_STAGES * KT_BYTES;        // [V_STAGES][V_BYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + V_STAGES * V_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + K_STAGES;
  uint64_t* v_full = k_empty + K_STAGES;
  uint64_t* v_empty = v_full + V_STAGES;
  uint64_t* s_full = v_empty + V_STAGES;   // [2] by buffer
  uint64_t* p_full = s_full + 2;           // [2]
  uint64_t* o_done = p_full + 2;           // [2] PV(j) complete, by j parity
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tile = blockIdx.x, h = blockIdx.y;
  long long* const tr = (p.trace && tile == p.trace_tile && blockIdx.y == 0) ? p.trace : nullptr;
  const int kvh = h / (p.n_heads / p.n_kv);

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < K_STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < V_STAGES; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 4);
      mbar_init(&o_done[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&qmap);
    tma_prefetch(&kvmap);
  }
  if (warp == 1) tmem_alloc(tmem_ptr, 512);
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  pdl_trigger();
  pdl_wait();

  const int seq = p.tiles[2 * tile], q_start = p.tiles[2 * tile + 1];
  const int tok0 = p.cu_seqlens[seq];
  const int len = p.cu_seqlens[seq + 1] - tok0;
  const int off = p.ctx_off ? p.ctx_off[seq] : 0;  // chunked prefill: cached tokens before the chunk
  const int n_keys = off + min(q_start + TQ, len);  // causal: keys < off + q_start + 128
  const int n_blk = (n_keys + TK - 1) / TK;
  const int n_t = (n_keys + TKT - 1) / TKT;
  const int* bt = p.block_tables + (int64_t)seq * p.bt_ld;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, Q_BYTES);
      for (int pn = 0; pn < 2; ++pn) tma_load_3d(sQ + pn * (TQ * 128), &qmap, q_full, pn * 64, h, tok0 + q_start);
      // pool rows: ((block * L + layer) * 2 + kv) * Mkv * 64 + kvh * 64 + token
      auto row = [&](int b, int kv) {
        const int blk = bt[b < n_blk ? b : 0];
        return (int)(((((int64_t)blk * p.n_layers + p.layer) * 2 + kv) * p.n_kv + kvh) * TK);
      };
      for (int j = 0; j < n_t; ++j) {
        const int ks = j % K_STAGES;
        if (j >= K_STAGES) mbar_wait(&k_empty[ks], ((j / K_STAGES) - 1) & 1);
        uint8_t* sk = sK + ks * KT_BYTES;
        mbar_arrive_expect_tx(&k_full[ks], KT_BYTES);
        for (int hb = 0; hb < 2; ++hb) {
          const int kr = row(2 * j + hb, 0);
          for (int pn = 0; pn < 2; ++pn)
            tma_load_2d(sk + pn * (TKT * 128) + hb * (TK * 128), &kvmap, &k_full[ks], pn * 64, kr);
        }
        for (int hb = 0; hb < 2; ++hb) {
          const int b = 2 * j + hb, vs = b % V_STAGES;
          if (b >= V_STAGES) mbar_wait(&v_empty[vs], ((b / V_STAGES) - 1) & 1);
          uint8_t* sv = sV + vs * V_BYTES;
          const int vr = row(b, 1);
          mbar_arrive_expect_tx(&v_full[vs], V_BYTES);
          for (int pn = 0; pn < 2; ++pn) tma_load_2d(sv + pn * (TK * 128), &kvmap, &v_full[vs], pn * 64, vr);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = idesc(TQ, TKT, 0);
      constexpr uint32_t id_o = idesc(TQ, HD, 1);
      const uint32_t aq = smem_u32(sQ);
      auto mma_s = [&](int j) {  // S[j%2] = Q K_j^T
        const int ks = j % K_STAGES;
        mbar_wait(&k_full[ks], (j / K_STAGES) & 1);
        tc_fence_after();
        const uint32_t ak = smem_u32(sK + ks * KT_BYTES);
        const uint32_t d = tmem + S_COL + (j & 1) * 128;
#pragma unroll
        for (int pn = 0; pn < 2; ++pn) {
          const uint64_t da = umma_desc_sw128(aq + pn * (TQ * 128)), db = umma_desc_sw128(ak + pn * (TKT * 128));
#pragma unroll
          for (int k = 0; k < 4; ++k) tc_mma_f16(d, da + 2 * k, db + 2 * k, id_s, (pn | k) ? 1u : 0u);
        }
        tc_commit(&s_full[j & 1]);
        tc_commit(&k_empty[ks]);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      mma_s(0);
      if (n_t > 1) mma_s(1);
      for (int j = 0; j < n_t; ++j) {
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        tc_fence_after();
        if (tr && j < 64) tr[16 * 64 + j] = clock64();   // row 16: P_j seen by the issuer
        const uint32_t ap = tmem + P_COL + (j & 1) * 64;
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          const int b = 2 * j + hb, vs = b % V_STAGES;
          mbar_wait(&v_full[vs], (b / V_STAGES) & 1);
          tc_fence_after();
          const uint32_t av = smem_u32(sV + vs * V_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k)  // 16 keys per MMA: +8 TMEM columns of P, +2 x 1024 B along V rows
            tc_mma_ts(tmem + O_COL, ap + 8 * (4 * hb + k), desc_mn_sw128(av + k * 2048, TK * 128), id_o,
                      (j > 0 || hb > 0 || k > 0) ? 1u : 0u);
          tc_commit(&v_empty[vs]);
        }
        tc_commit(&o_done[j & 1]);
        if (j + 2 < n_t) {
          mma_s(j + 2);
          if (tr && j < 64) tr[18 * 64 + j] = clock64();   // row 18: S(j+2) issued
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int q = warp & 3;                   // TMEM lane quarter accessible to this warp
    const int r = q * 32 + lane;              // query row = TMEM lane
    const int qpos = off + q_start + r;       // position of this query row
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n_t; ++j) {
      const uint32_t sb = lane_base + S_COL + (j & 1) * 128;
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      const bool trw = tr && lane == 0 && j < 64;
      if (trw) tr[(8 + warp - 2) * 64 + j] = clock64();   // rows 8..11: S_j seen by softmax warp
      float sv[TKT];
#pragma unroll
      for (int c0 = 0; c0 < TKT; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(sb + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c0 + i] = __uint_as_float(v[i]);
      }
      // causal mask on the diagonal tiles; the row max in raw score units (scale > 0)
      if (j * TKT + TKT - 1 > off + q_start) {
#pragma unroll
        for (int c = 0; c < TKT; ++c)
          if (j * TKT + c > qpos) sv[c] = -INFINITY;
      }
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = sv[i];
#pragma unroll
      for (int c = 8; c < TKT; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], sv[c]);
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * p.scale_log2;
      const float m_new = fmaxf(m_run, mx);
      if (j == 0) {
        m_run = m_new;
      } else {
        const bool need = m_new > m_run + RESCALE_LOG2;
        if (__any_sync(0xffffffffu, need)) {
          // O (TMEM) *= exp2(m_run - m_new) for the rows whose max grew past the threshold;
          // PV(j-1) must have landed, PV(j) is not issued before this warp's P_j arrives
          const float corr = need ? exp2f(m_run - m_new) : 1.f;
          if (need) m_run = m_new;
          l_run *= corr;
          mbar_wait(&o_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c0 = 0; c0 < HD; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(lane_base + O_COL + c0, v);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st32(lane_base + O_COL + c0, v);
          }
        }
      }
      // P = 2^(s * scale - m_run); key 0 is never masked, so m_run is finite for every row
      float rs8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rs8[i] = 0.f;
      const float neg_m = -m_run;
      // P[j%2] was last read by PV(j-2): wait for it before overwriting (long complete)
      if (j >= 2) {
        mbar_wait(&o_done[j & 1], ((j - 2) >> 1) & 1);
        tc_fence_after();
      }
#pragma unroll
      for (int h32 = 0; h32 < 2; ++h32) {  // 64 keys -> 32 columns of bf16 pairs per store
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const int cc = h32 * 64 + c;
          const bool poly = ((c >> 1) & 7) < POLY;
          const float xa = fmaf(sv[cc], p.scale_log2, neg_m), xb = fmaf(sv[cc + 1], p.scale_log2, neg_m);
          const float a = poly ? poly_ex2(xa) : fast_ex2(xa);
          const float b = poly ? poly_ex2(xb) : fast_ex2(xb);
          rs8[(c >> 1) & 7] += a + b;
          pk[c / 2] = pack_bf16x2(a, b);
        }
        tmem_st32(lane_base + P_COL + (j & 1) * 64 + h32 * 32, pk);
      }
      l_run += ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
      tc_wait_st();
      if (trw) tr[(warp - 2) * 64 + j] = clock64();   // rows 0..3: P_j stored by softmax warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[j & 1]);
    }
    if (n_t > 0) {
      mbar_wait(&o_done[(n_t - 1) & 1], ((n_t - 1) >> 1) & 1);
      tc_fence_after();
    }
    const float inv = 1.f / l_run;
    const int lrow = q_start + r;             // row of the chunk
    bf16* dst = p.out + (int64_t)(tok0 + lrow) * p.n_heads * HD + h * HD;
#pragma unroll
    for (int c0 = 0; c0 < HD; c0 += 32) {
      uint32_t v[32];
      tmem_ld32(lane_base + O_COL + c0, v);
      tc_wait_ld();
      if (lrow < len) {
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(dst + c0 + i) = make_uint4(
              pack_bf16x2(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv),
              pack_bf16x2(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv),
              pack_bf16x2(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv),
              pack_bf16x2(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv));
      }
    }
  }
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
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

static long long* g_trace = nullptr;
static int g_trace_tile = 0;
void attn_tc_set_trace(long long* trace, int trace_tile) {
  g_trace = trace;
  g_trace_tile = trace_tile;
}

cudaError_t attn_prefill_tc_launch(const CUtensorMap* qmap, const CUtensorMap* kvmap, const int* cu_seqlens,
                                   const int* block_tables, int bt_ld, const int* tiles, int n_tiles, bf16* out,
                                   int n_heads, int n_kv, int layer, int n_layers, cudaStream_t s,
                                   const int* ctx_off, int mean_keys) {
  if (n_kv < 1 || n_heads % n_kv) return cudaErrorInvalidValue;
  // ECOSERVE_ATTN_T128 = 0 / 1 / 2 forces the choice; unset: the 128-key kernel when the
  // batch's queries attend >= 2048 keys on average (prompts of ~4k tokens and more). Measured
  // (profiles/r02_attn_prefill_t128_ab.log): 1 x 8k 616 vs 702 us, 4 x 2k equal (mean 1024
  // keys), 8 x U{512..2048} 176.6 vs 170.0 us (mean ~720 keys), 16 x 512 113.8 vs 92.2 us.
  static const int t128_env = [] {
    const char* ev = getenv("ECOSERVE_ATTN_T128");
    return ev ? atoi(ev) : -1;
  }();
  const int t128_mode = t128_env >= 0 ? t128_env : (mean_keys >= 2048 ? 1 : 0);
  if (t128_mode) {  // 128-key kernel; 2 = with the poly-exp2 offload
    auto k = t128_mode == 2 ? attn_prefill_t128_kernel<1> : attn_prefill_t128_kernel<0>;
    cudaError_t e = ensure_smem(k, t128::SMEM);
    if (e != cudaSuccess || n_tiles == 0) return e;
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
    p.ctx_off = ctx_off;
    p.pv_wait = 0;
    p.trace = g_trace;
    p.trace_tile = g_trace_tile;
    return launch_k(k, dim3(n_tiles, n_heads), dim3(t128::THREADS), t128::SMEM, s, *qmap, *kvmap, p);
  }
  const bool pair = (n_heads / n_kv) % 2 == 0;  // two q heads of one kv head per CTA
  cudaError_t e = pair ? ensure_smem(attn_prefill_tc_kernel<2>, AttnCfg<2>::SMEM)
                       : ensure_smem(attn_prefill_tc_kernel<1>, AttnCfg<1>::SMEM);
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
  p.ctx_off = ctx_off;
  p.trace = nullptr;
  p.trace_tile = 0;
  {
    const char* ev = getenv("ECOSERVE_ATTN_PVWAIT");
    p.pv_wait = (ev && ev[0] == '0') ? 0 : 1;
  }
  if (pair)
    return launch_k(attn_prefill_tc_kernel<2>, dim3(n_tiles, n_heads / 2), dim3(AttnCfg<2>::THREADS),
                    AttnCfg<2>::SMEM, s, *qmap, *kvmap, p);
  return launch_k(attn_prefill_tc_kernel<1>, dim3(n_tiles, n_heads), dim3(AttnCfg<1>::THREADS), AttnCfg<1>::SMEM, s,
                  *qmap, *kvmap, p);
}

}  // namespace eco
