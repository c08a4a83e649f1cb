// Attention over the paged KV pool (Eq. 2; Table 2 rows
// "Attention QK^T" / "(QK^T)V"; PagedAttention P:824).
//
// * Prefill: causal varlen flash attention. One CTA = one
//   64-query tile of one sequence x one q head; 4 warps x 16 query rows; K/V
//   streamed one 64-token pool block at a time (cp.async double buffer, XOR
//   swizzled smem), QK^T and PV on mma.sync m16n8k16 (bf16 -> f32), online
//   softmax in the exp2 domain; only the diagonal tile is masked.
// * Decode (a14): split-K over the context. One CTA = (sequence, kv head,
//   split); the G = M/Mkv q heads sharing the kv head are packed into the 16
//   MMA rows so every K/V byte read from HBM feeds G heads (GQA). Each of the
//   4 warps owns 16 of the 64 tokens of every block; per-warp online softmax,
//   then a fixed-order combine across warps and (if split) across splits.
//
// The pool must be zero-initialised at allocation (slots beyond a sequence's
// length are read and masked; masked V rows must be finite).
#include <math.h>
#include <string.h>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace eco {

// 16-byte chunk index of (row r, chunk c) in a swizzled [rows][D] bf16 tile.
template <int D>
__device__ __forceinline__ int swz(int r, int c) {
  constexpr int CPR = D / 8;
  if constexpr (CPR >= 8)
    return r * CPR + (c ^ (r & 7));
  else
    return r * CPR + (c ^ ((r >> 1) & 3));
}

// Load a [64][D] bf16 tile (64 rows contiguous in global) into swizzled smem.
template <int D, int NT>
__device__ __forceinline__ void load_tile64(bf16* smem, const bf16* g, int tid) {
  constexpr int CPR = D / 8;
  const uint32_t base = smem_u32(smem);
#pragma unroll
  for (int i = tid; i < 64 * CPR; i += NT) {
    const int r = i / CPR, c = i % CPR;
    cp_async16(base + swz<D>(r, c) * 16, g + (int64_t)r * D + c * 8);
  }
}

// ------------------------------------------------------------------ prefill
template <int D>
__global__ void __launch_bounds__(128) attn_prefill_kernel(PrefillAttnArgs a) {
  constexpr int CPR = D / 8;
  constexpr int NK = D / 16;  // k16 steps over the head dim
  constexpr int ND = D / 8;   // n8 tiles over the head dim
  extern __shared__ __align__(128) uint8_t sm[];
  bf16* sQ = reinterpret_cast<bf16*>(sm);
  bf16* sK = sQ + 64 * D;  // [2][64][D]
  bf16* sV = sK + 2 * 64 * D;
  pdl_trigger();
  pdl_wait();

  const int tile = blockIdx.x, h = blockIdx.y;
  const int seq = a.tiles[2 * tile], q_start = a.tiles[2 * tile + 1];
  const int tok0 = a.cu_seqlens[seq];
  const int len = a.cu_seqlens[seq + 1] - tok0;
  const int off = a.ctx_off ? a.ctx_off[seq] : 0;  // chunked prefill: cached tokens before the chunk
  const int kvh = h / (a.n_heads / a.n_kv);
  const int* bt = a.block_tables + (int64_t)seq * a.bt_ld;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;

  // Q tile (rows past the sequence end are clamped to its last row, results discarded)
  {
    const uint32_t base = smem_u32(sQ);
    for (int i = tid; i < 64 * CPR; i += 128) {
      const int r = i / CPR, c = i % CPR;
      const int qrow = min(q_start + r, len - 1);
      cp_async16(base + swz<D>(r, c) * 16, a.q + ((int64_t)(tok0 + qrow) * a.n_heads + h) * D + c * 8);
    }
  }
  const int n_kv_tiles = (off + min(q_start + 64, len) + 63) / 64;
  auto kv_ptr = [&](const bf16* cache, int j) {
    return cache + (int64_t)bt[j] * a.blk_stride + (int64_t)kvh * 64 * D;
  };
  load_tile64<D, 128>(sK, kv_ptr(a.k_cache, 0), tid);
  load_tile64<D, 128>(sV, kv_ptr(a.v_cache, 0), tid);
  cp_async_commit();

  uint32_t qf[NK][4];
  float o[ND][4];
#pragma unroll
  for (int i = 0; i < ND; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const int g = lane >> 2, t4 = lane & 3;
  const int qpos0 = off + q_start + warp * 16 + g;  // positions of rows g and g+8 of this warp

  for (int j = 0; j < n_kv_tiles; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_kv_tiles) {
      load_tile64<D, 128>(sK + (buf ^ 1) * 64 * D, kv_ptr(a.k_cache, j + 1), tid);
      load_tile64<D, 128>(sV + (buf ^ 1) * 64 * D, kv_ptr(a.v_cache, j + 1), tid);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
      const uint32_t qb = smem_u32(sQ);
#pragma unroll
      for (int kk = 0; kk < NK; ++kk) {
        const int r = warp * 16 + (lane & 15);
        ldmatrix_x4(qb + swz<D>(r, kk * 2 + (lane >> 4)) * 16, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const uint32_t kb = smem_u32(sK + buf * 64 * D), vb = smem_u32(sV + buf * 64 * D);
    // S = Q K^T : 16 x 64 per warp
    float s[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
#pragma unroll
      for (int n = 0; n < 8; n += 2) {
        uint32_t b0, b1, b2, b3;
        const int r = n * 8 + (lane & 7) + ((lane >> 4) << 3);
        ldmatrix_x4(kb + swz<D>(r, kk * 2 + ((lane >> 3) & 1)) * 16, b0, b1, b2, b3);
        mma_bf16_16816(s[n], qf[kk], b0, b1);
        mma_bf16_16816(s[n + 1], qf[kk], b2, b3);
      }
    }
    // scale, causal mask on the diagonal tile, online softmax (log2 domain)
    const bool diag = (j * 64 + 63 > off + q_start);
    float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[n][e] * a.scale_log2;
        if (diag) {
          const int kpos = j * 64 + n * 8 + 2 * t4 + (e & 1);
          const int qpos = qpos0 + (e >> 1) * 8;
          if (kpos > qpos) v = -INFINITY;
        }
        s[n][e] = v;
        mnew[e >> 1] = fmaxf(mnew[e >> 1], v);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 1));
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 2));
    }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) corr[r] = (mrow[r] == -INFINITY) ? 0.f : exp2f(mrow[r] - mnew[r]);
    uint32_t pf[4][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p0 = (mnew[0] == -INFINITY) ? 0.f : exp2f(s[n][0] - mnew[0]);
      float p1 = (mnew[0] == -INFINITY) ? 0.f : exp2f(s[n][1] - mnew[0]);
      float p2 = (mnew[1] == -INFINITY) ? 0.f : exp2f(s[n][2] - mnew[1]);
      float p3 = (mnew[1] == -INFINITY) ? 0.f : exp2f(s[n][3] - mnew[1]);
      rs[0] += p0 + p1;
      rs[1] += p2 + p3;
      pf[n >> 1][(n & 1) * 2 + 0] = pack_bf16x2(p0, p1);
      pf[n >> 1][(n & 1) * 2 + 1] = pack_bf16x2(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      lrow[r] = lrow[r] * corr[r] + rs[r];
      mrow[r] = mnew[r];
    }
#pragma unroll
    for (int i = 0; i < ND; ++i) {
      o[i][0] *= corr[0]; o[i][1] *= corr[0];
      o[i][2] *= corr[1]; o[i][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      // A fragment: a0 (row g, keys 16kk+2t..), a1 (row g+8), a2 (row g, keys +8), a3 (row g+8, keys +8)
      uint32_t af[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
      for (int dn = 0; dn < ND; dn += 2) {
        uint32_t b0, b1, b2, b3;
        const int r = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        ldmatrix_x4_trans(vb + swz<D>(r, dn + (lane >> 4)) * 16, b0, b1, b2, b3);
        mma_bf16_16816(o[dn], af, b0, b1);
        mma_bf16_16816(o[dn + 1], af, b2, b3);
      }
    }
    __syncthreads();
  }
  // row sums across the quad, normalise, store bf16
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  const float inv0 = 1.f / lrow[0], inv1 = 1.f / lrow[1];
  const int ld = a.n_heads * D;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qrow = q_start + warp * 16 + g + r * 8;
    if (qrow < len) {
      bf16* dst = a.out + (int64_t)(tok0 + qrow) * ld + h * D;
      const float inv = r ? inv1 : inv0;
#pragma unroll
      for (int i = 0; i < ND; ++i)
        *reinterpret_cast<uint32_t*>(dst + i * 8 + 2 * t4) = pack_bf16x2(o[i][2 * r] * inv, o[i][2 * r + 1] * inv);
    }
  }
}

// ------------------------------------------------------------------ decode

// byte offset of 16-byte chunk c (0..15) of row r in a [64][128] bf16 tile staged by
// TMA with 128B swizzle as two [64][64] panels (chunk c%8 of a panel row at c ^ (r%8))
__device__ __forceinline__ uint32_t tma_swz(int r, int c) {
  return (uint32_t)((c >> 3) * 8192 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// TMA: K/V tiles arrive by cp.async.bulk.tensor (one elected thread, mbarrier per
// stage) into 128B-swizzled panels; otherwise cp.async into the XOR-swizzled layout.
// DEC_STAGES = 3 (2 CTAs per SM) or 2 (68 KB of smem: 3 CTAs per SM, one block of
// prefetch per CTA; more CTAs in flight when the grid is a few waves of uniform lengths)
template <int D, bool TMA, int DEC_STAGES = 3>
__global__ void __launch_bounds__(128) attn_decode_kernel(DecodeAttnArgs a, const __grid_constant__ CUtensorMap kvmap) {
  constexpr int NK = D / 16, ND = D / 8;
  extern __shared__ __align__(128) uint8_t sm_raw[];
  uint8_t* sm = TMA ? reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023))
                    : sm_raw;
  bf16* sK = reinterpret_cast<bf16*>(sm);                  // [STAGES][64][D]
  bf16* sV = sK + DEC_STAGES * 64 * D;
  bf16* sQ = sV + DEC_STAGES * 64 * D;                     // [16][D]
  uint64_t* full = reinterpret_cast<uint64_t*>(sQ + 16 * D);  // [STAGES] (TMA)
  uint64_t* empty = full + DEC_STAGES;                         // [STAGES]: the 4 warps consumed the stage
  int* s_bt = reinterpret_cast<int*>(empty + DEC_STAGES);      // (TMA) [256] this CTA's block-table range
  float* red = reinterpret_cast<float*>(sm);               // reused after the main loop
  if (TMA && threadIdx.x == 0) {
    for (int s = 0; s < DEC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_barrier_init();
    tma_prefetch(&kvmap);
  }
  pdl_trigger();
  pdl_wait();

  // CTAs in longest-context-first order, all kv heads of a sequence adjacent (LPT:
  // the long sequences start in the first wave, short ones fill the tail)
  const int rank = blockIdx.x / a.n_kv, kvh = blockIdx.x % a.n_kv, split = blockIdx.z;
  const int b = a.order ? a.order[rank] : rank;
  const int G = a.n_heads / a.n_kv;
  const int ctx = a.ctx_lens[b];
  const int n_blocks = (ctx + 63) / 64;
  const int blk0 = split * a.blocks_per_split;
  const int blk1 = min(n_blocks, blk0 + a.blocks_per_split);
  const int* bt = a.block_tables + (int64_t)b * a.bt_ld;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g = lane >> 2, t4 = lane & 3;

  // (TMA) the CTA's block-table range staged in smem by all threads at once: the issuing
  // thread otherwise reads bt[] from global right before every refill (an L2 round trip
  // on the critical path of each 64-token block)
  // (the first refill reads it after the prologue barrier; the prologue loads below read
  // bt[] directly, so the first K/V loads go out before any other global round trip)
  const bool sbt = TMA && blk1 - blk0 <= 256;
  if (sbt)
    for (int i = tid; i < blk1 - blk0; i += 128) s_bt[i] = bt[blk0 + i];
  auto issue = [&](int blk, int st) {
    if constexpr (TMA) {
      if (tid == 0) {
        // pool rows: ((block * L + layer) * 2 + kv) * Mkv * 64 + kvh * 64 + token
        const int64_t base =
            ((int64_t)((sbt && blk >= blk0 + DEC_STAGES - 1) ? s_bt[blk - blk0] : bt[blk]) * a.n_layers + a.layer) * 2;
        const int krow = (int)((base * a.n_kv + kvh) * 64);
        const int vrow = (int)(((base + 1) * a.n_kv + kvh) * 64);
        mbar_arrive_expect_tx(&full[st], 2 * 64 * D * 2);
        for (int pn = 0; pn < 2; ++pn) {
          tma_load_2d(reinterpret_cast<uint8_t*>(sK + st * 64 * D) + pn * 8192, &kvmap, &full[st], pn * 64, krow);
          tma_load_2d(reinterpret_cast<uint8_t*>(sV + st * 64 * D) + pn * 8192, &kvmap, &full[st], pn * 64, vrow);
        }
      }
    } else {
      const int64_t off = (int64_t)bt[blk] * a.blk_stride + (int64_t)kvh * 64 * D;
      load_tile64<D, 128>(sK + st * 64 * D, a.k_cache + off, tid);
      load_tile64<D, 128>(sV + st * 64 * D, a.v_cache + off, tid);
    }
  };
  // K/V tile chunk offsets (bytes) in either staging layout
  auto kv_off = [&](int r, int c) -> uint32_t {
    if constexpr (TMA) return tma_swz(r, c);
    else return (uint32_t)swz<D>(r, c) * 16;
  };
  const bool fused_qkv = TMA && a.qkv_part != nullptr;  // (kernel-uniform)
  // the current token's K / V are written by this CTA (fused QKV) into the last block:
  // that block's TMA load must follow the writes
  const bool writes_kv = fused_qkv && blk1 == n_blocks;
  const int late = writes_kv ? n_blocks - 1 : -1;  // block whose load waits for the K / V write
  // prologue: the first K/V blocks, then the q rows (their loads overlap)
#pragma unroll
  for (int s = 0; s < DEC_STAGES - 1; ++s) {
    if (blk0 + s < blk1 && blk0 + s != late) issue(blk0 + s, s);
    if (!TMA) cp_async_commit();
  }
  if (fused_qkv) {
    // q = RoPE(sum of the splits) for the G heads, and the new k (RoPE) / v row
    const int half = D / 2, qd = a.n_heads * D, kd = a.n_kv * D;
    const int p = a.pos[b];
    const int64_t plane = (int64_t)a.B * a.qkv_ld;
    const float* src = a.qkv_part + (int64_t)b * a.qkv_ld;
    if (tid < 16 * (D / 8) - G * (D / 8))  // zero q rows G..15
      for (int i = G * (D / 8) + tid; i < 16 * (D / 8); i += 128) {
        const int r = i / (D / 8), c = i % (D / 8);
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sQ) + swz<D>(r, c) * 16) = make_uint4(0, 0, 0, 0);
      }
    for (int i = tid; i < (G + 2) * half; i += 128) {
      const int r = i / half, j = i % half;  // r < G: q head; G: k; G + 1: v (pair j = columns 2j, 2j + 1)
      const int col = r < G ? (kvh * G + r) * D + 2 * j : r == G ? qd + kvh * D + 2 * j : qd + kd + kvh * D + 2 * j;
      float x0 = 0.f, x1 = 0.f;
      for (int sp = 0; sp < a.qkv_splits; ++sp) {  // split order, as the reduction kernel
        const float2 v = *reinterpret_cast<const float2*>(src + sp * plane + col);
        x0 += v.x;
        x1 += v.y;
      }
      if (r <= G) {
        const float cs = a.rope_cos[(int64_t)p * half + j], sn = a.rope_sin[(int64_t)p * half + j];
        const float y0 = x0 * cs - x1 * sn, y1 = x1 * cs + x0 * sn;  // dims j and j + D/2
        if (r < G) {
          uint8_t* q8 = reinterpret_cast<uint8_t*>(sQ);
          *reinterpret_cast<bf16*>(q8 + swz<D>(r, j / 8) * 16 + (j % 8) * 2) = __float2bfloat16_rn(y0);
          *reinterpret_cast<bf16*>(q8 + swz<D>(r, (j + half) / 8) * 16 + ((j + half) % 8) * 2) = __float2bfloat16_rn(y1);
        } else if (writes_kv) {
          const int sl = a.slot[b];
          bf16* dst = const_cast<bf16*>(a.k_cache) + (int64_t)(sl >> 6) * a.blk_stride + ((int64_t)kvh * 64 + (sl & 63)) * D;
          dst[j] = __float2bfloat16_rn(y0);
          dst[j + half] = __float2bfloat16_rn(y1);
        }
      } else if (writes_kv) {
        const int sl = a.slot[b];
        bf16* dst = const_cast<bf16*>(a.v_cache) + (int64_t)(sl >> 6) * a.blk_stride + ((int64_t)kvh * 64 + (sl & 63)) * D;
        *reinterpret_cast<uint32_t*>(dst + 2 * j) = pack_bf16x2(x0, x1);
      }
    }
    if (writes_kv) asm volatile("fence.proxy.async.global;" ::: "memory");  // generic K/V writes -> TMA reads
  } else {
    // q rows: head kvh*G + r for r < G, zero rows above
    for (int i = tid; i < 16 * (D / 8); i += 128) {
      const int r = i / (D / 8), c = i % (D / 8);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < G) v = *reinterpret_cast<const uint4*>(a.q + ((int64_t)b * a.n_heads + kvh * G + r) * D + c * 8);
      *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sQ) + swz<D>(r, c) * 16) = v;
    }
  }
  __syncthreads();
  if (late >= blk0 && late < blk0 + DEC_STAGES - 1) {  // the last block was held back: load it now
    if (tid == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
    issue(late, late - blk0);
  }
  uint32_t qf[NK][4];
  {
    const uint32_t qb = smem_u32(sQ);
#pragma unroll
    for (int kk = 0; kk < NK; ++kk)
      ldmatrix_x4(qb + swz<D>(lane & 15, kk * 2 + (lane >> 4)) * 16, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
  }
  float o[ND][4];
#pragma unroll
  for (int i = 0; i < ND; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};

  for (int blk = blk0; blk < blk1; ++blk) {
    const int it = blk - blk0;
    {
      const int nb = blk + DEC_STAGES - 1;
      // TMA: the stage was read in iteration it - 1; wait until all 4 warps released it
      // (per-stage empty barrier instead of a CTA-wide barrier every block)
      if (TMA && tid == 0 && nb < blk1 && it >= 1) mbar_wait(&empty[(it - 1) % DEC_STAGES], ((it - 1) / DEC_STAGES) & 1);
      if (nb < blk1) issue(nb, (it + DEC_STAGES - 1) % DEC_STAGES);
      if (!TMA) cp_async_commit();
    }
    const int st = it % DEC_STAGES;
    if constexpr (TMA) {
      mbar_wait(&full[st], (it / DEC_STAGES) & 1);
    } else {
      cp_async_wait<DEC_STAGES - 1>();
      __syncthreads();
    }
    const uint32_t kb = smem_u32(sK + st * 64 * D), vb = smem_u32(sV + st * 64 * D);
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
      uint32_t b0, b1, b2, b3;
      const int r = warp * 16 + (lane & 7) + ((lane >> 4) << 3);
      ldmatrix_x4(kb + kv_off(r, kk * 2 + ((lane >> 3) & 1)), b0, b1, b2, b3);
      mma_bf16_16816(s[0], qf[kk], b0, b1);
      mma_bf16_16816(s[1], qf[kk], b2, b3);
    }
    // Rows 8..15 of the MMA (accumulator elements 2, 3) hold heads 8..15 of the group:
    // with G <= 8 (every shape here) they are padding, so their max / exp / rescale work
    // is skipped and their P is zero (the decode step is issue-bound at power-capped clocks)
    const bool hi_rows = G > 8;  // block-uniform
    float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (e >= 2 && !hi_rows) continue;
        const int kpos = blk * 64 + warp * 16 + n * 8 + 2 * t4 + (e & 1);
        float v = (kpos < ctx) ? s[n][e] * a.scale_log2 : -INFINITY;
        s[n][e] = v;
        mnew[e >> 1] = fmaxf(mnew[e >> 1], v);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (r == 1 && !hi_rows) continue;
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 1));
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 2));
    }
    float corr[2] = {1.f, 1.f}, rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (r == 1 && !hi_rows) continue;
      corr[r] = (mrow[r] == -INFINITY) ? 0.f : exp2f(mrow[r] - mnew[r]);
    }
    uint32_t af[4];
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      float p0 = (mnew[0] == -INFINITY) ? 0.f : exp2f(s[n][0] - mnew[0]);
      float p1 = (mnew[0] == -INFINITY) ? 0.f : exp2f(s[n][1] - mnew[0]);
      float p2 = 0.f, p3 = 0.f;
      if (hi_rows) {
        p2 = (mnew[1] == -INFINITY) ? 0.f : exp2f(s[n][2] - mnew[1]);
        p3 = (mnew[1] == -INFINITY) ? 0.f : exp2f(s[n][3] - mnew[1]);
      }
      rs[0] += p0 + p1;
      rs[1] += p2 + p3;
      af[n * 2 + 0] = pack_bf16x2(p0, p1);
      af[n * 2 + 1] = pack_bf16x2(p2, p3);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      lrow[r] = lrow[r] * corr[r] + rs[r];
      mrow[r] = mnew[r];
    }
    // rescale O only when some row of the warp raised its max (rare after the first blocks)
    if (__any_sync(0xffffffffu, corr[0] != 1.f || corr[1] != 1.f)) {
#pragma unroll
      for (int i = 0; i < ND; ++i) {
        o[i][0] *= corr[0]; o[i][1] *= corr[0];
        o[i][2] *= corr[1]; o[i][3] *= corr[1];
      }
    }
#pragma unroll
    for (int dn = 0; dn < ND; dn += 2) {
      uint32_t b0, b1, b2, b3;
      const int r = warp * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
      ldmatrix_x4_trans(vb + kv_off(r, dn + (lane >> 4)), b0, b1, b2, b3);
      mma_bf16_16816(o[dn], af, b0, b1);
      mma_bf16_16816(o[dn + 1], af, b2, b3);
    }
    if constexpr (TMA) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    } else {
      __syncthreads();
    }
  }
  if (!TMA) cp_async_wait<0>();
  __syncthreads();
  // quad sums of l
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  // cross-warp combine (fixed order): red = [4 warps][16 rows][D + 2]
  constexpr int RS = D + 2;
  float* myred = red + warp * 16 * RS;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = g + r * 8;
#pragma unroll
    for (int i = 0; i < ND; ++i) {
      myred[row * RS + i * 8 + 2 * t4] = o[i][2 * r];
      myred[row * RS + i * 8 + 2 * t4 + 1] = o[i][2 * r + 1];
    }
    if (t4 == 0) {
      myred[row * RS + D] = mrow[r];
      myred[row * RS + D + 1] = lrow[r];
    }
  }
  __syncthreads();
  for (int i = tid; i < G * D; i += 128) {
    const int row = i / D, d = i % D;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, red[(w * 16 + row) * RS + D]);
    float acc = 0.f, l = 0.f;
    for (int w = 0; w < 4; ++w) {
      const float mw = red[(w * 16 + row) * RS + D];
      const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
      acc += f * red[(w * 16 + row) * RS + d];
      l += f * red[(w * 16 + row) * RS + D + 1];
    }
    const int h = kvh * G + row;
    if (a.n_splits == 1) {
      a.out[(int64_t)b * a.n_heads * D + h * D + d] = __float2bfloat16_rn(acc / l);
    } else {
      const int64_t pi = ((int64_t)b * a.n_heads + h) * a.n_splits + split;
      a.part_o[pi * D + d] = acc;
      if (d == 0) {
        a.part_ml[pi * 2] = M;
        a.part_ml[pi * 2 + 1] = l;
      }
    }
  }
}

// ------------------------------------------------------------------ decode, stream-K
// Persistent variant of the TMA decode kernel (head_dim 128, G <= 8 q heads per kv head).
// tools/attn_decode_probe.py: at B = 128 the per-item kernel pays ~37 us per launch on
// top of streaming (ctx 1300: 129.5 us; ctx 2600: 222.3 us, i.e. 7.4 TB/s marginal) --
// each CTA's start-up round trips and the last partial wave (1024 CTAs = 3.46 waves of
// 296). Here sk_grid CTAs (2 per SM) stream equal shares of the (rank, kv head, block)
// units in LPT order, one start-up each; the K / V ring runs across item boundaries.
// An item cut between CTAs leaves each part's (m, l, o) in the workspace; its last
// contributor (per-item counter) combines the parts in order and writes the output.
constexpr int SK_MAXPARTS = 32;  // parts (items) per CTA
constexpr int SK_UNITS = 256;    // units per CTA (pool row table in smem)

template <int DEC_STAGES>
__global__ void __launch_bounds__(128) attn_decode_sk_kernel(DecodeAttnArgs a, const __grid_constant__ CUtensorMap kvmap) {
  constexpr int D = 128, NK = D / 16, ND = D / 8, GMAX = 4, RS = D + 2;
  extern __shared__ __align__(128) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  bf16* sK = reinterpret_cast<bf16*>(sm);                      // [STAGES][64][D]
  bf16* sV = sK + DEC_STAGES * 64 * D;
  bf16* sQ = sV + DEC_STAGES * 64 * D;                         // [16][D]
  float* red = reinterpret_cast<float*>(sQ + 16 * D);          // [4 warps][GMAX rows][D + 2]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 4 * GMAX * RS);
  uint64_t* empty = full + DEC_STAGES;
  int* s_row = reinterpret_cast<int*>(empty + DEC_STAGES);     // [SK_UNITS] K pool row of each unit
  int* s_part = s_row + SK_UNITS;                              // [SK_MAXPARTS][8] part descriptors
  int* s_np = s_part + SK_MAXPARTS * 8;                        // [0] parts, [1] last-arriver flag
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g = lane >> 2, t4 = lane & 3;
  const int G = a.n_heads / a.n_kv;
  if (tid == 0) {
    for (int s = 0; s < DEC_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_barrier_init();
    tma_prefetch(&kvmap);
  }
  pdl_trigger();
  pdl_wait();
  const int NR = a.B;                 // LPT ranks
  const int Ctot = gridDim.x, c = blockIdx.x;
  const int U = a.sk_prefix[NR] * a.n_kv;
  const int u0 = (int)((long long)c * U / Ctot), u1 = (int)((long long)(c + 1) * U / Ctot);
  // ---- this CTA's parts: descriptor = {rank, kvh, blk0, blk1, nb, seq, ctx, first unit}
  if (tid == 0) {
    int lo = 0, hi = NR;  // the rank r with prefix[r] * n_kv <= u0 < prefix[r + 1] * n_kv
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (a.sk_prefix[mid] * a.n_kv <= u0) lo = mid;
      else hi = mid;
    }
    int np = 0, u = u0, r = lo;
    while (u < u1 && np < SK_MAXPARTS) {
      const int p0 = a.sk_prefix[r], nb = a.sk_prefix[r + 1] - p0;
      if (nb == 0 || u >= (p0 + nb) * a.n_kv) {
        ++r;
        continue;
      }
      const int off = u - p0 * a.n_kv, kvh = off / nb, blk0 = off % nb;
      const int blk1 = min(nb, blk0 + (u1 - u));
      const int seq = a.order ? a.order[r] : r;
      int* d = s_part + np * 8;
      d[0] = r; d[1] = kvh; d[2] = blk0; d[3] = blk1; d[4] = nb; d[5] = seq; d[6] = a.ctx_lens[seq]; d[7] = u - u0;
      ++np;
      u += blk1 - blk0;
    }
    s_np[0] = (u < u1) ? -1 : np;  // -1: more parts than SK_MAXPARTS (the host sizes the grid so this never happens)
  }
  __syncthreads();
  const int np = s_np[0];
  const int n_units = min(u1 - u0, SK_UNITS);
  if (np < 0 || u1 - u0 > SK_UNITS) {  // (cannot happen for grids from attn_decode_sk_grid)
    if (tid == 0) __trap();
    return;
  }
  // ---- K pool row of every unit (one round trip for all, before the stream starts)
  for (int j = tid; j < n_units; j += 128) {
    int k = 0;
    while (k + 1 < np && s_part[(k + 1) * 8 + 7] <= j) ++k;
    const int* d = s_part + k * 8;
    const int blk = d[2] + (j - d[7]);
    const int64_t base = ((int64_t)a.block_tables[(int64_t)d[5] * a.bt_ld + blk] * a.n_layers + a.layer) * 2;
    s_row[j] = (int)((base * a.n_kv + d[1]) * 64);
  }
  __syncthreads();
  auto issue = [&](int j) {  // unit j into stage j % S (tid 0)
    const int st = j % DEC_STAGES;
    const int krow = s_row[j], vrow = krow + a.n_kv * 64;
    mbar_arrive_expect_tx(&full[st], 2 * 64 * D * 2);
    for (int pn = 0; pn < 2; ++pn) {
      tma_load_2d(reinterpret_cast<uint8_t*>(sK + st * 64 * D) + pn * 8192, &kvmap, &full[st], pn * 64, krow);
      tma_load_2d(reinterpret_cast<uint8_t*>(sV + st * 64 * D) + pn * 8192, &kvmap, &full[st], pn * 64, vrow);
    }
  };
  if (tid == 0)
    for (int j = 0; j < DEC_STAGES - 1 && j < n_units; ++j) issue(j);

  const float* part_o = a.part_o;   // [item][maxp][G][D]
  float* part_w = a.part_o;
  float* part_ml = a.part_o + (int64_t)NR * a.n_kv * a.sk_maxp * G * D;  // [item][maxp][G][2]
  // q rows of part k (head kvh * G + row; rows >= G zero): each thread's 2 x 16 B of the
  // [16][D] tile, loaded into registers one part ahead (the loads of part k + 1 fly while
  // part k streams) and stored to sQ at the part boundary
  static_assert(16 * (D / 8) == 2 * 128, "two 16-byte q chunks per thread");
  auto fetch_q = [&](int k, uint4 (&qv)[2]) {
    const int* d = s_part + k * 8;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = tid + h * 128, row = i / (D / 8), cc = i % (D / 8);
      qv[h] = row < G ? *reinterpret_cast<const uint4*>(a.q + ((int64_t)d[5] * a.n_heads + d[1] * G + row) * D + cc * 8)
                      : make_uint4(0, 0, 0, 0);
    }
  };
  uint4 qnext[2];
  if (np > 0) fetch_q(0, qnext);
  for (int k = 0; k < np; ++k) {
    const int* d = s_part + k * 8;
    const int r = d[0], kvh = d[1], blk0 = d[2], blk1 = d[3], nb = d[4], seq = d[5], ctx = d[6], j0 = d[7];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = tid + h * 128, row = i / (D / 8), cc = i % (D / 8);
      *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sQ) + swz<D>(row, cc) * 16) = qnext[h];
    }
    __syncthreads();
    if (k + 1 < np) fetch_q(k + 1, qnext);
    uint32_t qf[NK][4];
    {
      const uint32_t qb = smem_u32(sQ);
#pragma unroll
      for (int kk = 0; kk < NK; ++kk)
        ldmatrix_x4(qb + swz<D>(lane & 15, kk * 2 + (lane >> 4)) * 16, qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
    }
    float o[ND][4];
#pragma unroll
    for (int i = 0; i < ND; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mrow = -INFINITY, lrow = 0.f;  // row g (rows g + 8 are padding: G <= 8)
    for (int blk = blk0; blk < blk1; ++blk) {
      const int j = j0 + (blk - blk0);
      if (tid == 0 && j + DEC_STAGES - 1 < n_units) {
        if (j >= 1) mbar_wait(&empty[(j - 1) % DEC_STAGES], ((j - 1) / DEC_STAGES) & 1);
        issue(j + DEC_STAGES - 1);
      }
      const int st = j % DEC_STAGES;
      mbar_wait(&full[st], (j / DEC_STAGES) & 1);
      const uint32_t kb = smem_u32(sK + st * 64 * D), vb = smem_u32(sV + st * 64 * D);
      float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < NK; ++kk) {
        uint32_t b0, b1, b2, b3;
        const int rr = warp * 16 + (lane & 7) + ((lane >> 4) << 3);
        ldmatrix_x4(kb + tma_swz(rr, kk * 2 + ((lane >> 3) & 1)), b0, b1, b2, b3);
        mma_bf16_16816(s[0], qf[kk], b0, b1);
        mma_bf16_16816(s[1], qf[kk], b2, b3);
      }
      float mnew = mrow;
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kpos = blk * 64 + warp * 16 + n * 8 + 2 * t4 + e;
          const float v = (kpos < ctx) ? s[n][e] * a.scale_log2 : -INFINITY;
          s[n][e] = v;
          mnew = fmaxf(mnew, v);
        }
      mnew = fmaxf(mnew, __shfl_xor_sync(0xffffffffu, mnew, 1));
      mnew = fmaxf(mnew, __shfl_xor_sync(0xffffffffu, mnew, 2));
      const float corr = (mrow == -INFINITY) ? 0.f : exp2f(mrow - mnew);
      float rs = 0.f;
      uint32_t af[4];
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        const float p0 = (mnew == -INFINITY) ? 0.f : exp2f(s[n][0] - mnew);
        const float p1 = (mnew == -INFINITY) ? 0.f : exp2f(s[n][1] - mnew);
        rs += p0 + p1;
        af[n * 2 + 0] = pack_bf16x2(p0, p1);
        af[n * 2 + 1] = 0u;  // rows 8..15: padding
      }
      lrow = lrow * corr + rs;
      mrow = mnew;
      if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll
        for (int i = 0; i < ND; ++i) {
          o[i][0] *= corr;
          o[i][1] *= corr;
        }
      }
#pragma unroll
      for (int dn = 0; dn < ND; dn += 2) {
        uint32_t b0, b1, b2, b3;
        const int rr = warp * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        ldmatrix_x4_trans(vb + tma_swz(rr, dn + (lane >> 4)), b0, b1, b2, b3);
        mma_bf16_16816(o[dn], af, b0, b1);
        mma_bf16_16816(o[dn + 1], af, b2, b3);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    // ---- the part's (m, l, o) over its blocks: warps combined in fixed order, GMAX rows
    //      of red at a time (G = 8: two rounds)
    lrow += __shfl_xor_sync(0xffffffffu, lrow, 1);
    lrow += __shfl_xor_sync(0xffffffffu, lrow, 2);
    float* myred = red + warp * GMAX * RS;
    const bool whole = blk0 == 0 && blk1 == nb;
    const int item = r * a.n_kv + kvh;
    // part index within the item: CTAs from the owner of the item's first unit
    const int iu0 = (a.sk_prefix[r] * a.n_kv) + kvh * nb;
    const int c_lo = (int)(((long long)(iu0 + 1) * Ctot - 1) / U);
    const int c_hi = (int)(((long long)(iu0 + nb) * Ctot - 1) / U);
    const int pidx = c - c_lo, nparts = c_hi - c_lo + 1;
    for (int rb = 0; rb < G; rb += GMAX) {
      const int nr = min(GMAX, G - rb);
      if (rb > 0) __syncthreads();  // previous round's reads of red are done
      if (g >= rb && g < rb + nr) {
        const int gr = g - rb;
#pragma unroll
        for (int i = 0; i < ND; ++i) {
          myred[gr * RS + i * 8 + 2 * t4] = o[i][0];
          myred[gr * RS + i * 8 + 2 * t4 + 1] = o[i][1];
        }
        if (t4 == 0) {
          myred[gr * RS + D] = mrow;
          myred[gr * RS + D + 1] = lrow;
        }
      }
      __syncthreads();
      for (int i = tid; i < nr * D; i += 128) {
        const int rr = i / D, row = rb + rr, dd = i % D;
        float M = -INFINITY;
        for (int w = 0; w < 4; ++w) M = fmaxf(M, red[(w * GMAX + rr) * RS + D]);
        float acc = 0.f, l = 0.f;
        for (int w = 0; w < 4; ++w) {
          const float mw = red[(w * GMAX + rr) * RS + D];
          const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
          acc += f * red[(w * GMAX + rr) * RS + dd];
          l += f * red[(w * GMAX + rr) * RS + D + 1];
        }
        if (whole) {
          a.out[(int64_t)seq * a.n_heads * D + (kvh * G + row) * D + dd] = __float2bfloat16_rn(acc / l);
        } else {
          const int64_t pi = (int64_t)item * a.sk_maxp + pidx;
          part_w[(pi * G + row) * D + dd] = acc;
          if (dd == 0) {
            part_ml[(pi * G + row) * 2] = M;
            part_ml[(pi * G + row) * 2 + 1] = l;
          }
        }
      }
    }
    if (!whole) {
      // the last of the item's parts to finish combines them all in part order
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        const int old = atomicAdd(&a.sk_cnt[item], 1);
        s_np[1] = old == nparts - 1;
        if (old == nparts - 1) a.sk_cnt[item] = 0;
      }
      __syncthreads();
      if (s_np[1]) {
        __threadfence();
        for (int i = tid; i < G * D; i += 128) {
          const int row = i / D, dd = i % D;
          const int64_t pb = (int64_t)item * a.sk_maxp;
          float M = -INFINITY;
          for (int pp = 0; pp < nparts; ++pp) M = fmaxf(M, __ldcg(part_ml + ((pb + pp) * G + row) * 2));
          float acc = 0.f, l = 0.f;
          for (int pp = 0; pp < nparts; ++pp) {
            const float mp = __ldcg(part_ml + ((pb + pp) * G + row) * 2);
            const float f = (mp == -INFINITY) ? 0.f : exp2f(mp - M);
            acc += f * __ldcg(part_o + ((pb + pp) * G + row) * D + dd);
            l += f * __ldcg(part_ml + ((pb + pp) * G + row) * 2 + 1);
          }
          a.out[(int64_t)seq * a.n_heads * D + (kvh * G + row) * D + dd] = __float2bfloat16_rn(acc / l);
        }
      }
    }
    __syncthreads();  // red / sQ free for the next part
  }
}

int attn_decode_sk_grid(int total_units, int max_item_blocks, int min_item_blocks, int n_heads, int n_kv,
                        int head_dim, int num_sms, int* maxp, bool force) {
  // ECOSERVE_ATTN_SK=1 enables the stream-K kernel. Off by default: standalone it removes the
  // per-item kernel's start-up / last-wave cost, but inside the decode step it measured
  // slower (8B B = 128: 8.08-8.16 vs 7.79-7.83 ms per step): every CTA ends together, while
  // the per-item kernel's LPT tail lets the O projection's CTAs start and prefetch weights
  // under PDL on the SMs it frees.
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("ECOSERVE_ATTN_SK");
    mode = (e && e[0] == '1') ? 1 : 0;
  }
  if (!(mode || force) || head_dim != 128 || n_heads / n_kv > 8) return 0;
  const int grid = 2 * num_sms;
  if (total_units < 4 * grid) return 0;  // (short work: the per-item kernel)
  const int per = total_units / grid;    // units per CTA (floor)
  if (per + 1 > SK_UNITS) return 0;
  // parts per item: ceil(len / per) + 1; parts per CTA: <= units per CTA (every part >= 1 unit)
  const int mp = (max_item_blocks + per - 1) / per + 1;
  if (mp > 64) return 0;
  *maxp = mp;
  // parts per CTA: a range of <= per + 1 units over items of >= min_item_blocks each
  if ((per + 1 + min_item_blocks - 1) / max(1, min_item_blocks) + 1 > SK_MAXPARTS) return 0;
  return grid;
}

template <int D>
__global__ void attn_combine_kernel(DecodeAttnArgs a) {
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x, h = blockIdx.y;
  const int64_t p0 = ((int64_t)b * a.n_heads + h) * a.n_splits;
  float M = -INFINITY;
  for (int s = 0; s < a.n_splits; ++s) M = fmaxf(M, a.part_ml[(p0 + s) * 2]);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.f, l = 0.f;
    for (int s = 0; s < a.n_splits; ++s) {
      const float ms = a.part_ml[(p0 + s) * 2];
      const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
      acc += f * a.part_o[(p0 + s) * D + d];
      l += f * a.part_ml[(p0 + s) * 2 + 1];
    }
    a.out[(int64_t)b * a.n_heads * D + h * D + d] = __float2bfloat16_rn(acc / l);
  }
}

// ------------------------------------------------------------------ launchers
template <int D>
static cudaError_t prefill_d(const PrefillAttnArgs& a, cudaStream_t s) {
  const int smem = 5 * 64 * D * 2;
  cudaError_t e = ensure_smem(attn_prefill_kernel<D>, smem);
  if (e != cudaSuccess) return e;
  if (a.n_tiles == 0) return cudaSuccess;
  return launch_k(attn_prefill_kernel<D>, dim3(a.n_tiles, a.n_heads), dim3(128), smem, s, a);
}

cudaError_t attn_prefill_launch(const PrefillAttnArgs& a, int head_dim, cudaStream_t s) {
  switch (head_dim) {
    case 32: return prefill_d<32>(a, s);
    case 64: return prefill_d<64>(a, s);
    case 128: return prefill_d<128>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

static size_t sk_smem(int stages) {
  return (size_t)stages * 2 * 64 * 128 * 2 + 16 * 128 * 2 + 4 * 4 * (128 + 2) * 4 + 2 * stages * 8 + SK_UNITS * 4 +
         SK_MAXPARTS * 8 * 4 + 16 + 1024;
}

template <int D, int ST>
static cudaError_t decode_st(const DecodeAttnArgs& a, cudaStream_t s) {
  if constexpr (D == 128) {
    if (a.sk_grid > 0 && a.kvmap) {
      const int smem = (int)sk_smem(ST);
      cudaError_t e = ensure_smem(attn_decode_sk_kernel<ST>, smem);
      if (e != cudaSuccess) return e;
      return launch_k(attn_decode_sk_kernel<ST>, dim3(a.sk_grid), dim3(128), smem, s, a, *a.kvmap);
    }
  }
  const bool tma = D == 128 && a.kvmap != nullptr;
  int smem = (2 * ST * 64 * D + 16 * D) * 2;
  const int red_bytes = 4 * 16 * (D + 2) * 4;
  if (smem < red_bytes) smem = red_bytes;
  if (tma) smem += 1024 + 64 + 256 * 4;  // 1 KB alignment slack + stage barriers + block-table range
  cudaError_t e = tma ? ensure_smem(attn_decode_kernel<D, true, ST>, smem)
                      : ensure_smem(attn_decode_kernel<D, false, ST>, smem);
  if (e != cudaSuccess) return e;
  if (a.B == 0) return cudaSuccess;
  if (a.n_heads / a.n_kv > 16) return cudaErrorInvalidValue;
  CUtensorMap dummy;
  memset(&dummy, 0, sizeof(dummy));
  const CUtensorMap& map = tma ? *a.kvmap : dummy;
  if (tma)
    e = launch_k(attn_decode_kernel<D, true, ST>, dim3(a.B * a.n_kv, 1, a.n_splits), dim3(128), smem, s, a, map);
  else
    e = launch_k(attn_decode_kernel<D, false, ST>, dim3(a.B * a.n_kv, 1, a.n_splits), dim3(128), smem, s, a, map);
  if (e != cudaSuccess || a.n_splits == 1) return e;
  return launch_k(attn_combine_kernel<D>, dim3(a.B, a.n_heads), dim3(D), 0, s, a);
}

template <int D>
static cudaError_t decode_d(const DecodeAttnArgs& a, cudaStream_t s) {
  static int st = -1;  // ECOSERVE_ATTN_STAGES=2: 3 CTAs per SM
  if (st < 0) {
    const char* e = getenv("ECOSERVE_ATTN_STAGES");
    st = (e && e[0] == '2') ? 2 : 3;
  }
  return st == 2 ? decode_st<D, 2>(a, s) : decode_st<D, 3>(a, s);
}

cudaError_t attn_decode_launch(const DecodeAttnArgs& a, int head_dim, cudaStream_t s) {
  switch (head_dim) {
    case 32: return decode_d<32>(a, s);
    case 64: return decode_d<64>(a, s);
    case 128: return decode_d<128>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace eco
