// tcgen05 / TMEM / TMA warp-specialised persistent GEMM for sm_100a with the
// fused epilogues of the PaDG instance hot path (SURVEY 8(a) rows a7, a9-a13,
// a15, a16; Table 2: the six projections are the dense
// contractions; Eq. 1, Eq. 3).
//
//   D[m, n] = sum_k A[m, k] * B[n, k]       A, B bf16 K-major, D f32 in TMEM
//
// CTA = 6 warps: warp 0 TMA producer, warp 1 MMA issuer (one elected lane)
// + TMEM owner, warps 2..5 epilogue (one TMEM lane quarter each, warp % 4).
// Tile 128 x BN x 64, multi-stage smem ring (full/empty mbarriers), two TMEM
// accumulators so the epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace eco {

static constexpr int BM = 128;
static constexpr int BK = 64;
static constexpr int GEMM_THREADS = 192;

// R = 128-row A tiles per work unit sharing one B tile (R = 2 in the decode GEMMs:
// two weight tiles per CTA stream behind one activation tile, so 2/3 of the staged
// bytes are weights instead of 1/2 -- more weight bytes in flight per SM).
// R = 3 selects the "lean" single-tile variant: 3 smem stages (< 114 KB of smem) so a
// CTA of the next kernel on the stream can be resident beside it -- with PDL its
// prologue and weight prefetch then overlap this kernel's tail.
// R = 4 selects split rings (decode): the weight (A) tiles and the activation (B) tiles
// get separate smem rings with their own barriers -- SA = 9-10 weight stages, SB = 3-4
// activation stages -- so ~150 KB of weights are in flight per SM instead of 96 KB. The
// activations come from L2 (short latency) and no longer take half of every stage.
template <int BN, int R = 1>
struct GemmCfg {
  static constexpr bool SPLIT = R == 4;
  static constexpr int RT = (R == 3 || R == 4) ? 1 : R;  // A tiles per unit
  static constexpr int A_BYTES = RT * BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // epilogue staging: half an accumulator tile in f32 (BN/2 tokens x 128 features) for
  // the bulk-store epilogues (BN <= 128, one A tile); otherwise just the argmax scratch
  static constexpr bool BULK_EPI = BN <= 128 && RT <= 2;
  // (argmax epilogue: 4 x BN (max, idx) + one padded [32][BM + 1] f32 chunk)
  static constexpr int ARGMAX_STG = 4 * BN * 8 + 32 * (BM + 1) * 4;
  static constexpr int STAGING = BULK_EPI ? ((BN / 2) * BM * 4 > ARGMAX_STG ? (BN / 2) * BM * 4 : ARGMAX_STG)
                                          : 4 * BN * 8;
  static constexpr int SMEM_MAX = 232448;  // 227 KB opt-in per CTA
  static constexpr int FIT = (SMEM_MAX - 1024 - 256 - STAGING) / STAGE_BYTES;
  static constexpr int STAGES = R == 3 ? 3 : FIT > 8 ? 8 : FIT;
  static constexpr int ACC_COLS = RT * BN;  // one accumulator stage
  static constexpr int TMEM_COLS = (2 * ACC_COLS) <= 32 ? 32 : (2 * ACC_COLS) <= 64 ? 64 : (2 * ACC_COLS) <= 128 ? 128
                                 : (2 * ACC_COLS) <= 256 ? 256 : 512;
  // split rings (R = 4)
  static constexpr int SB = BN >= 128 ? 3 : 4;
  static constexpr int BAR_BYTES = SPLIT ? 512 : 256;
  static constexpr int SA_FIT = (SMEM_MAX - 1024 - BAR_BYTES - STAGING - SB * B_BYTES) / A_BYTES;
  static constexpr int SA = SA_FIT > 12 ? 12 : SA_FIT;
  static constexpr int NA = SPLIT ? SA : STAGES;  // full/empty barrier pairs of the (A or A+B) ring
  static constexpr int NB = SPLIT ? SB : 0;       // ... of the B ring
  static constexpr int RING = SPLIT ? SA * A_BYTES + SB * B_BYTES : STAGES * STAGE_BYTES;
  static constexpr int SMEM = RING + STAGING + 1024 /*align*/ + BAR_BYTES /*barriers*/;
  static_assert((2 * NA + 2 * NB + 4) * 8 + 8 <= BAR_BYTES, "barriers fit");
  static_assert(4 * BN * 8 <= STAGING, "argmax scratch lives in the staging buffer");
  static_assert(2 * ACC_COLS <= 512, "two accumulator stages must fit the 512 TMEM columns");
};

__device__ __forceinline__ void trace_mark(const GemmEpi& e, int i) {
  if (e.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    e.trace[blockIdx.x * 16 + i] = t;
  }
}

// fast-math division: the IEEE "/" slow path (zero / tiny numerators) stalls the epilogue
__device__ __forceinline__ long long clk() { return clock64(); }
__device__ __forceinline__ void trace_put(const GemmEpi& e, int i, long long v) {
  if (e.trace) e.trace[blockIdx.x * 16 + i] = (unsigned long long)v;
}

// The producer's wait before its first dependent load. Normally the PDL wait for the
// previous kernel on the stream. With epi.flag_wait the GEMM instead waits until the flag
// reaches flag_epoch -- raised by an earlier kernel once its own inputs were complete
// (epi.flag_set) -- so it can run beside the kernel just before it (GemmEpi::flag_wait).
// With epi.flag_set, CTA 0 raises the flag once its PDL wait returned.
__device__ __forceinline__ void gemm_dep_wait(const GemmEpi& epi) {
  if (epi.flag_wait) {
    for (;;) {
      int v;
      asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(epi.flag_wait) : "memory");
      if (v >= epi.flag_epoch) break;
      __nanosleep(64);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // the TMA loads that follow
  } else {
    pdl_wait();
  }
  if (epi.flag_set && blockIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(epi.flag_set), "r"(epi.flag_epoch) : "memory");
  }
}

__device__ __forceinline__ float silu_f(float z) { return __fdividef(z, 1.f + __expf(-z)); }

// ---------------------------------------------------------------- epilogues
// Non-swapped: this thread owns output row `m` (token), columns n0..n0+31 in v[].
// 1/rms of row m from the per-(N tile) sums of squares a residual epilogue left (nrm_ss_in)
__device__ __forceinline__ float nrm_row_scale(const GemmEpi& e, int m) {
  if (!e.nrm_ss_in) return 1.f;
  float ss = 0.f;
  for (int t = 0; t < e.nrm_ss_n; ++t) ss += __ldcg(e.nrm_ss_in + (int64_t)t * e.nrm_ss_ld + m);
  return rsqrtf(ss * e.nrm_inv_h + e.nrm_eps);
}

// Prefill deferred RMSNorm (GemmEpi::nrm_*): a residual epilogue also writes
// h = bf16(x * gamma) and accumulates the row's sum of x^2 into *ssq; a consumer epilogue
// (QKV, SiLU) receives its row's 1/rms(x) as `scale`.
__device__ __forceinline__ void epi_rows(const GemmEpi& e, int m, int n0, int n_rows, const uint32_t (&v)[32],
                                         float scale = 1.f, float* ssq = nullptr) {
  float f[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]) * scale;
  const int ncols = min(32, n_rows - n0);
  switch (e.mode) {
    case EPI_F32: {
      float* o = reinterpret_cast<float*>(e.out) + (int64_t)m * e.ldo + n0;
      float* o2 = e.out2 ? e.out2 + (int64_t)m * e.ldo + n0 : nullptr;  // TP push (peer plane)
      if (ncols == 32) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 q4 = make_float4(f[i], f[i + 1], f[i + 2], f[i + 3]);
          *reinterpret_cast<float4*>(o + i) = q4;
          if (o2) *reinterpret_cast<float4*>(o2 + i) = q4;
        }
      } else {
        for (int i = 0; i < ncols; ++i) {
          o[i] = f[i];
          if (o2) o2[i] = f[i];
        }
      }
    } break;
    case EPI_BF16: {
      bf16* o = reinterpret_cast<bf16*>(e.out) + (int64_t)m * e.ldo + n0;
      if (ncols == 32) {
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(o + i) = make_uint4(pack_bf16x2(f[i], f[i + 1]), pack_bf16x2(f[i + 2], f[i + 3]),
                                                        pack_bf16x2(f[i + 4], f[i + 5]), pack_bf16x2(f[i + 6], f[i + 7]));
      } else {
        for (int i = 0; i < ncols; ++i) o[i] = __float2bfloat16_rn(f[i]);
      }
    } break;
    case EPI_RESID: {
      float* o = e.resid + (int64_t)m * e.ldr + n0;
      if (ncols == 32) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          float4 r = *reinterpret_cast<float4*>(o + i);
          r.x += f[i]; r.y += f[i + 1]; r.z += f[i + 2]; r.w += f[i + 3];
          *reinterpret_cast<float4*>(o + i) = r;
          f[i] = r.x; f[i + 1] = r.y; f[i + 2] = r.z; f[i + 3] = r.w;
        }
      } else {
        for (int i = 0; i < ncols; ++i) {
          o[i] += f[i];
          f[i] = o[i];
        }
      }
      if (e.nrm_h) {  // deferred RMSNorm: h = bf16(x * gamma), sum of x^2
        bf16* hd = e.nrm_h + (int64_t)m * e.nrm_ldh + n0;
        float sq = 0.f;
        if (ncols == 32) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            const uint4 gv = *reinterpret_cast<const uint4*>(e.nrm_gamma + n0 + i);
            *reinterpret_cast<uint4*>(hd + i) = make_uint4(
                pack_bf16x2(f[i] * bf16_lo(gv.x), f[i + 1] * bf16_hi(gv.x)),
                pack_bf16x2(f[i + 2] * bf16_lo(gv.y), f[i + 3] * bf16_hi(gv.y)),
                pack_bf16x2(f[i + 4] * bf16_lo(gv.z), f[i + 5] * bf16_hi(gv.z)),
                pack_bf16x2(f[i + 6] * bf16_lo(gv.w), f[i + 7] * bf16_hi(gv.w)));
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) sq += f[i] * f[i];
        } else {
          for (int i = 0; i < ncols; ++i) {
            hd[i] = __float2bfloat16_rn(f[i] * __bfloat162float(e.nrm_gamma[n0 + i]));
            sq += f[i] * f[i];
          }
        }
        if (ssq) *ssq += sq;
      }
    } break;
    case EPI_SILU: {  // rows of W_gu are interleaved (gate j, up j) -> output column n0/2 + j
      bf16* o = reinterpret_cast<bf16*>(e.out) + (int64_t)m * e.ldo + n0 / 2;
      uint32_t p[8];
#pragma unroll
      for (int j = 0; j < 16; j += 2)
        p[j / 2] = pack_bf16x2(silu_f(f[2 * j]) * f[2 * j + 1], silu_f(f[2 * j + 2]) * f[2 * j + 3]);
      if (ncols == 32) {
        *reinterpret_cast<uint4*>(o) = make_uint4(p[0], p[1], p[2], p[3]);
        *reinterpret_cast<uint4*>(o + 8) = make_uint4(p[4], p[5], p[6], p[7]);
      } else {
        for (int j = 0; j < ncols / 2; ++j) o[j] = __float2bfloat16_rn(silu_f(f[2 * j]) * f[2 * j + 1]);
      }
    } break;
    case EPI_QKV: {
      // 32 columns never straddle a head (D in {32, 64, 128, 256}, n0 % 32 == 0).
      const int D = e.head_dim, half = D / 2;
      const int qd = e.n_heads * D, kd = e.n_kv * D;
      const int p = e.pos[m];
      if (n0 < qd + kd) {
        const bool is_q = n0 < qd;
        const int head = is_q ? n0 / D : (n0 - qd) / D;
        const int j0 = (n0 % D) / 2;  // pair index of f[0]
        const float4* cs4 = reinterpret_cast<const float4*>(e.rope_cos + (int64_t)p * half + j0);
        const float4* sn4 = reinterpret_cast<const float4*>(e.rope_sin + (int64_t)p * half + j0);
        float cs[16], sn[16];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 c = __ldg(cs4 + q4), s = __ldg(sn4 + q4);
          cs[4 * q4] = c.x; cs[4 * q4 + 1] = c.y; cs[4 * q4 + 2] = c.z; cs[4 * q4 + 3] = c.w;
          sn[4 * q4] = s.x; sn[4 * q4 + 1] = s.y; sn[4 * q4 + 2] = s.z; sn[4 * q4 + 3] = s.w;
        }
        uint32_t lo[8], hi[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          float c0 = cs[j], s0 = sn[j], c1 = cs[j + 1], s1 = sn[j + 1];
          float a0 = f[2 * j], b0 = f[2 * j + 1], a1 = f[2 * j + 2], b1 = f[2 * j + 3];
          lo[j / 2] = pack_bf16x2(a0 * c0 - b0 * s0, a1 * c1 - b1 * s1);
          hi[j / 2] = pack_bf16x2(b0 * c0 + a0 * s0, b1 * c1 + a1 * s1);
        }
        bf16* dst;
        if (is_q) {
          dst = e.q_out + ((int64_t)m * e.n_heads + head) * D;
        } else {
          const int s = e.slot[m];
          dst = e.k_cache + (int64_t)(s >> 6) * e.blk_stride + ((int64_t)head * 64 + (s & 63)) * D;
        }
        *reinterpret_cast<uint4*>(dst + j0) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        *reinterpret_cast<uint4*>(dst + j0 + 8) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
        *reinterpret_cast<uint4*>(dst + half + j0) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(dst + half + j0 + 8) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
      } else {
        const int c = n0 - qd - kd;
        const int head = c / D, d0 = c % D;
        const int s = e.slot[m];
        bf16* dst = e.v_cache + (int64_t)(s >> 6) * e.blk_stride + ((int64_t)head * 64 + (s & 63)) * D + d0;
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(dst + i) = make_uint4(pack_bf16x2(f[i], f[i + 1]), pack_bf16x2(f[i + 2], f[i + 3]),
                                                          pack_bf16x2(f[i + 4], f[i + 5]), pack_bf16x2(f[i + 6], f[i + 7]));
      }
    } break;
    default:
      break;
  }
}

// Swapped (decode) epilogue: this thread owns feature `m` (TMEM lane), tokens n0..n0+31
// in f[]. Pair-interleaved rows (RoPE, SiLU) sit in adjacent lanes: exchange by shuffle,
// so every lane executes the shuffles before any bounds check.
__device__ __forceinline__ void epi_swap(const GemmEpi& e, int m, int m_rows, int n0, int n_rows, int lane,
                                         const float (&f_in)[32]) {
  const bool mv = m < m_rows;
  float f[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = f_in[i];
  if (e.rvec && e.mode == EPI_SWAP_QKV) {  // deferred RMSNorm (decode flow path)
#pragma unroll
    for (int i = 0; i < 32; ++i) f[i] *= (n0 + i < n_rows) ? e.rvec[n0 + i] : 0.f;
  }
  const int ncols = min(32, n_rows - n0);
  switch (e.mode) {
    case EPI_SWAP_BF16: {
      bf16* o = reinterpret_cast<bf16*>(e.out);
      if (mv)
        for (int i = 0; i < ncols; ++i) o[(int64_t)(n0 + i) * e.ldo + m] = __float2bfloat16_rn(f[i]);
    } break;
    case EPI_SWAP_RESID: {
      if (mv)
        for (int i = 0; i < ncols; ++i) e.resid[(int64_t)(n0 + i) * e.ldr + m] += f[i];
    } break;
    case EPI_SWAP_STORE: {
      if (mv) {
        for (int i = 0; i < ncols; ++i) e.resid[(int64_t)(n0 + i) * e.ldr + m] = f[i];
        if (e.out2)  // TP push: the peer's receive plane (a warp writes 128 contiguous bytes per token)
          for (int i = 0; i < ncols; ++i) e.out2[(int64_t)(n0 + i) * e.ldr + m] = f[i];
      }
    } break;
    case EPI_SWAP_SILU: {
      bf16* o = reinterpret_cast<bf16*>(e.out);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float up = __shfl_xor_sync(0xffffffffu, f[i], 1);
        if (mv && !(lane & 1) && i < ncols) o[(int64_t)(n0 + i) * e.ldo + m / 2] = __float2bfloat16_rn(silu_f(f[i]) * up);
      }
    } break;
    case EPI_SWAP_QKV: {
      const int D = e.head_dim, half = D / 2;
      const int qd = e.n_heads * D, kd = e.n_kv * D;
      const bool odd = lane & 1;
      if (m < qd + kd) {  // warp-uniform: 32 rows never straddle the q/k | v boundary (D % 32 == 0)
        const bool is_q = m < qd;
        const int head = is_q ? m / D : (m - qd) / D;
        const int j = (m % D) / 2;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float other = __shfl_xor_sync(0xffffffffu, f[i], 1);
          if (mv && i < ncols) {
            const int n = n0 + i;
            const int p = e.pos[n];
            const float c = e.rope_cos[(int64_t)p * half + j], s = e.rope_sin[(int64_t)p * half + j];
            // even lane holds x_j (a), odd lane holds x_{j+D/2} (b)
            const float a = odd ? other : f[i], b = odd ? f[i] : other;
            const float y = odd ? (b * c + a * s) : (a * c - b * s);
            bf16* dst;
            if (is_q) {
              dst = e.q_out + ((int64_t)n * e.n_heads + head) * D;
            } else {
              const int sl = e.slot[n];
              dst = e.k_cache + (int64_t)(sl >> 6) * e.blk_stride + ((int64_t)head * 64 + (sl & 63)) * D;
            }
            dst[odd ? j + half : j] = __float2bfloat16_rn(y);
          }
        }
      } else if (mv) {
        const int c = m - qd - kd;
        const int head = c / D, d = c % D;
        for (int i = 0; i < ncols; ++i) {
          const int sl = e.slot[n0 + i];
          e.v_cache[(int64_t)(sl >> 6) * e.blk_stride + ((int64_t)head * 64 + (sl & 63)) * D + d] =
              __float2bfloat16_rn(f[i]);
        }
      }
    } break;
    default:
      break;
  }
}

// The p-th work piece of this CTA: weight tile mt, token tile nt, K blocks [kb0, kb1),
// partial plane ks. Uniform split: unit w = blockIdx.x + p * gridDim.x of the
// (tile, split) grid. Balanced split (epi.sk_L > 0, one token tile): the tiles this CTA's
// chunk [c * L, (c + 1) * L) of the (tile, K block) sequence touches, in order.
struct GemmPieces {
  int n_work, splits, n_tiles, kb_total, kb_per, sk_L, sk_units;
  __device__ __forceinline__ bool get(int p, int& mt, int& nt, int& ks, int& kb0, int& kb1) const {
    if (sk_L > 0) {
      const int u0 = blockIdx.x * sk_L, u1 = min(sk_units, u0 + sk_L);
      const int t = u0 / kb_total + p;
      if (t * kb_total >= u1) return false;
      mt = t;
      nt = 0;
      kb0 = max(u0, t * kb_total) - t * kb_total;
      kb1 = min(u1, (t + 1) * kb_total) - t * kb_total;
      ks = blockIdx.x - (t * kb_total) / sk_L;
      return true;
    }
    const int w = blockIdx.x + p * gridDim.x;
    if (w >= n_work) return false;
    ks = w % splits;
    const int t = w / splits;
    mt = t / n_tiles;
    nt = t % n_tiles;
    kb0 = ks * kb_per;
    kb1 = min(kb_total, kb0 + kb_per);
    return true;
  }
};

template <int BN, int RV>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int m_rows,
                   int n_rows, int K, int splits, GemmEpi epi) {
  using C = GemmCfg<BN, RV>;
  constexpr int R = C::RT;  // 128-row A tiles per work unit
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + C::RING;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + C::STAGING);
  uint64_t* empty_bar = full_bar + C::NA;
  uint64_t* full_b = empty_bar + C::NA;   // split rings: the B ring's barriers
  uint64_t* empty_b = full_b + C::NB;
  uint64_t* tfull_bar = empty_b + C::NB;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_ptr = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int& s_last = *reinterpret_cast<int*>(tmem_base_ptr + 1);
  auto am_v = reinterpret_cast<float(*)[BN]>(staging);               // [4][BN] argmax scratch
  auto am_i = reinterpret_cast<int(*)[BN]>(staging + 4 * BN * 4);
  uint8_t* ring_b = smem + C::SA * C::A_BYTES;  // split rings: B ring after the SA weight stages

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m_tiles = (m_rows + BM * R - 1) / (BM * R);  // work units of R x 128 rows
  const int n_tiles = (n_rows + BN - 1) / BN;
  const int kb_total = (K + BK - 1) / BK;
  const int kb_per = (kb_total + splits - 1) / splits;
  const int n_work = m_tiles * n_tiles * splits;
  const GemmPieces pcs{n_work, splits, n_tiles, kb_total, kb_per, epi.sk_L, m_tiles * kb_total};
  // bulk-store epilogue: f32 partials / SiLU output with 16-byte aligned token rows
  const bool bulk_epi =
      C::BULK_EPI && (reinterpret_cast<uintptr_t>(epi.out) & 15) == 0 &&
      ((epi.mode == EPI_SWAP_F32 && m_rows % 4 == 0 && epi.ldo % 4 == 0) ||
       (epi.mode == EPI_SWAP_SILU && splits == 1 && m_rows % 16 == 0 && epi.ldo % 8 == 0));
  // ... whose staged token rows leave by async bulk copies (one per row, issued by one
  // thread each) instead of 16-byte st.global from 4 warps (epi.bulk_copy): the per-CTA
  // trace measured that copy-out at ~4700 cycles of the ~3.4 us epilogue tail
  // (profiles/r01_gemm_trace_epi.log), but the decode step got slower with it
  // (8B 7.95-8.02 vs 7.86-7.89 ms, profiles/r02_epi_bulk_copy_ab.jsonl)
  const bool bulk_copy = bulk_epi && !epi.out2 && epi.bulk_copy;

  if (threadIdx.x == 0) {
    trace_mark(epi, 0);  // CTA start
    for (int s = 0; s < C::NA; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < C::NB; ++s) {
      mbar_init(&full_b[s], 1);
      mbar_init(&empty_b[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
  }
  if (warp == 1) tmem_alloc(tmem_base_ptr, C::TMEM_COLS);
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_ptr;
  // prologue done (smem, barriers, TMEM, descriptor prefetch): let the next kernel launch.
  // Threads wait for the previous kernel (PDL) right before their first dependent access.
  pdl_trigger();
  if (threadIdx.x == 0) trace_mark(epi, 1);  // prologue done

  if (C::SPLIT && warp == 0) {
    // ------------------------------------------------------------ TMA producer (split rings)
    if (lane == 0) {
      // two cursors over this CTA's (work unit, K block) sequence: the weights run SA
      // iterations ahead of the MMA, the activations SB; the MMA of iteration j frees
      // weight slot j % SA and activation slot j % SB
      struct Cur {
        int w, kb, kb1, mt, nt;
      };
      auto next = [&](Cur& c) -> bool {
        if (c.kb >= 0 && c.kb + 1 < c.kb1) { ++c.kb; return true; }
        if (c.kb >= 0) c.w += gridDim.x;
        if (c.w >= n_work) return false;
        const int ks = c.w % splits, t = c.w / splits;
        c.mt = t / n_tiles;
        c.nt = t % n_tiles;
        c.kb = ks * kb_per;
        c.kb1 = min(kb_total, c.kb + kb_per);
        return true;
      };
      Cur ca{(int)blockIdx.x, -1, 0, 0, 0}, cb{(int)blockIdx.x, -1, 0, 0, 0};
      bool a_more = true, b_more = true;
      int na = 0, nb = 0;
      for (; na < C::SA && (a_more = next(ca)); ++na) {  // weights: before the PDL wait
        mbar_arrive_expect_tx(&full_bar[na], C::A_BYTES);
        tma_load_2d(smem + na * C::A_BYTES, &mapA, &full_bar[na], ca.kb * BK, ca.mt * BM);
      }
      gemm_dep_wait(epi);
      for (; nb < C::SB && (b_more = next(cb)); ++nb) {
        mbar_arrive_expect_tx(&full_b[nb], C::B_BYTES);
        tma_load_2d(ring_b + nb * C::B_BYTES, &mapB, &full_b[nb], cb.kb * BK, cb.nt * BN);
      }
      for (int j = 0; a_more || b_more; ++j) {
        if (a_more && (a_more = next(ca))) {
          const int s = j % C::SA;
          mbar_wait(&empty_bar[s], (j / C::SA) & 1);
          mbar_arrive_expect_tx(&full_bar[s], C::A_BYTES);
          tma_load_2d(smem + s * C::A_BYTES, &mapA, &full_bar[s], ca.kb * BK, ca.mt * BM);
        }
        if (b_more && (b_more = next(cb))) {
          const int s = j % C::SB;
          mbar_wait(&empty_b[s], (j / C::SB) & 1);
          mbar_arrive_expect_tx(&full_b[s], C::B_BYTES);
          tma_load_2d(ring_b + s * C::B_BYTES, &mapB, &full_b[s], cb.kb * BK, cb.nt * BN);
        }
      }
    }
  } else if (C::SPLIT && warp == 1) {
    // ------------------------------------------------------------ MMA issuer (split rings)
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int acc = 0, j = 0;
      uint32_t acc_phase = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const int ks = w % splits;
        const int kb0 = ks * kb_per, kb1 = min(kb_total, kb0 + kb_per);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
        for (int kb = kb0; kb < kb1; ++kb, ++j) {
          const int sa = j % C::SA, sb = j % C::SB;
          mbar_wait(&full_bar[sa], (j / C::SA) & 1);
          mbar_wait(&full_b[sb], (j / C::SB) & 1);
          tc_fence_after();
          const uint64_t da = umma_desc_sw128(smem_u32(smem + sa * C::A_BYTES));
          const uint64_t db = umma_desc_sw128(smem_u32(ring_b + sb * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc_mma_f16(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          tc_commit(&empty_bar[sa]);
          tc_commit(&empty_b[sb]);
        }
        tc_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // iteration cursor over this CTA's (work piece, K block) sequence
      int p = 0, kb = -1, kb1 = 0, mt = 0, nt = 0;
      auto next = [&]() -> bool {
        if (kb >= 0 && kb + 1 < kb1) { ++kb; return true; }
        if (kb >= 0) ++p;
        int ks_, kb0_;
        if (!pcs.get(p, mt, nt, ks_, kb0_, kb1)) return false;
        kb = kb0_;
        return true;
      };
      // 1) the operand that does not depend on the previous kernel (the weights) is
      //    streamed into the first stages before the PDL wait
      int pre_mt[8], pre_nt[8], pre_kb[8], npre = 0;
      const int indep = epi.indep;
      if (indep != 0) {
        while (npre < C::STAGES && next()) {
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
          if (indep == 1) tma_load_2d(sa, &mapA, &full_bar[stage], kb * BK, mt * BM * R);
          else tma_load_2d(sa + C::A_BYTES, &mapB, &full_bar[stage], kb * BK, nt * BN);
          pre_mt[npre] = mt; pre_nt[npre] = nt; pre_kb[npre] = kb;
          ++npre;
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        // 1b) decode: the weight K blocks beyond the smem ring into L2 (up to l2_pf_kb), so
        //     the previous kernel's tail (attention / reduction, SMs freeing up under PDL)
        //     also streams this GEMM's weights; the loads after the wait then hit L2
        if (indep == 1 && epi.l2_pf_kb > 0) {
          const int sw = p, skb = kb, skb1 = kb1, smt = mt, snt = nt;
          for (int n = 0; n < epi.l2_pf_kb && next(); ++n)
            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                             reinterpret_cast<uint64_t>(&mapA)),
                         "r"(kb * BK), "r"(mt * BM * R)
                         : "memory");
          p = sw; kb = skb; kb1 = skb1; mt = smt; nt = snt;  // rewind the cursor
        }
      }
      gemm_dep_wait(epi);
      // 2) their dependent operand
      for (int i = 0; i < npre; ++i) {
        uint8_t* sa = smem + i * C::STAGE_BYTES;
        if (indep == 1) tma_load_2d(sa + C::A_BYTES, &mapB, &full_bar[i], pre_kb[i] * BK, pre_nt[i] * BN);
        else tma_load_2d(sa, &mapA, &full_bar[i], pre_kb[i] * BK, pre_mt[i] * BM * R);
      }
      // 3) steady state
      while (next()) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * C::STAGE_BYTES;
        uint8_t* sb = sa + C::A_BYTES;
        mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
        tma_load_2d(sa, &mapA, &full_bar[stage], kb * BK, mt * BM * R);
        tma_load_2d(sb, &mapB, &full_bar[stage], kb * BK, nt * BN);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      trace_mark(epi, 6);  // last load issued
      // fill the HBM gap at the kernel boundary: the next GEMM's first weight stages -> L2
      if (epi.pf_map) {
        const int w2 = blockIdx.x;
        const int m_tiles2 = (epi.pf_m_rows + BM - 1) / BM;
        if (w2 < m_tiles2 * epi.pf_n_tiles * epi.pf_splits) {
          const int kb_total2 = (epi.pf_K + BK - 1) / BK;
          const int kb_per2 = (kb_total2 + epi.pf_splits - 1) / epi.pf_splits;
          const int ks2 = w2 % epi.pf_splits, mt2 = (w2 / epi.pf_splits) / epi.pf_n_tiles;
          const int kb0 = ks2 * kb_per2, kb1 = min(kb_total2, kb0 + min(kb_per2, epi.pf_kb));
          for (int k2 = kb0; k2 < kb1; ++k2)
            asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                             reinterpret_cast<uint64_t>(epi.pf_map)),
                         "r"(k2 * BK), "r"(mt2 * BM * R)
                         : "memory");
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      bool first = true;
      int mt_, nt_, ks_, kb0, kb1;
      for (int p = 0; pcs.get(p, mt_, nt_, ks_, kb0, kb1); ++p) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (first) { trace_mark(epi, 2); first = false; }  // first stage landed
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
          const uint64_t db = umma_desc_sw128(sb);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint64_t da = umma_desc_sw128(sa + r * BM * BK * 2);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // advance 16 bf16 = 32 B along K inside the 128 B swizzle row: +2 in 16-byte units
              tc_mma_f16(d_tmem + r * BN, da + 2 * k, db + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          tc_commit(&empty_bar[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      trace_mark(epi, 3);  // last MMA issued
    }
  } else {
    // ------------------------------------------------------------ epilogue
    if (!epi.flag_wait) pdl_wait();  // the epilogue reads/writes buffers of the previous kernels
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int ep_tid = (warp - 2) * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    int mt, nt, ks, kb0_, kb1_;
    for (int p = 0; pcs.get(p, mt, nt, ks, kb0_, kb1_); ++p) {
      const int t = mt * n_tiles + nt;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      if (threadIdx.x == 64) trace_mark(epi, 5);  // accumulator ready
      const int row = q * 32 + lane;  // accumulator row (TMEM lane)
      const int m = mt * BM * R + row;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * C::ACC_COLS;
      if (epi.mode == EPI_SWAP_ARGMAX && C::BULK_EPI && R == 1) {
        // per 32-token chunk: the 128 x 32 accumulator slice goes to smem transposed
        // ([token][row], padded row stride), then thread t scans rows 32*(t/32).. of token
        // t%32 -- 32 compares per thread instead of a 5-round shuffle argmax per token
        const int n_valid = min(BN, n_rows - nt * BN);
        float* stg = reinterpret_cast<float*>(staging + 4 * BN * 8);  // after am_v / am_i
        constexpr int LDS = BM + 1;
        const int tok = ep_tid & 31, qq = ep_tid >> 5;
        for (int c0 = 0; c0 < n_valid; c0 += 32) {  // warp-uniform
          uint32_t v[32];
          tmem_ld32(tbase + c0, v);
          tc_wait_ld();
          asm volatile("bar.sync 1, 128;" ::: "memory");  // previous chunk's scans are done
#pragma unroll
          for (int i = 0; i < 32; ++i) stg[i * LDS + row] = (m < m_rows) ? __uint_as_float(v[i]) : -INFINITY;
          asm volatile("bar.sync 1, 128;" ::: "memory");
          // rows in increasing order: ties keep the lowest index (reading A6); NaN wins
          const float* col = stg + tok * LDS + qq * 32;
          float bv = col[0];
          int bi = mt * BM + qq * 32;
#pragma unroll 8
          for (int r = 1; r < 32; ++r) {
            const float x = col[r];
            if (x > bv || (isnan(x) && !isnan(bv))) { bv = x; bi = mt * BM + qq * 32 + r; }
          }
          am_v[qq][c0 + tok] = bv;
          am_i[qq][c0 + tok] = bi;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int c = ep_tid; c < n_valid; c += 128) {
          const int n = nt * BN + c;
          float bv = am_v[0][c];
          int bi = am_i[0][c];
          for (int k = 1; k < 4; ++k) {
            const float ov = am_v[k][c];
            const int oi = am_i[k][c];
            if ((ov > bv) || (ov == bv && oi < bi) || (isnan(ov) && !isnan(bv))) { bv = ov; bi = oi; }
          }
          epi.am_val[(int64_t)n * epi.am_ld + mt] = bv;
          epi.am_idx[(int64_t)n * epi.am_ld + mt] = bi;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      } else if (epi.mode == EPI_SWAP_ARGMAX) {
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c0, v);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float val = (m < m_rows) ? __uint_as_float(v[i]) : -INFINITY;
            int idx = m;
            // warp argmax, lowest index on ties (reading A6); NaN propagates as "largest"
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              float ov = __shfl_xor_sync(0xffffffffu, val, off);
              int oi = __shfl_xor_sync(0xffffffffu, idx, off);
              bool take = (ov > val) || (ov == val && oi < idx) || (isnan(ov) && !isnan(val));
              if (take) { val = ov; idx = oi; }
            }
            if (lane == 0) { am_i[q][c0 + i] = idx; am_v[q][c0 + i] = val; }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int c = ep_tid; c < BN; c += 128) {
          const int n = nt * BN + c;
          if (n < n_rows) {
            float bv = am_v[0][c];
            int bi = am_i[0][c];
            for (int qq = 1; qq < 4; ++qq) {
              float ov = am_v[qq][c];
              int oi = am_i[qq][c];
              if ((ov > bv) || (ov == bv && oi < bi) || (isnan(ov) && !isnan(bv))) { bv = ov; bi = oi; }
            }
            epi.am_val[(int64_t)n * epi.am_ld + mt] = bv;
            epi.am_idx[(int64_t)n * epi.am_ld + mt] = bi;
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      } else if (C::BULK_EPI && bulk_epi) {
        // accumulator -> smem, transposed to [token][feature] -> 16-byte coalesced row
        // stores (instead of 128 scattered 4-byte stores per thread), half a tile at a time
        const bool silu = epi.mode == EPI_SWAP_SILU;
        constexpr int HALF = BN / 2;
        long long c_wr = 0, c_ld = 0, c_math = 0, c_out = 0, c0_ = 0;
#pragma unroll 1
        for (int rt = 0; rt < R; ++rt) {  // the unit's 128-row weight tiles (R = 2: one wave for gate/up)
          const int m0 = (mt * R + rt) * BM;
          const int mcount = max(0, min(BM, m_rows - m0));             // (R = 2: the 2nd tile may be empty)
          const int vec_per_row = silu ? mcount / 16 : mcount / 4;     // 16-byte vectors per token row
          const int stg_row = silu ? BM / 2 * 2 : BM * 4;              // staging row bytes
          char* gbase = silu ? reinterpret_cast<char*>(reinterpret_cast<bf16*>(epi.out) + m0 / 2)
                             : reinterpret_cast<char*>(reinterpret_cast<float*>(epi.out) +
                                                       (int64_t)ks * n_rows * epi.ldo + m0);
          const int64_t gstride = silu ? epi.ldo * 2 : epi.ldo * 4;
          // TP push (N2): the f32 partials also go to the peer's receive plane over NVLink
          char* gbase2 = (!silu && epi.out2) ? reinterpret_cast<char*>(epi.out2 + (int64_t)ks * n_rows * epi.ldo + m0)
                                             : nullptr;
          const uint32_t stg_base = smem_u32(staging);
          for (int h = 0; h < 2; ++h) {
            c0_ = clk();
            if (bulk_copy) bulk_wait_read0();  // this thread's row copies have read the staging
            asm volatile("bar.sync 1, 128;" ::: "memory");  // staging free (previous copy-out done)
            c_wr += clk() - c0_;
#pragma unroll 1
            for (int cc = 0; cc < HALF; cc += 32) {
              uint32_t v[32];
              c0_ = clk();
              tmem_ld32(tbase + rt * BN + h * HALF + cc, v);
              tc_wait_ld();
              const long long c1_ = clk();
              c_ld += c1_ - c0_;
              c0_ = c1_;
              if (silu) {
                // lanes 2j / 2j+1 hold gate_j / up_j; one exchange per token pair gives the
                // even lane (gate, up) of token i and the odd lane those of token i + 1
                const bool odd = lane & 1;
                const uint32_t sbase = stg_base + (uint32_t)(row / 2) * 2u;
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                  const float send = odd ? __uint_as_float(v[i]) : __uint_as_float(v[i + 1]);
                  const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                  const float g = odd ? recv : __uint_as_float(v[i]);
                  const float u = odd ? __uint_as_float(v[i + 1]) : recv;
                  const int tok = cc + i + (odd ? 1 : 0);
                  sts_u16(sbase + (uint32_t)(tok * stg_row), __bfloat16_as_ushort(__float2bfloat16_rn(silu_f(g) * u)));
                }
              } else {
                const uint32_t sbase = stg_base + (uint32_t)row * 4u;
#pragma unroll
                for (int i = 0; i < 32; ++i) sts_f32(sbase + (uint32_t)((cc + i) * stg_row), __uint_as_float(v[i]));
              }
              c_math += clk() - c0_;
            }
            c0_ = clk();
            if (h == 1 && rt == R - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty_bar[acc]);
            }
            if (bulk_copy) fence_proxy_async();  // this thread's st.shared -> the bulk copies
            asm volatile("bar.sync 1, 128;" ::: "memory");  // staging complete
            const int n0 = nt * BN + h * HALF;
            const int rows = max(0, min(HALF, n_rows - n0));
            if (bulk_copy) {
              if (ep_tid < rows && vec_per_row > 0) {
                bulk_store(gbase + (int64_t)(n0 + ep_tid) * gstride, staging + ep_tid * stg_row, vec_per_row * 16);
                bulk_commit();
              }
            } else {
              for (int idx = ep_tid; idx < rows * vec_per_row; idx += 128) {
                const int r = idx / vec_per_row, c = idx % vec_per_row;
                const uint4 val = lds128(stg_base + (uint32_t)(r * stg_row + c * 16));
                *reinterpret_cast<uint4*>(gbase + (int64_t)(n0 + r) * gstride + c * 16) = val;
                if (gbase2) *reinterpret_cast<uint4*>(gbase2 + (int64_t)(n0 + r) * gstride + c * 16) = val;
              }
            }
            c_out += clk() - c0_;
          }
        }
        if (bulk_copy) bulk_wait_read0();  // (the staging is reused by the next unit / freed at exit)
        if (threadIdx.x == 64) {
          trace_put(epi, 8, c_wr);
          trace_put(epi, 9, c_ld);
          trace_put(epi, 10, c_math);
          trace_put(epi, 11, c_out);
        }
      } else if (epi.mode == EPI_SWAP_F32) {
        float* out = reinterpret_cast<float*>(epi.out) + (int64_t)ks * n_rows * epi.ldo;
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
          const int mr = m + r * BM;
          for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + r * BN + c0, v);
            tc_wait_ld();
            if (mr < m_rows) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const int n = nt * BN + c0 + i;
                if (n < n_rows) out[(int64_t)n * epi.ldo + mr] = __uint_as_float(v[i]);
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      } else if (epi.mode >= EPI_SWAP_BF16) {
        if (splits == 1) {
#pragma unroll 1
          for (int r = 0; r < R; ++r) {
            for (int c0 = 0; c0 < BN; c0 += 32) {
              uint32_t v[32];
              tmem_ld32(tbase + r * BN + c0, v);
              tc_wait_ld();
              float f[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
              epi_swap(epi, m + r * BM, m_rows, nt * BN + c0, n_rows, lane, f);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        } else {
          // 1) this split's partial -> workspace (coalesced over the lanes = features)
          const int64_t plane = (int64_t)n_rows * m_rows;
          float* mine = epi.part + (int64_t)ks * plane;
          for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tbase + c0, v);
            tc_wait_ld();
            if (m < m_rows) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const int n = nt * BN + c0 + i;
                if (n < n_rows) mine[(int64_t)n * m_rows + m] = __uint_as_float(v[i]);
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[acc]);
          // 2) the last CTA to finish a split of this tile reduces all splits in split order
          __threadfence();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (ep_tid == 0) {
            const int old = atomicAdd(&epi.counters[t], 1);
            s_last = (old == splits - 1) ? 1 : 0;
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (s_last) {
            __threadfence();
            for (int c0 = 0; c0 < BN; c0 += 32) {
              float f[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) f[i] = 0.f;
              if (m < m_rows) {
                for (int s = 0; s < splits; ++s) {
                  const float* ps = epi.part + (int64_t)s * plane;
#pragma unroll
                  for (int i = 0; i < 32; ++i) {
                    const int n = nt * BN + c0 + i;
                    if (n < n_rows) f[i] += __ldcg(ps + (int64_t)n * m_rows + m);
                  }
                }
              }
              epi_swap(epi, m, m_rows, nt * BN + c0, n_rows, lane, f);
            }
            if (ep_tid == 0) epi.counters[t] = 0;
          }
        }
      } else {
        const float rsc = m < m_rows ? nrm_row_scale(epi, m) : 1.f;
        float ssq = 0.f;
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c0, v);
          tc_wait_ld();
          const int n0 = nt * BN + c0;
          if (m < m_rows && n0 < n_rows) epi_rows(epi, m, n0, n_rows, v, rsc, &ssq);
        }
        if (epi.nrm_ss_out && m < m_rows) epi.nrm_ss_out[(int64_t)nt * epi.nrm_ss_ld + m] = ssq;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (threadIdx.x == 64) trace_mark(epi, 4);  // (last) epilogue done
    }
    if (epi.out2) __threadfence_system();  // TP push complete before the grid ends
  }
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
  // a flag-gated GEMM did not wait for the kernel before it on the stream: it completes only
  // after that kernel does, so the kernels after it still see both (see GemmEpi::flag_wait)
  if (epi.flag_wait && threadIdx.x == 0) pdl_wait();
}

// ---------------------------------------------------------------- cluster split-K decode GEMM
// Swap-AB decode projection with its K range split over the S CTAs of one thread-block
// cluster (one 128-feature weight tile per cluster). The split partials are reduced
// through distributed shared memory instead of HBM: CTA `rank` owns the token columns
// [rank*CW, rank*CW + CW) of the tile; every CTA pushes the columns it does not own to
// their owner (st.shared::cluster, [slot][token][feature] f32) and release-arrives on
// the owner's mbarrier; the owner sums all S partials in rank order (the same order as
// the f32-partials reduction kernel, so results are bit-identical to it) and applies
// the epilogue (QKV RoPE + paged KV write, residual add, SiLU, bf16) to its columns.
// No partial buffer, no reduction kernel.
template <int BN, int S>
struct ClusterCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int CW = 16 * ((BN / 16 + S - 1) / S);  // token columns owned per rank
  static constexpr int RECV = (S - 1) * CW * BM * 4;
  static constexpr int FIT = (232448 - 1024 - 256 - RECV) / STAGE_BYTES;
  static constexpr int STAGES = FIT > 8 ? 8 : FIT;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + RECV + 1024 + 256;
};

template <int BN, int S>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_cluster_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                        int m_rows, int n_rows, int K, GemmEpi epi) {
  using C = ClusterCfg<BN, S>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* recv = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(recv + C::RECV);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* recv_full = tfull_bar + 1;
  uint32_t* tmem_base_ptr = reinterpret_cast<uint32_t*>(recv_full + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rank = blockIdx.x % S;  // == %cluster_ctarank (1-D clusters of S CTAs along x)
  const int tile = blockIdx.x / S;
  const int m_tiles = (m_rows + BM - 1) / BM;
  const int mt = tile % m_tiles, nt = tile / m_tiles;
  const int kb_total = (K + BK - 1) / BK;
  const int kb_per = (kb_total + S - 1) / S;
  const int kb0 = rank * kb_per, kb1 = min(kb_total, kb0 + kb_per);

  if (threadIdx.x == 0) {
    trace_mark(epi, 0);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(tfull_bar, 1);
    mbar_init(recv_full, (S - 1) * 128);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
  }
  if (warp == 1) tmem_alloc(tmem_base_ptr, C::TMEM_COLS);
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  cluster_sync();  // every CTA's barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_ptr;
  pdl_trigger();
  if (threadIdx.x == 0) trace_mark(epi, 1);

  if (warp == 0) {
    if (lane == 0) {
      // weights (independent of the previous kernel) into the first stages before the PDL wait
      const int n = kb1 - kb0;
      const int npre = min(n, C::STAGES);
      for (int i = 0; i < npre; ++i) {
        mbar_arrive_expect_tx(&full_bar[i], C::STAGE_BYTES);
        tma_load_2d(smem + i * C::STAGE_BYTES, &mapA, &full_bar[i], (kb0 + i) * BK, mt * BM);
      }
      pdl_wait();
      for (int i = 0; i < npre; ++i)
        tma_load_2d(smem + i * C::STAGE_BYTES + C::A_BYTES, &mapB, &full_bar[i], (kb0 + i) * BK, nt * BN);
      int stage = npre % C::STAGES;
      uint32_t phase = npre == C::STAGES ? 1 : 0;
      for (int i = npre; i < n; ++i) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * C::STAGE_BYTES;
        mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
        tma_load_2d(sa, &mapA, &full_bar[stage], (kb0 + i) * BK, mt * BM);
        tma_load_2d(sa + C::A_BYTES, &mapB, &full_bar[stage], (kb0 + i) * BK, nt * BN);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      trace_mark(epi, 6);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (kb == kb0) trace_mark(epi, 2);
        const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
        const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) tc_mma_f16(tmem_base, da + 2 * k, db + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
        tc_commit(&empty_bar[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      tc_commit(tfull_bar);
      trace_mark(epi, 3);
    }
  } else {
    pdl_wait();
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int m = mt * BM + row;
    const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16);
    const int n_base = nt * BN;
    const int n_valid = min(BN, n_rows - n_base);
    const uint32_t recv_u32 = smem_u32(recv);
    mbar_wait(tfull_bar, 0);
    tc_fence_after();
    if (threadIdx.x == 64) trace_mark(epi, 5);
    // 1) push the columns owned by the other ranks
#pragma unroll 1
    for (int o = 0; o < S; ++o) {
      if (o == rank) continue;
      const int lo = o * C::CW, hi = min(min(BN, lo + C::CW), n_valid);
      const int slot = rank < o ? rank : rank - 1;
      const uint32_t rb = mapa_u32(recv_u32 + (uint32_t)(slot * C::CW * BM * 4), (uint32_t)o);
      // receive layout [slot][token / 4][feature][4]: one 16-byte store per 4 tokens, a warp
      // writes 512 contiguous bytes (columns past `hi` are never read by the owner)
#pragma unroll 1
      for (int c = lo; c < hi; c += 16) {
        uint32_t v[16];
        tmem_ld16(tbase + c, v);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          if (c + i < hi)
            st_cluster_v4(rb + (uint32_t)((((c - lo + i) >> 2) * BM + row) * 16), __uint_as_float(v[i]),
                          __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
      }
      mbar_arrive_remote(mapa_u32(smem_u32(recv_full), (uint32_t)o));
    }
    // 2) own columns: sum the S partials in rank order, then the epilogue
    const int lo = rank * C::CW, hi = min(min(BN, lo + C::CW), n_valid);
    if (S > 1) mbar_wait_cluster(recv_full, 0);
#pragma unroll 1
    for (int c = lo; c < hi; c += 32) {
      float f[32];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (c + 16 * h < hi) {  // warp-uniform
          uint32_t v[16];
          tmem_ld16(tbase + c + 16 * h, v);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const int j = c + 16 * h + i - lo;  // token column within the owned range (multiple of 4)
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int s = 0; s < S; ++s) {
              float4 part;
              if (s == rank) {
                part = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                                   __uint_as_float(v[i + 3]));
              } else {
                const int slot = s < rank ? s : s - 1;
                part = lds_f32x4(recv_u32 + (uint32_t)(((slot * (C::CW / 4) + (j >> 2)) * BM + row) * 16));
              }
              acc.x += part.x;
              acc.y += part.y;
              acc.z += part.z;
              acc.w += part.w;
            }
            f[16 * h + i] = acc.x;
            f[16 * h + i + 1] = acc.y;
            f[16 * h + i + 2] = acc.z;
            f[16 * h + i + 3] = acc.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) f[16 * h + i] = 0.f;
        }
      }
      epi_swap(epi, m, m_rows, n_base + c, n_base + hi, lane, f);
    }
    if (threadIdx.x == 64) trace_mark(epi, 4);
  }
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int BN, int S>
static cudaError_t launch_cluster(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K,
                                  const GemmEpi& epi, cudaStream_t stream) {
  using C = ClusterCfg<BN, S>;
  cudaError_t e = ensure_smem(gemm_cluster_kernel<BN, S>, C::SMEM);
  if (e != cudaSuccess) return e;
  const int tiles = ((m_rows + BM - 1) / BM) * ((n_rows + BN - 1) / BN);
  if (tiles <= 0) return cudaSuccess;
  return launch_kc(gemm_cluster_kernel<BN, S>, dim3(tiles * S), dim3(GEMM_THREADS), C::SMEM, stream, S, *mapA, *mapB,
                   m_rows, n_rows, K, epi);
}

template <int BN, int S>
static int max_active_clusters() {
  using C = ClusterCfg<BN, S>;
  if (ensure_smem(gemm_cluster_kernel<BN, S>, C::SMEM) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(S * 64);
  cfg.blockDim = dim3(GEMM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_cluster_kernel<BN, S>, &cfg) != cudaSuccess) return 0;
  return n;
}

int gemm_cluster_max_active(int bn, int splits) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> cache;  // (device, key)
  int dev = 0;
  cudaGetDevice(&dev);
  const int key = bn * 10 + splits;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({dev, key});
  if (it != cache.end()) return it->second;
  int n = 0;
  switch (key) {
    case 642: n = max_active_clusters<64, 2>(); break;
    case 643: n = max_active_clusters<64, 3>(); break;
    case 644: n = max_active_clusters<64, 4>(); break;
    case 1282: n = max_active_clusters<128, 2>(); break;
    case 1283: n = max_active_clusters<128, 3>(); break;
    case 1284: n = max_active_clusters<128, 4>(); break;
    default: n = 0;
  }
  cache[{dev, key}] = n;
  return n;
}

cudaError_t gemm_cluster_launch(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K,
                                int bn, int splits, const GemmEpi& epi, cudaStream_t stream) {
  if (epi.mode < EPI_SWAP_BF16 || gemm_effective_splits(K, splits) != splits) return cudaErrorInvalidValue;
  const int key = bn * 10 + splits;
  switch (key) {
    case 642: return launch_cluster<64, 2>(mapA, mapB, m_rows, n_rows, K, epi, stream);
    case 643: return launch_cluster<64, 3>(mapA, mapB, m_rows, n_rows, K, epi, stream);
    case 644: return launch_cluster<64, 4>(mapA, mapB, m_rows, n_rows, K, epi, stream);
    case 1282: return launch_cluster<128, 2>(mapA, mapB, m_rows, n_rows, K, epi, stream);
    case 1283: return launch_cluster<128, 3>(mapA, mapB, m_rows, n_rows, K, epi, stream);
    case 1284: return launch_cluster<128, 4>(mapA, mapB, m_rows, n_rows, K, epi, stream);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------- CTA-pair GEMM
// cta_group::2 variant for the prefill projections: a cluster of 2 CTAs computes a
// 256 x 256 tile with one tcgen05.mma.cta_group::2 M=256 N=256 per 16-wide K step,
// issued by the even CTA. CTA r stages A rows [r*128, r*128+128) and B rows
// [r*128, r*128+128) of the tile (half the B traffic of a 1-CTA 128 x 256 tile per
// SM) and owns accumulator rows r*128.. in its TMEM (2 x 256 columns, double buffered).
// TMA completions land on the even CTA's full barriers; MMA completions are
// multicast to both CTAs' empty / tmem-full barriers; both CTAs' epilogues release
// the accumulator on the even CTA's tmem-empty barrier.
struct Gemm2Cfg {
  static constexpr int BN = 256;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = 6;
  static constexpr int TMEM_COLS = 512;
  static constexpr int PUSH_STG = 4 * 32 * 32 * 4;  // TP push staging, 16 KB (after the barriers)
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256 + PUSH_STG;
};

// Tile order of the persistent pair GEMM: bands of GM token panels (A), weight panels
// (B) advancing across a band, token panels fastest inside it. The ~74 tiles in flight
// then touch ~GM A panels and ~74/GM B panels, and each weight panel is read from HBM
// once per band instead of once per token panel (the gate/up prefill projection read
// 9 GB per launch with n-fastest order, 9x its operands; 1.5 GB with GM = 8). Less
// HBM traffic is less power: under sw_power_cap the SM clock, and with it this
// tensor-bound GEMM, rises (bench A/B on one box: GM 4 / 8 / 16 -> 42.9k / 43.7k /
// 44.0k tok/s; default 16, ECOSERVE_GEMM_BAND overrides).
__device__ __forceinline__ void tile_mn(int w, int m_tiles, int n_tiles, int GM, int& mt, int& nt) {
  const int band = w / (GM * n_tiles);
  const int m0 = band * GM;
  const int gm = min(GM, m_tiles - m0);
  const int r = w - band * GM * n_tiles;
  mt = m0 + r % gm;
  nt = r / gm;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int m_rows,
                    int n_rows, int K, GemmEpi epi) {
  using C = Gemm2Cfg;
  constexpr int BN = C::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_ptr = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rank = (int)cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
  const int m_tiles = (m_rows + 2 * BM - 1) / (2 * BM);
  const int n_tiles = (n_rows + BN - 1) / BN;
  const int kb_total = (K + BK - 1) / BK;
  const int n_work = m_tiles * n_tiles;
  const int band = epi.band > 0 ? epi.band : 16;  // token panels per band (tile_mn)
  // TP push epilogue (f32 output to this GPU and the peer): needs 16-byte aligned rows
  const bool push = epi.out2 && epi.mode == EPI_F32 && n_rows % 32 == 0 && epi.ldo % 4 == 0;
  uint8_t* push_stg = smem + C::STAGES * C::STAGE_BYTES + 256;  // [4 warps][32][32] f32, after the barriers

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 8);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
  }
  if (warp == 1) tmem_alloc2(tmem_base_ptr, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_ptr;
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int w = cid, kb = -1, mt = 0, nt = 0;
      auto next = [&]() -> bool {
        if (kb >= 0 && kb + 1 < kb_total) { ++kb; return true; }
        if (kb >= 0) w += ncl;
        if (w >= n_work) return false;
        tile_mn(w, m_tiles, n_tiles, band, mt, nt);
        kb = 0;
        return true;
      };
      const int arow = rank * BM, brow = rank * (BN / 2);
      int pre_mt[C::STAGES], pre_nt[C::STAGES], pre_kb[C::STAGES], npre = 0;
      const int indep = epi.indep;
      if (indep != 0) {
        while (npre < C::STAGES && next()) {
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * C::STAGE_BYTES);
          if (indep == 1) tma_load_2d_pair(sa, &mapA, &full_bar[stage], kb * BK, mt * 2 * BM + arow);
          else tma_load_2d_pair(sa + C::A_BYTES, &mapB, &full_bar[stage], kb * BK, nt * BN + brow);
          pre_mt[npre] = mt; pre_nt[npre] = nt; pre_kb[npre] = kb;
          ++npre;
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
      pdl_wait();
      for (int i = 0; i < npre; ++i) {
        uint8_t* sa = smem + i * C::STAGE_BYTES;
        if (indep == 1) tma_load_2d_pair(sa + C::A_BYTES, &mapB, &full_bar[i], pre_kb[i] * BK, pre_nt[i] * BN + brow);
        else tma_load_2d_pair(sa, &mapA, &full_bar[i], pre_kb[i] * BK, pre_mt[i] * 2 * BM + arow);
      }
      while (next()) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + stage * C::STAGE_BYTES;
        if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * C::STAGE_BYTES);
        tma_load_2d_pair(sa, &mapA, &full_bar[stage], kb * BK, mt * 2 * BM + arow);
        tma_load_2d_pair(sa + C::A_BYTES, &mapB, &full_bar[stage], kb * BK, nt * BN + brow);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int w = cid; w < n_work; w += ncl) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < kb_total; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc_mma_f16_pair(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb > 0 || k > 0) ? 1u : 0u);
          tc_commit_pair(&empty_bar[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit_pair(&tfull_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    pdl_wait();
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int w = cid; w < n_work; w += ncl) {
      int mt, nt;
      tile_mn(w, m_tiles, n_tiles, band, mt, nt);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int m = mt * 2 * BM + rank * BM + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (push) {
        // TP push (N2): this warp's 32 x 32 f32 block goes through smem (16-byte chunks
        // XOR-swizzled by row) so that every store instruction writes 4 token rows x 128
        // contiguous bytes -- to this GPU's receive plane and over NVLink to the peer's
        const int m_w = mt * 2 * BM + rank * BM + q * 32;
        const uint32_t stg = smem_u32(push_stg) + (uint32_t)(q * 4096);
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c0, v);
          tc_wait_ld();
#pragma unroll
          for (int c = 0; c < 8; ++c)
            sts128(stg + (uint32_t)(lane * 128 + ((c ^ (lane & 7)) * 16)),
                   make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]));
          __syncwarp();
          const int n0 = nt * BN + c0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int rr = 4 * j + (lane >> 3), cc = lane & 7;
            const uint4 val = lds128(stg + (uint32_t)(rr * 128 + ((cc ^ (rr & 7)) * 16)));
            if (m_w + rr < m_rows && n0 < n_rows) {
              const int64_t off = (int64_t)(m_w + rr) * epi.ldo + n0 + 4 * cc;
              *reinterpret_cast<uint4*>(reinterpret_cast<float*>(epi.out) + off) = val;
              *reinterpret_cast<uint4*>(epi.out2 + off) = val;
            }
          }
          __syncwarp();
        }
      } else {
        const float rsc = m < m_rows ? nrm_row_scale(epi, m) : 1.f;
        float ssq = 0.f;
        for (int c0 = 0; c0 < BN; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tbase + c0, v);
          tc_wait_ld();
          const int n0 = nt * BN + c0;
          if (m < m_rows && n0 < n_rows) epi_rows(epi, m, n0, n_rows, v, rsc, &ssq);
        }
        if (epi.nrm_ss_out && m < m_rows) epi.nrm_ss_out[(int64_t)nt * epi.nrm_ss_ld + m] = ssq;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_peer0(&tempty_bar[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (push) __threadfence_system();  // TP push complete before the grid ends
  }
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc2(tmem_base, C::TMEM_COLS);
  }
}

cudaError_t gemm2_launch(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K,
                         const GemmEpi& epi_in, int num_sms, cudaStream_t stream) {
  static int band_env = -1;  // ECOSERVE_GEMM_BAND: token panels per band of the tile order (default 16)
  if (band_env < 0) {
    const char* ev = getenv("ECOSERVE_GEMM_BAND");
    band_env = ev ? atoi(ev) : 0;
  }
  GemmEpi epi = epi_in;
  if (epi.band <= 0) epi.band = band_env;
  if (epi.mode >= EPI_SWAP_F32) return cudaErrorInvalidValue;  // prefill (non-swapped) epilogues only
  cudaError_t e = ensure_smem(gemm_tc2_kernel, Gemm2Cfg::SMEM);
  if (e != cudaSuccess) return e;
  const int work = ((m_rows + 255) / 256) * ((n_rows + 255) / 256);
  int clusters = num_sms / 2;
  if (work < clusters) clusters = work;
  if (clusters <= 0) return cudaSuccess;
  return launch_k(gemm_tc2_kernel, dim3(2 * clusters), dim3(GEMM_THREADS), Gemm2Cfg::SMEM, stream, *mapA, *mapB,
                  m_rows, n_rows, K, epi);
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  auto enc = get_encode();
  if (!enc) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

int make_tmap_2d_plain(CUtensorMap* map, const void* ptr, int f32, int64_t rows, int64_t cols, int box_cols,
                       int box_rows) {
  auto enc = get_encode();
  if (!enc) return -1;
  const int esz = f32 ? 4 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * esz};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

int make_tmap_bf16_nd(CUtensorMap* map, const void* ptr, int rank, const int64_t* dims, const int64_t* strides_bytes,
                      const int* box) {
  auto enc = get_encode();
  if (!enc || rank < 1 || rank > 5) return -1;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = (cuuint64_t)dims[i];
    b[i] = (cuuint32_t)box[i];
    e[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) s[i] = (cuuint64_t)strides_bytes[i];
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr), d, s, b, e,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

int gemm_effective_splits(int K, int splits) {
  // every split must own at least one K block (an empty split would publish an unwritten accumulator)
  const int kb_total = (K + BK - 1) / BK;
  if (splits > kb_total) splits = kb_total;
  if (splits < 1) splits = 1;
  const int kb_per = (kb_total + splits - 1) / splits;
  return (kb_total + kb_per - 1) / kb_per;
}

int gemm_choose_splits(int m_rows, int n_rows, int K, int bn, int num_sms, int max_splits) {
  const int tiles = ((m_rows + BM - 1) / BM) * ((n_rows + bn - 1) / bn);
  const int kb_total = (K + BK - 1) / BK;
  int best = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= max_splits; ++s) {
    const int eff = gemm_effective_splits(K, s);
    if (eff != s && s > 1) continue;
    const int kb_per = (kb_total + eff - 1) / eff;
    const int waves = (tiles * eff + num_sms - 1) / num_sms;
    // K blocks streamed by the busiest CTA, plus ~1 block-equivalent per split for the reduction
    const double cost = (double)waves * kb_per + (eff > 1 ? 0.5 * eff : 0.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = eff;
    }
  }
  return best;
}

// Split-K factor of a swap-AB decode projection (one 128-row weight tile per work unit,
// one CTA per SM): the s in 1..4 with the fewest K blocks streamed by the busiest CTA
// (waves x K blocks per split), plus ~half a block per split for the reduction. This
// matches the measured sweep on the 8B shapes (QKV 3, O 4, down 4) and avoids
// the 160-unit second wave the old "tiles x s ~ SMs" rule gave the 70B/TP=2 QKV (40 tiles).
int gemm_decode_splits(int m_rows, int K, int num_sms) {
  const int tiles = (m_rows + BM - 1) / BM;
  // tiles covering >= 3/4 of the SMs run unsplit: their epilogue (SiLU, LM-head argmax)
  // stays in the GEMM, which the sweep measured faster than partials + a reduction
  if (4 * tiles >= 3 * num_sms) return 1;
  const int kb_total = (K + BK - 1) / BK;
  int best = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= 4; ++s) {
    const int eff = gemm_effective_splits(K, s);
    if (eff != s) continue;
    const int kb_per = (kb_total + eff - 1) / eff;
    const int waves = (tiles * eff + num_sms - 1) / num_sms;
    const double cost = (double)waves * kb_per + (eff > 1 ? 0.5 * eff : 0.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = eff;
    }
  }
  return best;
}

int gemm_sk_chunk(int m_tiles, int kbt, int num_sms, int max_slots) {
  const int U = m_tiles * kbt;
  if (m_tiles <= 0 || kbt <= 0 || m_tiles >= num_sms) return 0;
  for (int L = (U + num_sms - 1) / num_sms; L <= kbt; ++L) {
    int mx = 0;
    for (int t = 0; t < m_tiles; ++t) mx = std::max(mx, sk_slots(t, kbt, L));
    if (mx <= max_slots) return L;
  }
  return 0;
}

int gemm_smem_bytes(int bn) {
  switch (bn) {
    case 64: return GemmCfg<64, 1>::SMEM;
    case 128: return GemmCfg<128, 1>::SMEM;
    default: return GemmCfg<256, 1>::SMEM;
  }
}

template <int BN, int R>
static cudaError_t launch_bn(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K,
                             int splits, const GemmEpi& epi, int num_sms, cudaStream_t stream) {
  using C = GemmCfg<BN, R>;
  cudaError_t e = ensure_smem(gemm_tc_kernel<BN, R>, C::SMEM);
  if (e != cudaSuccess) return e;
  const int m_tiles = (m_rows + BM * C::RT - 1) / (BM * C::RT), n_tiles = (n_rows + BN - 1) / BN;
  const int work = m_tiles * n_tiles * splits;
  int grid = work < num_sms ? work : num_sms;
  if (epi.sk_L > 0) grid = (m_tiles * epi.sk_kbt + epi.sk_L - 1) / epi.sk_L;  // one chunk per CTA
  if (grid <= 0) return cudaSuccess;
  return launch_k(gemm_tc_kernel<BN, R>, dim3(grid), dim3(GEMM_THREADS), C::SMEM, stream, *mapA, *mapB, m_rows,
                  n_rows, K, splits, epi);
}

cudaError_t gemm_launch_r(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K, int bn,
                          int r, int splits, const GemmEpi& epi, int num_sms, cudaStream_t stream) {
  if (splits < 1) return cudaErrorInvalidValue;
  if (epi.sk_L > 0 && (epi.mode != EPI_SWAP_F32 || r != 1 || splits != 1 || n_rows > bn ||
                       epi.sk_kbt != (K + BK - 1) / BK ||
                       (int64_t)((m_rows + BM - 1) / BM) * epi.sk_kbt > (int64_t)epi.sk_L * num_sms))
    return cudaErrorInvalidValue;
  if (splits > 1 && epi.mode != EPI_SWAP_F32 && epi.mode < EPI_SWAP_BF16) return cudaErrorInvalidValue;
  if (splits > 1 && epi.mode >= EPI_SWAP_BF16 && (!epi.part || !epi.counters)) return cudaErrorInvalidValue;
  splits = gemm_effective_splits(K, splits);
  if (r == 2) {
    // two weight tiles per unit: swapped epilogues without the in-kernel split reduction
    if (epi.mode != EPI_SWAP_F32 && !(epi.mode >= EPI_SWAP_BF16 && splits == 1)) return cudaErrorInvalidValue;
    switch (bn) {
      case 64: return launch_bn<64, 2>(mapA, mapB, m_rows, n_rows, K, splits, epi, num_sms, stream);
      case 128: return launch_bn<128, 2>(mapA, mapB, m_rows, n_rows, K, splits, epi, num_sms, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  if (r == 4) {  // split weight / activation rings (decode)
    switch (bn) {
      case 64: return launch_bn<64, 4>(mapA, mapB, m_rows, n_rows, K, splits, epi, num_sms, stream);
      case 128: return launch_bn<128, 4>(mapA, mapB, m_rows, n_rows, K, splits, epi, num_sms, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  if (r == 3) {  // lean single-tile variant (co-resident with the next kernel's CTA)
    switch (bn) {
      case 64: return launch_bn<64, 3>(mapA, mapB, m_rows, n_rows, K, splits, epi, num_sms, stream);
      case 128: return launch_bn<128, 3>(mapA, mapB, m_rows, n_rows, K, splits, epi, num_sms, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  if (r != 1) return cudaErrorInvalidValue;
  switch (bn) {
    case 64: return launch_bn<64, 1>(mapA, mapB, m_rows, n_rows, K, splits, epi, num_sms, stream);
    case 128: return launch_bn<128, 1>(mapA, mapB, m_rows, n_rows, K, splits, epi, num_sms, stream);
    case 256: return launch_bn<256, 1>(mapA, mapB, m_rows, n_rows, K, splits, epi, num_sms, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t gemm_launch(const CUtensorMap* mapA, const CUtensorMap* mapB, int m_rows, int n_rows, int K, int bn,
                        int splits, const GemmEpi& epi, int num_sms, cudaStream_t stream) {
  return gemm_launch_r(mapA, mapB, m_rows, n_rows, K, bn, 1, splits, epi, num_sms, stream);
}

// ---------------------------------------------------------------- decode layer chain
// (kernels.h: ChainStep). One CTA per SM with the 1-CTA GEMM's warp roles (warp 0 TMA
// producer, warp 1 MMA issuer, warps 2..5 epilogue); the smem ring and the two TMEM
// accumulators carry over from one GEMM step to the next.
using ChainCfg = GemmCfg<128, 1>;
constexpr int CH_SILU_STG = 0;                 // [64 tok][128 B] SiLU output staging
constexpr int CH_RVEC = 64 * 128;              // [512] f32 RMSNorm scales of the step's tokens
constexpr int CH_RED = CH_RVEC + 512 * 4;      // [4 warps][32] f32 sum-of-squares partials
constexpr int CH_FLAG = CH_RED + 4 * 32 * 4;   // last-arriver flag
static_assert(CH_FLAG + 16 <= ChainCfg::STAGING, "chain scratch fits the staging buffer");

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until the barrier counter reaches `target`. A grid that is not co-resident (another
// kernel holding SMs) would wait forever: after 2 s flag the error and fall through.
__device__ __noinline__ void chain_grid_wait(const ChainCall& c, unsigned long long target) {
  if (ld_acquire_u64(c.bar) >= target) return;
  const unsigned long long t0 = gtime_ns();
  while (ld_acquire_u64(c.bar) < target) {
    if (*reinterpret_cast<volatile int*>(c.err)) return;
    __nanosleep(32);
    if (gtime_ns() - t0 > 2000000000ull) {
      atomicExch(c.err, 1);
      return;
    }
  }
}

// stream-K partition of T flattened iterations over G CTAs
__device__ __forceinline__ long long sk_begin(int c, long long T, int G) { return (long long)c * T / G; }
__device__ __forceinline__ int sk_cta_of(long long i, long long T, int G) { return (int)(((i + 1) * G - 1) / T); }

// 32 values per lane -> lane i holds the sum over the warp's lanes of value i (31 shuffles)
__device__ __forceinline__ float warp_transpose_sum(float (&v)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool hi = lane & off;
#pragma unroll
    for (int j = 0; j < off; ++j) {
      const float send = hi ? v[j] : v[j + off];
      const float keep = hi ? v[j + off] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}


// 32 accumulator columns (tokens c0..c0+31 of the tile) of this thread's TMEM lane, or --
// for a tile split between CTAs -- of the tile's f32 sum that the CTAs accumulated in
// `acc_tile` ([128 tok][128 m]); the reader (the last CTA) zeroes it for the next use.
__device__ __forceinline__ void chain_src(bool from_ws, float* acc_tile, uint32_t tbase, int c0, int row, int n_valid,
                                          float (&f)[32]) {
  if (!from_ws) {
    uint32_t v[32];
    tmem_ld32(tbase + c0, v);
    tc_wait_ld();
#pragma unroll
    for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
    return;
  }
  float* src = acc_tile + (int64_t)c0 * 128 + row;
#pragma unroll
  for (int i = 0; i < 32; ++i) f[i] = (c0 + i < n_valid) ? __ldcg(src + i * 128) : 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (c0 + i < n_valid) src[i * 128] = 0.f;
}

__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    decode_chain_kernel(const ChainStep* __restrict__ steps, int n_steps, ChainCall call) {
  using C = ChainCfg;
  constexpr int BN = 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* staging = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + C::STAGING);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_ptr = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_tok = call.n_tok;
  const int n_tiles = (n_tok + BN - 1) / BN;
  const unsigned long long grid = gridDim.x;
  const int G = gridDim.x, me = blockIdx.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_base_ptr, C::TMEM_COLS);
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_ptr;
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int si = 0; si < n_steps; ++si) {
        const ChainStep& S = steps[si];
        const CUtensorMap* wm = S.wmap;
        const CUtensorMap* xm = S.xmap;
        const int kpt = (S.K + BK - 1) / BK;
        const long long T = (long long)((S.m_rows + BM - 1) / BM) * n_tiles * kpt;
        const long long i0 = sk_begin(me, T, G), i1 = sk_begin(me + 1, T, G);
        // 1) weights (independent of the previous steps) into free stages
        int pre_st[C::STAGES], pre_kb[C::STAGES], pre_nt[C::STAGES], npre = 0;
        long long i = i0;
        for (; i < i1 && npre < C::STAGES; ++i) {
          const int t = (int)(i / kpt), kb = (int)(i % kpt);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
          tma_load_2d(smem + stage * C::STAGE_BYTES, wm, &full_bar[stage], kb * BK, (t / n_tiles) * BM);
          pre_st[npre] = stage; pre_kb[npre] = kb; pre_nt[npre] = t % n_tiles;
          ++npre;
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        // 2) the activations: produced by the previous step on every CTA
        if (si == 0) pdl_wait();
        else chain_grid_wait(call, call.bar_base + (unsigned long long)si * grid);
        if (call.trace) call.trace[(me * 32 + si) * 4 + 0] = gtime_ns();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        for (int k = 0; k < npre; ++k)
          tma_load_2d(smem + pre_st[k] * C::STAGE_BYTES + C::A_BYTES, xm, &full_bar[pre_st[k]], pre_kb[k] * BK,
                      pre_nt[k] * BN);
        // 3) steady state
        for (; i < i1; ++i) {
          const int t = (int)(i / kpt), kb = (int)(i % kpt);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
          tma_load_2d(sa, wm, &full_bar[stage], kb * BK, (t / n_tiles) * BM);
          tma_load_2d(sa + C::A_BYTES, xm, &full_bar[stage], kb * BK, (t % n_tiles) * BN);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int si = 0; si < n_steps; ++si) {
        const ChainStep& S = steps[si];
        const int kpt = (S.K + BK - 1) / BK;
        const long long T = (long long)((S.m_rows + BM - 1) / BM) * n_tiles * kpt;
        const long long i1 = sk_begin(me + 1, T, G);
        for (long long j = sk_begin(me, T, G); j < i1;) {  // one segment = this CTA's part of one tile
          const long long seg_end = min(i1, (j / kpt + 1) * kpt);
          mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
          for (long long jj = j; jj < seg_end; ++jj) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
            const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              tc_mma_f16(d_tmem, da + 2 * k, db + 2 * k, idesc, (jj > j || k > 0) ? 1u : 0u);
            tc_commit(&empty_bar[stage]);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          tc_commit(&tfull_bar[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          j = seg_end;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogues
    if (call.trace && threadIdx.x == 64) call.trace[(me * 32 + 0) * 4 + 3] = gtime_ns();  // CTA start
    pdl_wait();
    const int q = warp & 3;
    const int ep_tid = (warp - 2) * 32 + lane;
    const int row = q * 32 + lane;  // accumulator row (TMEM lane)
    const uint32_t stg_base = smem_u32(staging + CH_SILU_STG);
    float* rvec = reinterpret_cast<float*>(staging + CH_RVEC);
    float* red = reinterpret_cast<float*>(staging + CH_RED);
    int* s_last = reinterpret_cast<int*>(staging + CH_FLAG);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int si = 0; si < n_steps; ++si) {
      const ChainStep& S = steps[si];
      const int mode = S.mode;
      const int m_rows = S.m_rows;
      const int kpt = (S.K + BK - 1) / BK;
      const long long T = (long long)((m_rows + BM - 1) / BM) * n_tiles * kpt;
      // the step's inputs (previous steps of every CTA) are in memory
      if (si > 0) {
        if (ep_tid == 0) chain_grid_wait(call, call.bar_base + (unsigned long long)si * grid);
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      if (mode != CE_RESID_SS) {  // the RMSNorm scale of every token of the step
        for (int n = ep_tid; n < n_tok; n += 128) {
          float ssum = 0.f;
          for (int t = 0; t < S.ssp_tiles; ++t) ssum += __ldcg(S.ssp_in + (int64_t)t * call.ss_ld + n);
          rvec[n] = rsqrtf(ssum / S.H + S.eps);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      GemmEpi eq;
      if (mode == CE_QKV_R) {
        eq = S.e;
        eq.pos = call.pos;
        eq.slot = call.slot;
      }
      const long long i1 = sk_begin(me + 1, T, G);
      const int first_tile = (int)(sk_begin(me, T, G) / kpt);
      for (long long j = sk_begin(me, T, G); j < i1;) {
        const int t = (int)(j / kpt);
        const long long seg_end = min(i1, (long long)(t + 1) * kpt);
        const int mt = t / n_tiles, nt = t % n_tiles;
        const int n_valid = min(BN, n_tok - nt * BN);  // tokens of this tile
        bool from_ws = false;
        float* acc_tile = call.ws + (int64_t)t * 128 * 128;
        const bool full = j == (long long)t * kpt && seg_end == (long long)(t + 1) * kpt;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        if (call.trace && ep_tid == 0 && j == sk_begin(me, T, G)) call.trace[(me * 32 + si) * 4 + 1] = gtime_ns();
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * C::ACC_COLS;
        bool run_epi = full;
        if (!full) {
          // partial tile: this CTA's K range is added (f32 atomics in L2) to the tile's sum --
          // for the residual modes straight into x -- and the last CTA to arrive finishes it
          const int m = mt * BM + row;
          for (int c0 = 0; c0 < n_valid; c0 += 32) {  // warp-uniform
            uint32_t v[32];
            tmem_ld32(tbase + c0, v);
            tc_wait_ld();
            if (m < m_rows) {
              if (mode == CE_RESID_SS) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (c0 + i < n_valid) red_add_f32(S.x + (int64_t)(nt * BN + c0 + i) * m_rows + m, __uint_as_float(v[i]));
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (c0 + i < n_valid) red_add_f32(acc_tile + (int64_t)(c0 + i) * 128 + row, __uint_as_float(v[i]));
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[acc]);
          const int c_lo = sk_cta_of((long long)t * kpt, T, G), c_hi = sk_cta_of((long long)(t + 1) * kpt - 1, T, G);
          int nseg = 0;  // CTAs with a non-empty part of the tile
          for (int c = c_lo; c <= c_hi; ++c) nseg += sk_begin(c + 1, T, G) > sk_begin(c, T, G) ? 1 : 0;
          __threadfence();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (ep_tid == 0) {
            const int old = atomicAdd(&S.counters[t], 1);
            *s_last = old == nseg - 1;
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
          run_epi = *s_last != 0;
          if (run_epi) {
            __threadfence();
            from_ws = true;
            if (ep_tid == 0) S.counters[t] = 0;
          }
        }
        if (run_epi) {
          const int m = mt * BM + row;
          const bool mv = m < m_rows;
          if (mode == CE_SILU_R) {
            // SiLU(gate) * up with the RMSNorm scale, staged to 16-byte coalesced token rows
            constexpr int HALF = BN / 2;
            const int mcount = min(BM, m_rows - mt * BM);
            const int vec_per_row = mcount / 16;
            char* gbase = reinterpret_cast<char*>(reinterpret_cast<bf16*>(S.e.out) + mt * BM / 2);
            const int64_t gstride = S.e.ldo * 2;
            for (int hh = 0; hh < 2; ++hh) {
              asm volatile("bar.sync 1, 128;" ::: "memory");  // staging free
#pragma unroll 1
              for (int cc = 0; cc < HALF; cc += 32) {
                float f[32];
                chain_src(from_ws, acc_tile, tbase, hh * HALF + cc, row, n_valid, f);
                const bool odd = lane & 1;
                const uint32_t sbase = stg_base + (uint32_t)(row / 2) * 2u;
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                  const int n = nt * BN + hh * HALF + cc + i;
                  const float r0 = n < n_tok ? rvec[n] : 0.f, r1 = n + 1 < n_tok ? rvec[n + 1] : 0.f;
                  const float send = odd ? f[i] * r0 : f[i + 1] * r1;
                  const float recv = __shfl_xor_sync(0xffffffffu, send, 1);
                  const float g = odd ? recv : f[i] * r0;
                  const float u = odd ? f[i + 1] * r1 : recv;
                  const int tok = cc + i + (odd ? 1 : 0);
                  sts_u16(sbase + (uint32_t)(tok * 128), __bfloat16_as_ushort(__float2bfloat16_rn(silu_f(g) * u)));
                }
              }
              if (hh == 1 && !from_ws) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty_bar[acc]);
              }
              asm volatile("bar.sync 1, 128;" ::: "memory");  // staging complete
              const int n0 = nt * BN + hh * HALF;
              const int rows = min(HALF, n_tok - n0);
              for (int idx = ep_tid; idx < rows * vec_per_row; idx += 128) {
                const int r = idx / vec_per_row, cv = idx % vec_per_row;
                const uint4 val = lds128(stg_base + (uint32_t)(r * 128 + cv * 16));
                *reinterpret_cast<uint4*>(gbase + (int64_t)(n0 + r) * gstride + cv * 16) = val;
              }
            }
          } else {
            for (int c0 = 0; c0 < BN; c0 += 32) {
              const int n0 = nt * BN + c0;
              if (n0 >= n_tok) break;  // block-uniform
              float f[32];
              if (mode == CE_RESID_SS && from_ws) {
#pragma unroll
                for (int i = 0; i < 32; ++i) f[i] = 0.f;  // the partials are already in x
              } else {
                chain_src(from_ws, acc_tile, tbase, c0, row, n_valid, f);
              }
              if (mode == CE_RESID_SS) {
                float xv[32];
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  xv[i] = (mv && n0 + i < n_tok) ? __ldcg(S.x + (int64_t)(n0 + i) * m_rows + m) : 0.f;
                const float gm = mv ? __bfloat162float(S.gamma[m]) : 0.f;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                  xv[i] += f[i];
                  if (mv && n0 + i < n_tok) {
                    S.x[(int64_t)(n0 + i) * m_rows + m] = xv[i];
                    S.hb[(int64_t)(n0 + i) * m_rows + m] = __float2bfloat16_rn(xv[i] * gm);
                  }
                  xv[i] = (mv && n0 + i < n_tok) ? xv[i] * xv[i] : 0.f;
                }
                const float wsum = warp_transpose_sum(xv, lane);  // token n0 + lane, this warp's 32 rows
                red[q * 32 + lane] = wsum;
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (ep_tid < 32 && n0 + ep_tid < n_tok)  // fixed order over the 4 row quarters
                  S.ssp_out[(int64_t)mt * call.ss_ld + n0 + ep_tid] =
                      ((red[ep_tid] + red[32 + ep_tid]) + red[64 + ep_tid]) + red[96 + ep_tid];
                asm volatile("bar.sync 1, 128;" ::: "memory");
              } else {  // CE_QKV_R
#pragma unroll
                for (int i = 0; i < 32; ++i) f[i] *= (n0 + i < n_tok) ? rvec[n0 + i] : 0.f;
                eq.mode = EPI_SWAP_QKV;
                epi_swap(eq, m, m_rows, n0, n_tok, lane, f);
              }
            }
            if (!from_ws) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty_bar[acc]);
            }
          }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        j = seg_end;
      }
      // arrive: this CTA's part of step si is in memory
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (ep_tid == 0) {
        __threadfence();
        atomicAdd(call.bar, 1ull);
        if (call.trace) call.trace[(me * 32 + si) * 4 + 2] = gtime_ns();
      }
    }
  }
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

cudaError_t decode_chain_launch(const ChainStep* d_steps, int n_steps, const ChainCall& c, int num_sms,
                                cudaStream_t stream) {
  cudaError_t e = ensure_smem(decode_chain_kernel, ChainCfg::SMEM);
  if (e != cudaSuccess) return e;
  if (c.n_tok <= 0 || n_steps <= 0) return cudaSuccess;
  if (c.n_tok > 512) return cudaErrorInvalidValue;
  return launch_k(decode_chain_kernel, dim3(num_sms), dim3(GEMM_THREADS), ChainCfg::SMEM, stream, d_steps, n_steps,
                  c);
}

}  // namespace eco
