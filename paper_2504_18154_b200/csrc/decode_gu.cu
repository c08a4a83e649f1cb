// Decode gate/up projection + SiLU*up (SURVEY 8(a) row a15 for a10; Eq. 3
// P:181-185, Table 2 "Dim expansion" P:233) with a balanced stream-K partition.
//
// At decode the gate/up GEMM streams 2F x H bf16 weights (8B: 235 MB; 70B/TP=2 rank:
// 470 MB) and is HBM-bound. Its 2F/128 = 224 weight tiles (both shapes) on 148 SMs
// make 1.51 waves: in the second wave only 76 SMs stream, and one SM cannot pull more
// than ~48 GB/s of weights next to its activation tiles (the per-SM TMA ingest is
// ~95 GB/s, half of it activations at B = 128), so the tail runs at ~3.6 TB/s.
//
// Here every CTA streams the same number of (tile, 64-wide K block) units: CTA c owns
// units [c*U/G, (c+1)*U/G) in tile-major order. When a CTA's range is at least one
// tile long (U/G >= K blocks per tile; 8B and 70B/TP=2 both qualify) every tile has at
// most TWO contributors: the CTA whose range ends inside it (it runs the tile's head,
// K blocks 0..y, as its LAST part) and the next CTA (the tail, y+1..end, as its FIRST
// part). The tail owner stores its f32 partial early and raises a flag; the head owner,
// at the end of its range, adds that partial to its accumulator and applies SiLU*up.
// A sum of two terms is commutative, so the result is bitwise deterministic whichever
// CTA finishes first. Partial stores and the final act stores go through smem staging
// and TMA (async bulk) so the epilogue threads never wait on L2 round trips.
//
// CTA: 6 warps (0 TMA producer, 1 MMA + TMEM owner, 2..5 epilogue), tile 128 weight
// rows x BN tokens x 64 K, two TMEM accumulators -- the swap-AB layout of the other
// decode GEMMs (weights are the MMA M side).
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace eco {

namespace {

constexpr int SK_THREADS = 192;
constexpr int SK_BM = 128, SK_BK = 64;
constexpr int SK_SMEM_MAX = 232448;

template <int BN>
struct SkCfg {
  static constexpr int A_BYTES = SK_BM * SK_BK * 2;
  static constexpr int B_BYTES = BN * SK_BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STG = 32 * 128 * 4;  // staging: [32 tok][128 rows] f32 or [32 tok][64] bf16
  static constexpr int BAR_BYTES = 256;
  static constexpr int FIT = (SK_SMEM_MAX - 1024 - STG - BAR_BYTES) / STAGE;
  static constexpr int STAGES = FIT > 8 ? 8 : FIT;
  static constexpr int SMEM = STAGES * STAGE + STG + BAR_BYTES + 1024;
  static constexpr int TMEM_COLS = 2 * BN;
  static_assert((2 * STAGES + 4) * 8 + 8 <= BAR_BYTES, "barriers fit");
};

__device__ __forceinline__ int sk_beg(int c, int U, int G) { return (int)((long long)c * U / G); }

__device__ __forceinline__ void sk_epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void sk_tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void sk_st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int sk_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long sk_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// debug trace marks: 0 start, 1 first stage landed, 2 last MMA issued, 3 tail partial
// published, 4 head flag seen, 5 head partial landed, 6 epilogue done, 7 end
__device__ __forceinline__ void sk_mark(const GuSkArgs& a, int i) {
  if (a.trace) a.trace[blockIdx.x * 16 + i] = sk_now();
}
__device__ __forceinline__ float sk_silu(float z) { return __fdividef(z, 1.f + __expf(-z)); }

// this CTA's parts: (tile, kb0, kb1) in order
struct SkParts {
  int kpt, cur, end;
  __device__ SkParts(int tiles, int kpt_, int cta, int G) : kpt(kpt_) {
    const int U = tiles * kpt;
    cur = sk_beg(cta, U, G);
    end = sk_beg(cta + 1, U, G);
  }
  __device__ bool next(int& t, int& kb0, int& kb1) {
    if (cur >= end) return false;
    t = cur / kpt;
    kb0 = cur % kpt;
    const int u1 = min(end, (t + 1) * kpt);
    kb1 = u1 - t * kpt;
    cur = u1;
    return true;
  }
};

template <int BN>
__global__ void __launch_bounds__(SK_THREADS, 1)
    gu_sk_kernel(const __grid_constant__ CUtensorMap w_map, const __grid_constant__ CUtensorMap x_map,
                 const __grid_constant__ CUtensorMap act_map, const __grid_constant__ CUtensorMap part_map,
                 GuSkArgs a) {
  using C = SkCfg<BN>;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* stg = reinterpret_cast<float*>(smem + S * C::STAGE);  // 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::STAGE + C::STG);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* pbar = tempty + 2;  // partial-tile load into the staging buffer
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(pbar + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int G = gridDim.x, cta = blockIdx.x;
  const int tiles = a.m_rows / SK_BM, kpt = a.K / SK_BK;

  if (threadIdx.x == 0) {
    sk_mark(a, 0);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    mbar_init(pbar, 1);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&w_map);
    tma_prefetch(&x_map);
  }
  if (warp == 2 && lane == 0) {
    tma_prefetch(&act_map);
    tma_prefetch(&part_map);
  }
  if (warp == 1) tmem_alloc(tmem_ptr, C::TMEM_COLS);
  tc_fence_before();
  __syncwarp();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  pdl_trigger();

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      // the weights of the first stages before the PDL wait (they do not depend on the
      // previous kernel), then their activation tiles
      int j = 0, npre = 0;
      int pre_kb[S];
      {
        SkParts P(tiles, kpt, cta, G);
        int t, kb0, kb1;
        while (npre < S && P.next(t, kb0, kb1))
          for (int kb = kb0; kb < kb1 && npre < S; ++kb) {
            mbar_arrive_expect_tx(&full[npre], C::STAGE);
            tma_load_2d(smem + npre * C::STAGE, &w_map, &full[npre], kb * SK_BK, t * SK_BM);
            pre_kb[npre++] = kb;
          }
      }
      pdl_wait();
      for (int i = 0; i < npre; ++i)
        tma_load_2d(smem + i * C::STAGE + C::A_BYTES, &x_map, &full[i], pre_kb[i] * SK_BK, 0);
      SkParts P(tiles, kpt, cta, G);
      int t, kb0, kb1;
      while (P.next(t, kb0, kb1))
        for (int kb = kb0; kb < kb1; ++kb, ++j) {
          if (j < npre) continue;
          const int s = j % S;
          mbar_wait(&empty[s], ((j / S) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], C::STAGE);
          tma_load_2d(smem + s * C::STAGE, &w_map, &full[s], kb * SK_BK, t * SK_BM);
          tma_load_2d(smem + s * C::STAGE + C::A_BYTES, &x_map, &full[s], kb * SK_BK, 0);
        }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(SK_BM, BN);
      int j = 0, acc = 0;
      uint32_t acc_ph = 0;
      SkParts P(tiles, kpt, cta, G);
      int t, kb0, kb1;
      while (P.next(t, kb0, kb1)) {
        mbar_wait(&tempty[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++j) {
          const int s = j % S;
          mbar_wait(&full[s], (j / S) & 1);
          if (j == 0) sk_mark(a, 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * C::STAGE);
          const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
          for (int k = 0; k < SK_BK / 16; ++k) tc_mma_f16(d, da + 2 * k, db + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_ph ^= 1;
        }
      }
      sk_mark(a, 2);
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    pdl_wait();  // (the act / partial writes below follow every earlier kernel of the stream)
    const int q = warp & 3;
    const int row = q * 32 + lane;  // weight row of the tile = TMEM lane
    const int ep_tid = (warp - 2) * 32 + lane;
    const int B = a.B;
    const uint32_t stg_s = smem_u32(stg);
    int acc = 0;
    uint32_t acc_ph = 0, p_ph = 0;
    SkParts P(tiles, kpt, cta, G);
    int t, kb0, kb1;
    while (P.next(t, kb0, kb1)) {
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      const bool tail = kb0 > 0;                // the tile's tail: store the partial, raise the flag
      const bool head = !tail && kb1 < kpt;     // the tile's head: add the tail's partial
      if (head && ep_tid == 0) {
        // the tail owner ran this tile first in its range: its flag is normally long set
        const unsigned long long t0 = sk_now();
        while (sk_ld_acquire(a.flags + t) < a.epoch) {
          __nanosleep(64);
          if (sk_now() - t0 > 2000000000ull) {
            atomicExch(a.err, 1);
            break;
          }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // for the TMA loads of the partial
        sk_mark(a, 4);
      }
      if (tail) {
        // partial -> staging [32 tok][128 rows] f32 -> TMA store into the tile's slot (early
        // in this CTA's range: overlapped with its following tiles' mainloop)
        for (int c0 = 0; c0 < B; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tacc + c0, v);
          tc_wait_ld();
          if (ep_tid == 0) bulk_wait_read0();  // the previous chunk's store has read the staging
          sk_epi_bar();
#pragma unroll
          for (int i = 0; i < 32; ++i) sts_f32(stg_s + (uint32_t)(i * 128 + row) * 4u, __uint_as_float(v[i]));
          fence_proxy_async();
          sk_epi_bar();
          if (ep_tid == 0) {
            sk_tma_store_2d(&part_map, stg, 0, t * SK_BM + c0);
            bulk_commit();
          }
        }
      } else {
        // full tile or head: silu(gate) * up for all tokens; the act chunks get their own
        // 4 KB of the staging buffer each ([32 tok][64] bf16), so the chunks never wait on
        // each other's stores -- only on the previous part's (once)
        const uint32_t ring_s = smem_u32(smem);
        if (head && ep_tid == 0) {
          // the head is this CTA's last part: every MMA is done, the smem ring is free.
          // The tail's partial of all tokens, by TMA into the ring, one round trip.
          const int nch = (B + 31) / 32;
          mbar_arrive_expect_tx(pbar, nch * 32 * 128 * 4);
          for (int c = 0; c < nch; ++c)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];" ::"r"(ring_s + (uint32_t)c * (32 * 128 * 4)),
                "l"(reinterpret_cast<uint64_t>(&part_map)), "r"(0), "r"(t * SK_BM + c * 32), "r"(smem_u32(pbar))
                : "memory");
        }
        if (ep_tid == 0) bulk_wait_read0();  // the previous part's stores have read the staging
        sk_epi_bar();
        if (head) {
          mbar_wait(pbar, p_ph);
          p_ph ^= 1;
          if (ep_tid == 0) sk_mark(a, 5);
        }
        const int col = row >> 1;  // rows 2j / 2j+1 of the tile are gate_j / up_j
        for (int c0 = 0; c0 < B; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tacc + c0, v);
          tc_wait_ld();
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]);
          if (head) {
            const uint32_t pb = ring_s + (uint32_t)(c0 / 32) * (32 * 128 * 4);
#pragma unroll
            for (int i = 0; i < 32; ++i) f[i] += lds_f32(pb + (uint32_t)(i * 128 + row) * 4u);  // own + tail
          }
          const uint32_t sb = stg_s + (uint32_t)(c0 / 32) * (32 * 64 * 2);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float other = __shfl_xor_sync(0xffffffffu, f[i], 1);
            if (!(lane & 1))
              sts_u16(sb + (uint32_t)(i * 64 + col) * 2u, __bfloat16_as_ushort(__float2bfloat16_rn(sk_silu(f[i]) * other)));
          }
          fence_proxy_async();
          sk_epi_bar();
          if (ep_tid == 0) {
            sk_tma_store_2d(&act_map, stg + (c0 / 32) * (32 * 64 / 2), t * 64, c0);
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_ph ^= 1;
      }
      if (tail && ep_tid == 0) {
        bulk_wait0();  // the partial is in global memory
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
        sk_st_release(a.flags + t, a.epoch);
        sk_mark(a, 3);
      }
    }
    if (ep_tid == 0) bulk_wait0();  // act complete before the grid ends (PDL dependents)
    if (ep_tid == 0) sk_mark(a, 6);
  }
  tc_fence_before();
  __syncwarp();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) sk_mark(a, 7);
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace

bool gu_sk_applicable(int m_rows, int K, int B, int num_sms) {
  if (m_rows % SK_BM || K % SK_BK || B < 1 || B > 128) return false;
  const int tiles = m_rows / SK_BM;
  // more tiles than SMs (a second wave), and every CTA range at least one tile long
  // (so each tile has at most two contributors)
  return tiles > num_sms;  // (then U / G = tiles * kpt / G > kpt)
}

cudaError_t gu_sk_launch(const CUtensorMap* w_map, const CUtensorMap* x_map, const CUtensorMap* act_map,
                         const CUtensorMap* part_map, const GuSkArgs& a, int bn, int num_sms, cudaStream_t s) {
  if (!gu_sk_applicable(a.m_rows, a.K, a.B, num_sms) || (bn != 64 && bn != 128) || a.B > bn)
    return cudaErrorInvalidValue;
  if (bn == 64) {
    cudaError_t e = ensure_smem(gu_sk_kernel<64>, SkCfg<64>::SMEM);
    if (e != cudaSuccess) return e;
    return launch_k(gu_sk_kernel<64>, dim3(num_sms), dim3(SK_THREADS), SkCfg<64>::SMEM, s, *w_map, *x_map, *act_map,
                    *part_map, a);
  }
  cudaError_t e = ensure_smem(gu_sk_kernel<128>, SkCfg<128>::SMEM);
  if (e != cudaSuccess) return e;
  return launch_k(gu_sk_kernel<128>, dim3(num_sms), dim3(SK_THREADS), SkCfg<128>::SMEM, s, *w_map, *x_map, *act_map,
                  *part_map, a);
}

}  // namespace eco
