// Decode-step dataflow kernel: O projection -> gate/up (+SiLU) -> down projection of
// one decoder layer (SURVEY 8(a) rows a9-a11 at T = B, i.e. a15; Table 2
// P:231-236, Eq. 3) as ONE persistent kernel over all SMs.
//
// Why: at decode the three projections stream 386 MB of weights (8B shape) and are
// HBM-bound, but as separate kernels every boundary costs a ramp (first TMA data
// ~3 us after the CTA starts), a tail (the last tiles' epilogues, wave quantisation
// of the 224 gate/up tiles on 148 SMs) and a split-K reduction + RMSNorm kernel
// (tools/decode_ablate.py: 3.2 ms of a 7.7 ms step for 12.4 GB, 3.8 TB/s). Here the
// weight stream never waits for a boundary:
//
//  * Partition. Each GEMM's (tile, K block) units, tile-major, are split evenly over
//    the grid (stream-K): CTA c runs units [c*U/G, (c+1)*U/G) of O, then of gate/up,
//    then of down. Every CTA streams the same number of weight bytes per GEMM.
//  * Split tiles. A tile whose units span several CTAs is a set of contributors; each
//    writes its f32 partial to its slot, and the last to arrive (per-tile counter)
//    sums all slots in contributor (K) order -- deterministic -- and runs the epilogue.
//  * Dataflow. Warp 0 streams weights (TMA) as far ahead as the smem ring allows,
//    independent of everything. Warp 6 loads the activation K block of each unit only
//    once the tile that produces it is complete: gate/up K block kb needs O tile kb/2
//    (flag), down K block kb needs gate/up tile kb (flag). No grid barrier.
//  * Deferred RMSNorm (reading A4). x_next = x + O(x) needs a whole row for its
//    norm, which no O tile has. The O reducers write x, h = bf16(x * gamma_ffn) and the
//    tile's sum of squares per token; gate/up consumes h and multiplies its outputs by
//    r = 1/rms(x) (sum of the 32 tile sums) before SiLU, which is the same
//    rmsnorm(x) * gamma * W up to where the scalar r is applied. The down reducers do
//    the same for the next layer's QKV (h_out, ss_d, rvec) or the final norm (LM head
//    input; argmax is invariant to r > 0).
//
// CTA: 7 warps. 0 weight producer, 1 MMA issuer + TMEM owner, 2..5 epilogue (TMEM lane
// quarter warp % 4), 6 activation producer. Tile = 128 weight rows x BN tokens x 64 K
// (swap-AB as the decode GEMMs: weights are the MMA M side), two TMEM accumulators.
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace eco {

namespace {

constexpr int FL_THREADS = 224;
constexpr int FL_BM = 128, FL_BK = 64;
constexpr int FL_SMEM_MAX = 232448;

template <int BN>
struct FlowCfg {
  static constexpr int A_BYTES = FL_BM * FL_BK * 2;
  static constexpr int B_BYTES = BN * FL_BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STG = 32 * 128 * 4;  // epilogue staging: [32 tok][128] f32 / [32 tok][64] bf16
  static constexpr int SCRATCH = STG + 4 * 128 * 4 + 128 * 4 + 64;  // + red, r_o, ints
  static constexpr int BAR_BYTES = 512;
  static constexpr int FIT = (FL_SMEM_MAX - 1024 - SCRATCH - BAR_BYTES) / STAGE;
  static constexpr int STAGES = FIT > 10 ? 10 : FIT;
  static constexpr int SMEM = STAGES * STAGE + SCRATCH + BAR_BYTES + 1024;
  static constexpr int TMEM_COLS = 2 * BN;  // 128 or 256
  static_assert((3 * STAGES + 4) * 8 <= BAR_BYTES, "barriers fit");
};

// stream-K partition of U units over G CTAs
__device__ __forceinline__ int fl_beg(int c, int U, int G) { return (int)((long long)c * U / G); }
__device__ __forceinline__ int fl_owner(int u, int U, int G) { return (int)(((long long)(u + 1) * G - 1) / U); }

struct Geo {
  int tiles, kpt;
};

__device__ __forceinline__ Geo fl_geo(const FlowArgs& a, int g) {
  if (g == 0) return Geo{a.H / FL_BM, a.MD / FL_BK};
  if (g == 1) return Geo{2 * a.F / FL_BM, a.H / FL_BK};
  return Geo{a.H / FL_BM, a.F / FL_BK};
}

// The parts a CTA runs of GEMM g, in order: (tile, K blocks [kb0, kb1)). Gate/up is
// partitioned by whole tiles (tile t -> CTA t mod G: 224 tiles = 148 + 76, no split tile,
// no reduction; the CTAs with one tile go on to prefetch down weights); O and down (32
// tiles of long K) by stream-K ranges, split tiles reduced through slots.
struct Parts {
  int g, kpt, cur, end, G;
  __device__ Parts(const FlowArgs& a, int g_, int cta, int G_) : g(g_), G(G_) {
    const Geo geo = fl_geo(a, g);
    kpt = geo.kpt;
    if (g == 1) {
      cur = cta;
      end = geo.tiles;
    } else {
      const int U = geo.tiles * geo.kpt;
      cur = fl_beg(cta, U, G);
      end = fl_beg(cta + 1, U, G);
    }
  }
  __device__ bool next(int& t, int& kb0, int& kb1) {
    if (cur >= end) return false;
    if (g == 1) {
      t = cur;
      kb0 = 0;
      kb1 = kpt;
      cur += G;
      return true;
    }
    t = cur / kpt;
    kb0 = cur % kpt;
    const int u1 = min(end, (t + 1) * kpt);
    kb1 = u1 - t * kpt;
    cur = u1;
    return true;
  }
};

__device__ __forceinline__ unsigned long long fl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_volatile_s32(const int* p) {
  int v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int4 ld_volatile_v4(const int* p) {
  int4 v;
  asm volatile("ld.volatile.global.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// TMA tile store / f32 reduce-add (L2 performs the adds) from a row-major smem tile
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

// mbarrier wait that suspends the thread (up to the hint, woken by the phase change)
// instead of spinning: in this kernel producers and the MMA issuer can wait for tens of
// microseconds on a dependency, and spinning try_wait loops of three warps measurably
// slow the loads of the reducing epilogue warps on the same SM.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// Flags readiness cache of one producer thread: bit t of `ready` = flag t seen >= epoch.
// A miss reloads the 32 flags of t's group (one 128-byte line) and then fences, so the
// loads that follow are ordered after every flag observed ready (acquire pattern).
// Returns false on timeout (the producing CTA never ran: grid not co-resident).
struct FlagCache {
  unsigned ready[8];  // up to 256 tiles
  __device__ void clear() {
#pragma unroll
    for (int i = 0; i < 8; ++i) ready[i] = 0u;
  }
  __device__ bool wait(const int* flags, int n, int t, int epoch, int* err) {
    const int grp = t >> 5;
    if (ready[grp] >> (t & 31) & 1u) return true;
    // poll only the needed flag, with exponential back-off: ~150 pollers on one 128-byte
    // line without back-off saturate its L2 slice and slow every access that maps there
    const unsigned long long t0 = fl_now();
    unsigned ns = 64;
    while (ld_volatile_s32(flags + t) < epoch) {
      __nanosleep(ns);
      ns = ns < 2048 ? 2 * ns : ns;
      if (fl_now() - t0 > 2000000000ull) {
        atomicExch(err, 1);
        return false;
      }
    }
    // then pick up every flag of the group that is ready too (one line)
    unsigned m = 1u << (t & 31);
    const int base = grp * 32;
    for (int q = 0; q < 32 && base + q < n; q += 4) {
      if (base + q + 4 <= n) {
        const int4 v = ld_volatile_v4(flags + base + q);
        m |= (v.x >= epoch ? 1u : 0u) << q | (v.y >= epoch ? 1u : 0u) << (q + 1) |
             (v.z >= epoch ? 1u : 0u) << (q + 2) | (v.w >= epoch ? 1u : 0u) << (q + 3);
      } else {
        for (int r = q; r < 32 && base + r < n; ++r) m |= (ld_volatile_s32(flags + base + r) >= epoch ? 1u : 0u) << r;
      }
    }
    ready[grp] |= m;
    __threadfence();             // acquire: order the dependent loads after the flags
    fence_proxy_async_global();  // ... including the TMA (async proxy) loads
    return true;
  }
};

// debug trace marks (FlowArgs::trace): 0 start, 1 first weights landed, 2/3/4 last MMA of
// O / gate-up / down issued, 5/6/7 epilogue done with O / gate-up / down, 8 first gate-up
// activation load issued, 9 first down activation load issued, 10 end
__device__ __forceinline__ void fl_mark(const FlowArgs& a, int i) {
  if (a.trace) a.trace[blockIdx.x * 16 + i] = fl_now();
}

__device__ __forceinline__ float fl_silu(float z) { return __fdividef(z, 1.f + __expf(-z)); }

template <int BN>
__global__ void __launch_bounds__(FL_THREADS, 1)
    decode_flow_kernel(const __grid_constant__ CUtensorMap w_o, const __grid_constant__ CUtensorMap w_gu,
                       const __grid_constant__ CUtensorMap w_d, const __grid_constant__ CUtensorMap b_o,
                       const __grid_constant__ CUtensorMap b_gu, const __grid_constant__ CUtensorMap b_d,
                       const __grid_constant__ CUtensorMap x_map, const __grid_constant__ CUtensorMap act_map,
                       FlowArgs a) {
  using C = FlowCfg<BN>;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* stg = reinterpret_cast<float*>(smem + S * C::STAGE);  // [32][128] f32 staging (1024-aligned)
  float* red = stg + C::STG / 4;                               // [4][128]
  float* r_o = red + 4 * 128;                                  // [128]
  int* s_int = reinterpret_cast<int*>(r_o + 128);              // [0] last flag, [1] r_o ready, [2] last-down
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + S * C::STAGE + C::SCRATCH);
  uint64_t* fullB = fullA + S;
  uint64_t* empty = fullB + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int G = gridDim.x, cta = blockIdx.x;

  if (threadIdx.x == 0) {
    fl_mark(a, 0);
    for (int s = 0; s < S; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&fullB[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    s_int[1] = 0;
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&w_o);
    tma_prefetch(&w_gu);
    tma_prefetch(&w_d);
  }
  if (warp == 2 && lane == 0) {
    tma_prefetch(&x_map);
    tma_prefetch(&act_map);
  }
  if (warp == 6 && lane == 0) {
    tma_prefetch(&b_o);
    tma_prefetch(&b_gu);
    tma_prefetch(&b_d);
  }
  if (warp == 1) tmem_alloc(tmem_ptr, C::TMEM_COLS);
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  pdl_trigger();

  if (warp == 0) {
    // ---------------------------------------------------------------- weights (no dependencies)
    if (lane == 0) {
      int j = 0;
      for (int g = 0; g < 3; ++g) {
        const CUtensorMap* m = g == 0 ? &w_o : g == 1 ? &w_gu : &w_d;
        Parts P(a, g, cta, G);
        int t, kb0, kb1;
        while (P.next(t, kb0, kb1))
          for (int kb = kb0; kb < kb1; ++kb, ++j) {
            const int s = j % S;
            mbar_wait_sleep(&empty[s], ((j / S) & 1) ^ 1);
            mbar_arrive_expect_tx(&fullA[s], C::A_BYTES);
            tma_load_2d(smem + s * C::STAGE, m, &fullA[s], kb * FL_BK, t * FL_BM);
          }
      }
    }
  } else if (warp == 6) {
    // ---------------------------------------------------------------- activations (dataflow)
    if (lane == 0) {
      pdl_wait();  // the attention output of this layer
      FlagCache fo, fg;
      fo.clear();
      fg.clear();
      int j = 0;
      bool ok = true;
      for (int g = 0; g < 3; ++g) {
        const CUtensorMap* m = g == 0 ? &b_o : g == 1 ? &b_gu : &b_d;
        Parts P(a, g, cta, G);
        int t, kb0, kb1;
        bool first = true;
        while (P.next(t, kb0, kb1))
          for (int kb = kb0; kb < kb1; ++kb, ++j) {
            const int s = j % S;
            mbar_wait_sleep(&empty[s], ((j / S) & 1) ^ 1);
            if (ok && g == 1) ok = fo.wait(a.flags_o, a.H / FL_BM, kb / 2, a.epoch, a.err);
            if (ok && g == 2) ok = fg.wait(a.flags_gu, 2 * a.F / FL_BM, kb, a.epoch, a.err);
            if (g > 0 && first) fl_mark(a, 7 + g);
            first = false;
            mbar_arrive_expect_tx(&fullB[s], C::B_BYTES);
            tma_load_2d(smem + s * C::STAGE + C::A_BYTES, m, &fullB[s], kb * FL_BK, 0);
          }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(FL_BM, BN);
      int j = 0, acc = 0;
      uint32_t acc_ph = 0;
      for (int g = 0; g < 3; ++g) {
        Parts P(a, g, cta, G);
        int t, kb0, kb1;
        while (P.next(t, kb0, kb1)) {
          mbar_wait_sleep(&tempty[acc], acc_ph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + acc * BN;
          for (int kb = kb0; kb < kb1; ++kb, ++j) {
            const int s = j % S;
            const uint32_t ph = (j / S) & 1;
            mbar_wait_sleep(&fullA[s], ph);
            if (j == 0) fl_mark(a, 1);
            mbar_wait_sleep(&fullB[s], ph);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * C::STAGE);
            const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_BYTES);
#pragma unroll
            for (int k = 0; k < FL_BK / 16; ++k)
              tc_mma_f16(d, da + 2 * k, db + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
            tc_commit(&empty[s]);
          }
          tc_commit(&tfull[acc]);
          if (++acc == 2) {
            acc = 0;
            acc_ph ^= 1;
          }
        }
        fl_mark(a, 2 + g);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..5)
    pdl_wait();
    const int q = warp & 3;
    const int row = q * 32 + lane;  // weight row within the tile = TMEM lane
    const int ep_tid = (warp - 2) * 32 + lane, ep_warp = warp - 2;
    const int B = a.B;
    const uint32_t stg_s = smem_u32(stg);
    int acc = 0;
    uint32_t acc_ph = 0;
    // 1/rms per token after O, for the gate/up epilogues (once per CTA; every O tile is
    // complete by the time a gate/up accumulator exists, the poll only orders the reads)
    auto ensure_r_o = [&]() {
      if (s_int[1]) return;
      const int n_o = a.H / FL_BM;
      if (ep_tid < 32) {
        const unsigned long long t0 = fl_now();
        for (int k0 = 0; k0 < n_o; k0 += 32) {
          const int k = k0 + ep_tid;
          while (!__all_sync(0xffffffffu, k >= n_o || ld_volatile_s32(a.flags_o + k) >= a.epoch)) {
            __nanosleep(1024);
            if (fl_now() - t0 > 2000000000ull) {
              if (ep_tid == 0) atomicExch(a.err, 1);
              break;
            }
          }
        }
        __threadfence();
      }
      epi_bar();
      if (ep_tid < B) {
        float ss = 0.f;
        for (int k = 0; k < n_o; ++k) ss += __ldcg(a.ss_o + k * 128 + ep_tid);
        r_o[ep_tid] = rsqrtf(ss * a.inv_h + a.eps);
      }
      if (ep_tid == 0) s_int[1] = 1;  // every epilogue thread has read s_int[1] already
      epi_bar();
    };
    // After the tile's x rows are final (every contributor's reduce-add landed): h =
    // bf16(x * gamma) and the tile's per-token sum of squares for tokens [tb, te).
    // Warp = token, lane = 4 consecutive features (float4).
    auto share_rows = [&](int g, int t, int tb, int te) {
      const int f4 = lane * 4;
      const int feat = t * FL_BM + f4;
      const bf16* gp = (g == 0 ? a.gamma_o : a.gamma_d) + feat;
      const float4 gm = make_float4(__bfloat162float(gp[0]), __bfloat162float(gp[1]), __bfloat162float(gp[2]),
                                    __bfloat162float(gp[3]));
      bf16* hdst = g == 0 ? a.h : a.h_out;
      float* ssd = g == 0 ? a.ss_o : a.ss_d;
      constexpr int U4 = 4;  // tokens per warp per pass, loads in flight together
      for (int tok0 = tb + ep_warp; tok0 < te; tok0 += 4 * U4) {
        float4 xv[U4];
#pragma unroll
        for (int u = 0; u < U4; ++u) {
          const int tk = tok0 + 4 * u;
          xv[u] = tk < te ? __ldcg(reinterpret_cast<const float4*>(a.x + (int64_t)tk * a.H + feat))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U4; ++u) {
          const int tk = tok0 + 4 * u;
          if (tk >= te) continue;  // warp-uniform
          *reinterpret_cast<uint2*>(hdst + (int64_t)tk * a.H + feat) = make_uint2(
              pack_bf16x2(xv[u].x * gm.x, xv[u].y * gm.y), pack_bf16x2(xv[u].z * gm.z, xv[u].w * gm.w));
          float sq = xv[u].x * xv[u].x + xv[u].y * xv[u].y + xv[u].z * xv[u].z + xv[u].w * xv[u].w;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
          if (lane == 0) ssd[t * 128 + tk] = sq;
        }
      }
    };
    // a down tile is complete: the last one also leaves 1/rms per token for the next QKV
    auto down_tile_done = [&](int n_tiles) {
      if (ep_tid == 0) {
        const int old = atomicAdd(a.done_d, 1);
        s_int[2] = old == n_tiles - 1;
        if (old == n_tiles - 1) *a.done_d = 0;
      }
      epi_bar();
      if (s_int[2]) {
        __threadfence();
        if (ep_tid < B) {
          float ss = 0.f;
          for (int k = 0; k < n_tiles; ++k) ss += __ldcg(a.ss_d + k * 128 + ep_tid);
          a.rvec[ep_tid] = rsqrtf(ss * a.inv_h + a.eps);
        }
      }
    };
    for (int g = 0; g < 3; ++g) {
      const Geo geo = fl_geo(a, g);
      const int U = geo.tiles * geo.kpt;
      int pend_t[2] = {0, 0}, pend_n[2] = {0, 0}, pend_k[2] = {0, 0}, n_pend = 0;
      Parts P(a, g, cta, G);
      int t, kb0, kb1;
      while (P.next(t, kb0, kb1)) {
        mbar_wait_sleep(&tfull[acc], acc_ph);
        tc_fence_after();
        const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
        if (g == 1) {
          // ------------------------------------------ gate/up: a whole tile (thread = row)
          // silu(r g) * (r u) -> smem [32 tok][64] bf16 -> TMA store into act
          ensure_r_o();
          const int col = row >> 1;  // rows 2j / 2j+1 are gate_j / up_j (pair-interleaved W_gu)
          for (int c0 = 0; c0 < B; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(tacc + c0, v);
            tc_wait_ld();
            if (c0 > 0) {  // the previous chunk's store has read the staging tile
              if (ep_tid == 0) bulk_wait_read0();
              epi_bar();
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float f = __uint_as_float(v[i]);
              const float other = __shfl_xor_sync(0xffffffffu, f, 1);
              if (!(lane & 1)) {
                const float r = c0 + i < B ? r_o[c0 + i] : 0.f;
                sts_u16(stg_s + (uint32_t)(i * 64 + col) * 2u,
                        __bfloat16_as_ushort(__float2bfloat16_rn(fl_silu(r * f) * (r * other))));
              }
            }
            fence_proxy_async();
            epi_bar();
            if (ep_tid == 0) {
              tma_store_2d(&act_map, stg, t * 64, c0);
              bulk_commit();
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
          if (acc == 1) acc_ph ^= 1;
          acc ^= 1;
          if (ep_tid == 0) {
            bulk_wait0();  // the tile is in act
            __threadfence();
            fence_proxy_async_global();
            st_release_gpu(a.flags_gu + t, a.epoch);
          }
          epi_bar();  // staging free for the next part
          continue;
        }
        // -------------------------------------------- O / down: partial tile reduce-added into x
        for (int c0 = 0; c0 < B; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tacc + c0, v);
          tc_wait_ld();
          if (c0 > 0) {
            if (ep_tid == 0) bulk_wait_read0();
            epi_bar();
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) sts_f32(stg_s + (uint32_t)(i * 128 + row) * 4u, c0 + i < B ? __uint_as_float(v[i]) : 0.f);
          fence_proxy_async();
          epi_bar();
          if (ep_tid == 0) {
            tma_reduce_add_2d(&x_map, stg, t * FL_BM, c0);
            bulk_commit();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (acc == 1) acc_ph ^= 1;
        acc ^= 1;
        if (ep_tid == 0) {
          // contributors of tile t (CTAs with empty ranges skipped) and this CTA's index
          const int c_lo = fl_owner(t * geo.kpt, U, G), c_hi = fl_owner((t + 1) * geo.kpt - 1, U, G);
          int n = 0, k = 0;
          for (int c = c_lo; c <= c_hi; ++c) {
            if (fl_beg(c, U, G) == fl_beg(c + 1, U, G)) continue;
            if (c == cta) k = n;
            ++n;
          }
          bulk_wait0();  // this CTA's adds are performed
          __threadfence();
          fence_proxy_async_global();
          atomicAdd(&a.cnt[g * a.cnt_ld + t], 1);
          s_int[3] = n;
          s_int[4] = k;
        }
        epi_bar();  // staging free; n / k visible
        // every contributor reduces a share of the tokens -- after this CTA has arrived on
        // ALL its tiles of the GEMM (waiting here would chain the tiles through the CTAs
        // that hold two parts)
        if (n_pend < 2) {
          pend_t[n_pend] = t;
          pend_n[n_pend] = s_int[3];
          pend_k[n_pend] = s_int[4];
        }
        ++n_pend;
      }
      if (g == 1) {
        if (ep_tid == 0) fl_mark(a, 5 + g);
        continue;
      }
      for (int pi = 0; pi < n_pend && pi < 2; ++pi) {
        const int tt = pend_t[pi], n = pend_n[pi], k = pend_k[pi];
        if (ep_tid == 0) {
          const unsigned long long t0 = fl_now();
          unsigned ns = 32;
          while (ld_volatile_s32(a.cnt + g * a.cnt_ld + tt) < n) {
            __nanosleep(ns);
            ns = ns < 1024 ? 2 * ns : ns;
            if (fl_now() - t0 > 2000000000ull) {
              atomicExch(a.err, 1);
              break;
            }
          }
          __threadfence();
        }
        epi_bar();
        if (ep_tid == 0 && g == 0) fl_mark(a, 11);
        share_rows(g, tt, k * B / n, (k + 1) * B / n);
        epi_bar();
        if (ep_tid == 0) {
          if (g == 0) fl_mark(a, 12);
          __threadfence();
          const int old = atomicAdd(&a.cnt[(3 + g) * a.cnt_ld + tt], 1);
          s_int[0] = old == n - 1;
          if (old == n - 1) {  // every contributor is past its wait: reset both counters
            a.cnt[g * a.cnt_ld + tt] = 0;
            a.cnt[(3 + g) * a.cnt_ld + tt] = 0;
            __threadfence();
            fence_proxy_async_global();
            if (g == 0) st_release_gpu(a.flags_o + tt, a.epoch);
          }
        }
        epi_bar();
        if (g == 2 && s_int[0]) down_tile_done(geo.tiles);
      }
      if (n_pend > 2 && ep_tid == 0) atomicExch(a.err, 2);  // (a CTA has at most a first and a last part)
      if (ep_tid == 0) fl_mark(a, 5 + g);
    }
  }
  tc_fence_before();
  __syncwarp();  // lanes of the role warps reconverge: bar.sync counts whole warps
  __syncthreads();
  if (threadIdx.x == 0) fl_mark(a, 10);
  if (warp == 1) tmem_dealloc(tmem_base, C::TMEM_COLS);
}

}  // namespace

int64_t decode_flow_slot_floats(int num_sms) { return 3LL * num_sms * 2 * 128 * 128; }

cudaError_t decode_flow_launch(const CUtensorMap* w_o, const CUtensorMap* w_gu, const CUtensorMap* w_d,
                               const CUtensorMap* b_o, const CUtensorMap* b_gu, const CUtensorMap* b_d,
                               const CUtensorMap* x_map, const CUtensorMap* act_map, const FlowArgs& a, int bn,
                               int num_sms, cudaStream_t s) {
  if (a.B < 1 || a.B > bn || (bn != 64 && bn != 128)) return cudaErrorInvalidValue;
  if (a.H % FL_BM || a.MD % FL_BK || a.F % FL_BK || 2 * a.F / FL_BM > 256 || a.H / FL_BM > 128)
    return cudaErrorInvalidValue;
  if (bn == 64) {
    cudaError_t e = ensure_smem(decode_flow_kernel<64>, FlowCfg<64>::SMEM);
    if (e != cudaSuccess) return e;
    return launch_k(decode_flow_kernel<64>, dim3(num_sms), dim3(FL_THREADS), FlowCfg<64>::SMEM, s, *w_o, *w_gu, *w_d,
                    *b_o, *b_gu, *b_d, *x_map, *act_map, a);
  }
  cudaError_t e = ensure_smem(decode_flow_kernel<128>, FlowCfg<128>::SMEM);
  if (e != cudaSuccess) return e;
  return launch_k(decode_flow_kernel<128>, dim3(num_sms), dim3(FL_THREADS), FlowCfg<128>::SMEM, s, *w_o, *w_gu, *w_d,
                  *b_o, *b_gu, *b_d, *x_map, *act_map, a);
}

}  // namespace eco
