// Memory-bound helper kernels of the hot path:
//  * embedding gather (Fig. 2) -> fp32 residual stream
//  * RMSNorm (reading A4) of residual rows -> bf16 GEMM input
//  * fixed-order split-K reduction with the decode epilogues (a13, a15):
//    RoPE + paged KV append, residual add, SiLU*up
//  * greedy argmax reduction over LM-head tile partials (a12, a16; reading A6)
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "launch.cuh"

namespace eco {

__global__ void embed_kernel(const int* __restrict__ ids, const bf16* __restrict__ E, float* __restrict__ x, int H,
                             int V) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  // ids are range-checked on the host (prompts) or come from the argmax, whose NaN
  // sentinel the host rejects before it is fed back; clamp anyway so a bad id can
  // never read outside the table
  const int id = min(max(ids[t], 0), V - 1);
  const bf16* src = E + (int64_t)id * H;
  float* dst = x + (int64_t)t * H;
  for (int i = threadIdx.x * 8; i < H; i += blockDim.x * 8) {
    uint4 v = *reinterpret_cast<const uint4*>(src + i);
    float4 a = make_float4(bf16_lo(v.x), bf16_hi(v.x), bf16_lo(v.y), bf16_hi(v.y));
    float4 b = make_float4(bf16_lo(v.z), bf16_hi(v.z), bf16_lo(v.w), bf16_hi(v.w));
    *reinterpret_cast<float4*>(dst + i) = a;
    *reinterpret_cast<float4*>(dst + i + 4) = b;
  }
}

cudaError_t embed_launch(const int* ids, const bf16* E, float* x, int n, int H, int V, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  return launch_k(embed_kernel, dim3(n), dim3(128), 0, s, ids, E, x, H, V);
}

// out[i] = bf16( x[row_i] * rsqrt(mean(x[row_i]^2) + eps) * gamma ), row_i = rows ? rows[i] : i
__global__ void rmsnorm_kernel(const float* __restrict__ x, int64_t ldx, const int* __restrict__ rows,
                               const bf16* __restrict__ gamma, bf16* __restrict__ out, int H, float eps) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x;
  const int r = rows ? rows[i] : i;
  const float* src = x + (int64_t)r * ldx;
  float ss = 0.f;
  for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(src + c);
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / H + eps);
  bf16* dst = out + (int64_t)i * H;
  for (int c = threadIdx.x * 4; c < H; c += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(src + c);
    uint2 gv = *reinterpret_cast<const uint2*>(gamma + c);
    uint2 o;
    o.x = pack_bf16x2(v.x * inv * bf16_lo(gv.x), v.y * inv * bf16_hi(gv.x));
    o.y = pack_bf16x2(v.z * inv * bf16_lo(gv.y), v.w * inv * bf16_hi(gv.y));
    *reinterpret_cast<uint2*>(dst + c) = o;
  }
}

cudaError_t rmsnorm_launch(const float* x, int64_t ldx, const int* rows, const bf16* gamma, bf16* out, int n, int H,
                           float eps, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (H % 4) return cudaErrorInvalidValue;
  const int threads = H >= 4096 ? 512 : (H >= 1024 ? 256 : 128);
  return launch_k(rmsnorm_kernel, dim3(n), dim3(threads), 0, s, x, ldx, rows, gamma, out, H, eps);
}

__global__ void row_gather_kernel(const bf16* __restrict__ s0, const bf16* __restrict__ s1,
                                  const bf16* __restrict__ s2, const int* __restrict__ sel,
                                  const int* __restrict__ row, bf16* __restrict__ dst, int cols) {
  const int r = blockIdx.x;
  const bf16* src = (sel[r] == 0 ? s0 : sel[r] == 1 ? s1 : s2) + (int64_t)row[r] * cols;
  bf16* d = dst + (int64_t)r * cols;
  for (int c = threadIdx.x * 8; c < cols; c += blockDim.x * 8)
    *reinterpret_cast<uint4*>(d + c) = *reinterpret_cast<const uint4*>(src + c);
}

cudaError_t row_gather_launch(const bf16* s0, const bf16* s1, const bf16* s2, const int* sel, const int* row, bf16* dst,
                              int nrows, int cols, cudaStream_t s) {
  if (nrows == 0) return cudaSuccess;
  if (cols % 8) return cudaErrorInvalidValue;
  row_gather_kernel<<<nrows, 128, 0, s>>>(s0, s1, s2, sel, row, dst, cols);
  return cudaGetLastError();
}

// tokens[i] = argmax over parts of (val, idx): largest value, lowest index on ties.
// One NaN rule with the LM-head epilogue (gemm_sm100.cu, EPI_SWAP_ARGMAX): a NaN
// logit wins every comparison, and a row whose winner is NaN gets the token
// ECO_TOKEN_NAN (reading A6: NaN logits are an error), which the host rejects.
__device__ __forceinline__ bool am_better(float v, int x, float bv, int bi) {
  if (isnan(v)) return !isnan(bv) || x < bi;
  if (isnan(bv)) return false;
  return v > bv || (v == bv && x < bi);
}

__global__ void argmax_reduce_kernel(const float* __restrict__ val, const int* __restrict__ idx, int parts, int ld,
                                     int* __restrict__ tokens) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int p = threadIdx.x; p < parts; p += blockDim.x) {
    const float v = val[(int64_t)i * ld + p];
    const int x = idx[(int64_t)i * ld + p];
    if (am_better(v, x, bv, bi)) { bv = v; bi = x; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (am_better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x / 32); ++w)
      if (am_better(sv[w], si[w], bv, bi)) { bv = sv[w]; bi = si[w]; }
    tokens[i] = isnan(bv) ? ECO_TOKEN_NAN : bi;
  }
}

cudaError_t argmax_reduce_launch(const float* val, const int* idx, int n, int parts, int ld, int* tokens,
                                 cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  return launch_k(argmax_reduce_kernel, dim3(n), dim3(128), 0, s, val, idx, parts, ld, tokens);
}

// Decode O / down projection tail fused with the next RMSNorm: per row,
//   x += sum_s part[s][row][:]  (fixed split order)  ;  out = bf16(rmsnorm(x) * gamma)
// One CTA per row; each thread keeps its <= 4 float4 of the row in registers.
__global__ void __launch_bounds__(1024) splitk_resid_rmsnorm_kernel(const float* __restrict__ part, int splits, int rows,
                                            float* __restrict__ x, const bf16* __restrict__ gamma,
                                            bf16* __restrict__ out, int H, float eps, int sk_L, int sk_kbt) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x;
  const int64_t plane = (int64_t)rows * H;
  float4 v[4];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = (threadIdx.x + j * blockDim.x) * 4;
    if (c < H) {
      float4 a = *reinterpret_cast<const float4*>(x + (int64_t)row * H + c);
      const int ns = sk_L > 0 ? sk_slots(c / 128, sk_kbt, sk_L) : splits;
      for (int s = 0; s < ns; ++s) {
        const float4 p = *reinterpret_cast<const float4*>(part + s * plane + (int64_t)row * H + c);
        a.x += p.x; a.y += p.y; a.z += p.z; a.w += p.w;
      }
      *reinterpret_cast<float4*>(x + (int64_t)row * H + c) = a;
      ss += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w;
      v[j] = a;
    }
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / H + eps);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = (threadIdx.x + j * blockDim.x) * 4;
    if (c < H) {
      const uint2 gv = *reinterpret_cast<const uint2*>(gamma + c);
      uint2 o;
      o.x = pack_bf16x2(v[j].x * inv * bf16_lo(gv.x), v[j].y * inv * bf16_hi(gv.x));
      o.y = pack_bf16x2(v[j].z * inv * bf16_lo(gv.y), v[j].w * inv * bf16_hi(gv.y));
      *reinterpret_cast<uint2*>(out + (int64_t)row * H + c) = o;
    }
  }
}

cudaError_t splitk_resid_rmsnorm_launch(const float* part, int splits, int rows, float* x, const bf16* gamma,
                                        bf16* out, int H, float eps, cudaStream_t s, int sk_L, int sk_kbt) {
  if (rows == 0) return cudaSuccess;
  // one float4 per thread up to H = 4096 (more loads in flight: only `rows` CTAs run)
  const int threads = H >= 4096 ? 1024 : (H >= 1024 ? 256 : 64);
  if (H % 4 || H > threads * 16) return cudaErrorInvalidValue;
  return launch_k(splitk_resid_rmsnorm_kernel, dim3(rows), dim3(threads), 0, s, part, splits, rows, x, gamma, out, H,
                  eps, sk_L, sk_kbt);
}

// TP=2 all-reduce fused with the residual add and the next RMSNorm, over NVLink peer
// memory. The exchange itself rides in the
// epilogue of the O / down projection: every output tile of rank r is stored both into
// this rank's receive plane recv[par][r] and, over NVLink, into the peer's recv[par][r]
// (GemmEpi::out2), tile by tile while the GEMM still runs. This kernel then
//   1. signals the peer that this rank's GEMM is complete (every CTA: fence.sys,
//      st.release.sys flag := epoch -- the GEMM grid finished before pdl_wait returns),
//   2. waits until the peer's flag reaches the epoch (its pushes are in our HBM),
//   3. x = (x + acc_0) + acc_1 (rank order -> bitwise identical on both ranks, the same
//      sum the NCCL path forms), h = rmsnorm(x) * gamma.
// Receive planes are double-buffered by epoch parity; a rank is at most one exchange
// ahead of its peer (it waits for the peer's flag of every exchange), and epochs only
// grow, so the wait is `flag >= epoch`.
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until *flag >= epoch (ge) or == epoch. Bounded: if the peer never signals (it
// returned early on an error, so the epochs diverged) the wait gives up after
// timeout_ns, sets *err and lets the kernel finish; the host reads err after the step,
// marks the instance dead and reports it instead of hanging the GPU.
__device__ __forceinline__ void tp_wait_flag(const int* flag, int epoch, bool ge, int* err,
                                             unsigned long long timeout_ns) {
  unsigned long long t0 = 0;
  for (int it = 0;; ++it) {
    const int v = ld_acquire_sys(flag);
    if (ge ? v >= epoch : v == epoch) return;
    if ((it & 255) == 0) {
      const unsigned long long t = global_ns();
      if (it == 0) t0 = t;
      else if (t - t0 > timeout_ns) {
        atomicExch(err, 1);
        return;
      }
    }
  }
}

__global__ void __launch_bounds__(1024) tp_allreduce_norm_kernel(TpAllreduceArgs a) {
  pdl_trigger();
  pdl_wait();
  const int H = a.H;
  __shared__ float red[32];
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(a.peer_flag, a.epoch);
    tp_wait_flag(a.my_flag, a.epoch, true, a.err, a.timeout_ns);
  }
  __syncthreads();
  for (int row = blockIdx.x; row < a.rows; row += gridDim.x) {
    float4 v[4];
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = (threadIdx.x + j * blockDim.x) * 4;
      if (c < H) {
        const int64_t off = (int64_t)row * H + c, plane = (int64_t)a.rows * H;
        float4 a0 = __ldcg(reinterpret_cast<const float4*>(a.recv0 + off));
        float4 a1 = __ldcg(reinterpret_cast<const float4*>(a.recv1 + off));
        for (int sp = 1; sp < a.splits; ++sp) {  // split order, as the per-row path sums them
          const float4 p0 = __ldcg(reinterpret_cast<const float4*>(a.recv0 + sp * plane + off));
          const float4 p1 = __ldcg(reinterpret_cast<const float4*>(a.recv1 + sp * plane + off));
          a0.x += p0.x; a0.y += p0.y; a0.z += p0.z; a0.w += p0.w;
          a1.x += p1.x; a1.y += p1.y; a1.z += p1.z; a1.w += p1.w;
        }
        float4 xv = *reinterpret_cast<const float4*>(a.x + off);
        xv.x = (xv.x + a0.x) + a1.x;
        xv.y = (xv.y + a0.y) + a1.y;
        xv.z = (xv.z + a0.z) + a1.z;
        xv.w = (xv.w + a0.w) + a1.w;
        *reinterpret_cast<float4*>(a.x + off) = xv;
        ss += xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
        v[j] = xv;
      }
    }
    if (!a.gamma) continue;  // block-uniform
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    const float inv = rsqrtf(red[0] / H + a.eps);
    __syncthreads();  // red[] reused by the next row
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = (threadIdx.x + j * blockDim.x) * 4;
      if (c < H) {
        const uint2 gv = *reinterpret_cast<const uint2*>(a.gamma + c);
        uint2 o;
        o.x = pack_bf16x2(v[j].x * inv * bf16_lo(gv.x), v[j].y * inv * bf16_hi(gv.x));
        o.y = pack_bf16x2(v[j].z * inv * bf16_lo(gv.y), v[j].w * inv * bf16_hi(gv.y));
        *reinterpret_cast<uint2*>(a.h + (int64_t)row * H + c) = o;
      }
    }
  }
}

cudaError_t tp_allreduce_norm_launch(const TpAllreduceArgs& a, int num_sms, cudaStream_t s) {
  if (a.rows == 0) return cudaSuccess;
  const int threads = a.H >= 4096 ? 1024 : (a.H >= 1024 ? 256 : 64);
  if (a.H % 4 || a.H > threads * 16) return cudaErrorInvalidValue;
  // every CTA spins on the peer's flag: keep the grid co-resident (rows are grid-strided)
  const int per_sm = threads >= 1024 ? 1 : 2;
  const int grid = a.rows < per_sm * num_sms ? a.rows : per_sm * num_sms;
  return launch_k(tp_allreduce_norm_kernel, dim3(grid), dim3(threads), 0, s, a);
}

// Decode variant (B rows): the projection's split-K partials stay in this GPU's L2 and
// one CTA per token row sums them (split order), pushes the row to the peer's receive
// row (P2P stores), fence.sys + a per-row flag := epoch, waits for the peer's row and
// forms x = (x + acc_0) + acc_1 and the next RMSNorm. At decode sizes (a 32 KB row per
// CTA) this beats pushing from the GEMM epilogue, which measured 30.3 vs 24.4 ms per
// 70B TP=2 step: the in-GEMM split reduction and 128-byte remote stores sit on the tail.
__global__ void __launch_bounds__(1024) tp_push_rows_kernel(TpRowsArgs a) {
  pdl_trigger();
  pdl_wait();
  const int H = a.H;
  __shared__ float red[32];
  for (int row = blockIdx.x; row < a.rows; row += gridDim.x) {
    float4 v[4];
    // 1) this rank's partial of the row, pushed to the peer
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = (threadIdx.x + j * blockDim.x) * 4;
      if (c < H) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const int ns = a.sk_L > 0 ? sk_slots(c / 128, a.sk_kbt, a.sk_L) : a.splits;
        for (int s = 0; s < ns; ++s) {
          const float4 p = *reinterpret_cast<const float4*>(a.part + s * a.plane + (int64_t)row * a.ldp + c);
          acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
        }
        v[j] = acc;
        *reinterpret_cast<float4*>(a.peer_recv + (int64_t)row * H + c) = acc;
      }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      st_release_sys(a.peer_flags + row, a.epoch);
      tp_wait_flag(a.my_flags + row, a.epoch, false, a.err, a.timeout_ns);
    }
    __syncthreads();
    // 2) x = (x + acc_0) + acc_1
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = (threadIdx.x + j * blockDim.x) * 4;
      if (c < H) {
        const float4 o = __ldcv(reinterpret_cast<const float4*>(a.my_recv + (int64_t)row * H + c));
        const float4 a0 = a.rank == 0 ? v[j] : o, a1 = a.rank == 0 ? o : v[j];
        float4 xv = *reinterpret_cast<const float4*>(a.x + (int64_t)row * H + c);
        xv.x = (xv.x + a0.x) + a1.x;
        xv.y = (xv.y + a0.y) + a1.y;
        xv.z = (xv.z + a0.z) + a1.z;
        xv.w = (xv.w + a0.w) + a1.w;
        *reinterpret_cast<float4*>(a.x + (int64_t)row * H + c) = xv;
        ss += xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
        v[j] = xv;
      }
    }
    if (!a.gamma) continue;  // block-uniform
    // 3) h = rmsnorm(x) * gamma
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (threadIdx.x == 0) red[0] = t;
    }
    __syncthreads();
    const float inv = rsqrtf(red[0] / H + a.eps);
    __syncthreads();  // red[] reused by the next row
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = (threadIdx.x + j * blockDim.x) * 4;
      if (c < H) {
        const uint2 gv = *reinterpret_cast<const uint2*>(a.gamma + c);
        uint2 o;
        o.x = pack_bf16x2(v[j].x * inv * bf16_lo(gv.x), v[j].y * inv * bf16_hi(gv.x));
        o.y = pack_bf16x2(v[j].z * inv * bf16_lo(gv.y), v[j].w * inv * bf16_hi(gv.y));
        *reinterpret_cast<uint2*>(a.h + (int64_t)row * H + c) = o;
      }
    }
  }
}

cudaError_t tp_push_rows_launch(const TpRowsArgs& a, int num_sms, cudaStream_t s) {
  if (a.rows == 0) return cudaSuccess;
  const int threads = a.H >= 4096 ? 1024 : (a.H >= 1024 ? 256 : 64);
  if (a.H % 4 || a.H > threads * 16) return cudaErrorInvalidValue;
  // every CTA co-resident (rows are grid-strided): the two ranks wait on each other row by row
  const int per_sm = threads >= 1024 ? 1 : 2;
  const int grid = a.rows < per_sm * num_sms ? a.rows : per_sm * num_sms;
  return launch_k(tp_push_rows_kernel, dim3(grid), dim3(threads), 0, s, a);
}

__device__ __forceinline__ float silu_r(float z) { return __fdividef(z, 1.f + __expf(-z)); }

// part [split][row][ld_part] f32; one thread per (row, column pair).
__global__ void splitk_reduce_kernel(int mode, const float* __restrict__ part, int splits, int rows, int cols,
                                     int64_t ld_part, GemmEpi e) {
  pdl_trigger();
  pdl_wait();
  const int pairs = cols / 2;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)rows * pairs) return;
  const int row = gid / pairs, c = 2 * (int)(gid % pairs);
  float a = 0.f, b = 0.f;
  const int64_t plane = (int64_t)rows * ld_part;
  const int ns = e.sk_L > 0 ? sk_slots(c / 128, e.sk_kbt, e.sk_L) : splits;
  for (int s = 0; s < ns; ++s) {  // fixed order: deterministic
    const float2 v = *reinterpret_cast<const float2*>(part + s * plane + (int64_t)row * ld_part + c);
    a += v.x;
    b += v.y;
  }
  switch (mode) {
    case RED_F32: {
      float* o = reinterpret_cast<float*>(e.out) + (int64_t)row * e.ldo + c;
      o[0] = a;
      o[1] = b;
    } break;
    case RED_BF16:
      *reinterpret_cast<uint32_t*>(reinterpret_cast<bf16*>(e.out) + (int64_t)row * e.ldo + c) = pack_bf16x2(a, b);
      break;
    case RED_RESID: {
      float2* o = reinterpret_cast<float2*>(e.resid + (int64_t)row * e.ldr + c);
      float2 r = *o;
      r.x += a;
      r.y += b;
      *o = r;
    } break;
    case RED_SILU:
      reinterpret_cast<bf16*>(e.out)[(int64_t)row * e.ldo + c / 2] = __float2bfloat16_rn(silu_r(a) * b);
      break;
    case RED_QKV: {
      if (e.rvec) {  // deferred RMSNorm: the input was bf16(x * gamma)
        const float r = e.rvec[row];
        a *= r;
        b *= r;
      }
      const int D = e.head_dim, half = D / 2;
      const int qd = e.n_heads * D, kd = e.n_kv * D;
      if (c < qd + kd) {
        const bool is_q = c < qd;
        const int head = is_q ? c / D : (c - qd) / D;
        const int j = (c % D) / 2;
        const int p = e.pos[row];
        const float cs = e.rope_cos[(int64_t)p * half + j], sn = e.rope_sin[(int64_t)p * half + j];
        bf16* dst;
        if (is_q) {
          dst = e.q_out + ((int64_t)row * e.n_heads + head) * D;
        } else {
          const int s = e.slot[row];
          dst = e.k_cache + (int64_t)(s >> 6) * e.blk_stride + ((int64_t)head * 64 + (s & 63)) * D;
        }
        dst[j] = __float2bfloat16_rn(a * cs - b * sn);
        dst[j + half] = __float2bfloat16_rn(b * cs + a * sn);
      } else {
        const int cc = c - qd - kd;
        const int head = cc / D, d = cc % D;
        const int s = e.slot[row];
        bf16* dst = e.v_cache + (int64_t)(s >> 6) * e.blk_stride + ((int64_t)head * 64 + (s & 63)) * D + d;
        *reinterpret_cast<uint32_t*>(dst) = pack_bf16x2(a, b);
      }
    } break;
    default:
      break;
  }
}

cudaError_t splitk_reduce_launch(int mode, const float* part, int splits, int rows, int cols, int64_t ld_part,
                                 const GemmEpi& epi, cudaStream_t s) {
  const int64_t n = (int64_t)rows * (cols / 2);
  if (n == 0) return cudaSuccess;
  if (cols % 2) return cudaErrorInvalidValue;
  const int threads = 256;
  return launch_k(splitk_reduce_kernel, dim3((unsigned)((n + threads - 1) / threads)), dim3(threads), 0, s, mode, part,
                  splits, rows, cols, ld_part, epi);
}

}  // namespace eco
