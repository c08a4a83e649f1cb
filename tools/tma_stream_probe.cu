// Probe: HBM streaming bandwidth of TMA tile loads (no MMA) for the decode-GEMM
// weight access pattern. Each of `grid` CTAs streams K/64 tiles of 128 rows x 64
// bf16 (16 KB) through an S-stage mbarrier ring, either from a row-major [N][K]
// matrix (2D map: each tile = 128 rows x 128 B, rows K*2 bytes apart) or from a
// tile-contiguous copy [N/128][K/64][128][64] (4D map: each tile 16 KB contiguous).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_probe tools/tma_stream_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../paper_2504_18154_b200/csrc/common.cuh"

using namespace eco;

template <int S, bool TILED>
__global__ void stream_kernel(const __grid_constant__ CUtensorMap map, int n_tiles_m, int kb_total, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * 16384);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int acc = 0;
  const int total = n_tiles_m * kb_total;
  int issued = 0, done = 0;
  // iterations of this CTA: it = blockIdx.x + k * gridDim.x over (mt, kb) with kb fastest
  auto coords = [&](int it, int& mt, int& kb) { mt = it / kb_total; kb = it % kb_total; };
  int it_issue = blockIdx.x, it_done = blockIdx.x;
  for (int s = 0; s < S && it_issue < total; ++s, it_issue += gridDim.x, ++issued) {
    int mt, kb;
    coords(it_issue, mt, kb);
    mbar_arrive_expect_tx(&full[s], 16384);
    if (TILED)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
          ::"r"(smem_u32(smem + s * 16384)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(0), "r"(kb), "r"(mt),
          "r"(smem_u32(&full[s])) : "memory");
    else
      tma_load_2d(smem + s * 16384, &map, &full[s], kb * 64, mt * 128);
  }
  uint32_t phase = 0;
  int s = 0;
  while (it_done < total) {
    mbar_wait(&full[s], phase);
    acc += smem[s * 16384 + (done & 1023)];
    ++done;
    it_done += gridDim.x;
    if (it_issue < total) {
      int mt, kb;
      coords(it_issue, mt, kb);
      mbar_arrive_expect_tx(&full[s], 16384);
      if (TILED)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
            ::"r"(smem_u32(smem + s * 16384)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(0), "r"(kb), "r"(mt),
            "r"(smem_u32(&full[s])) : "memory");
      else
        tma_load_2d(smem + s * 16384, &map, &full[s], kb * 64, mt * 128);
      it_issue += gridDim.x;
    }
    if (++s == S) { s = 0; phase ^= 1; }
  }
  if (acc == 12345678) *sink = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int S, bool TILED>
float run(const CUtensorMap& m, int mt, int kb, int grid, int* sink) {
  const int smem = S * 16384 + 2048;
  cudaFuncSetAttribute(stream_kernel<S, TILED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) stream_kernel<S, TILED><<<grid, 32, smem>>>(m, mt, kb, sink);
  cudaEventRecord(a);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) stream_kernel<S, TILED><<<grid, 32, smem>>>(m, mt, kb, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const int N = 28672 * 4, K = 4096;  // 939 MB: larger than L2, like a layer's worth of weights x4
  void* w;
  cudaMalloc(&w, (size_t)N * K * 2);
  cudaMemset(w, 1, (size_t)N * K * 2);
  int* sink;
  cudaMalloc(&sink, 4);
  auto e = enc();
  CUtensorMap m2, m4;
  {
    cuuint64_t d[2] = {(cuuint64_t)K, (cuuint64_t)N}, st[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    e(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t d[4] = {64, 128, (cuuint64_t)K / 64, (cuuint64_t)N / 128};
    cuuint64_t st[3] = {64 * 2, 128 * 64 * 2, (cuuint64_t)(K / 64) * 128 * 64 * 2};
    cuuint32_t box[4] = {64, 128, 1, 1}, es[4] = {1, 1, 1, 1};
    e(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, w, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  const int mt = N / 128, kb = K / 64;
  const double gb = (double)N * K * 2 / 1e9;
  for (int grid : {38, 76, 112, 148, 296}) {  // fewer CTAs: the per-SM streaming cap
    printf("{\"grid\": %d, \"rowmajor_s6\": %.1f, \"tiled_s6\": %.1f, \"rowmajor_s12\": %.1f, \"tiled_s12\": %.1f}\n", grid,
           gb / run<6, false>(m2, mt, kb, grid, sink) * 1e3, gb / run<6, true>(m4, mt, kb, grid, sink) * 1e3,
           gb / run<12, false>(m2, mt, kb, grid, sink) * 1e3, gb / run<12, true>(m4, mt, kb, grid, sink) * 1e3);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
