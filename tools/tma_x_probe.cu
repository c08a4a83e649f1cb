// Probe: does the decode GEMM's activation re-read limit it? Each CTA streams W
// tiles (128 rows x 64 bf16 = 16 KB) of a [N][K] weight like the swap-AB decode
// GEMM, optionally together with the matching X tile (B=128 rows x 64 of a
// [128][K] activation, 16 KB, the same for every W tile -> served from L2), and
// optionally with X multicast across a CS-CTA cluster (each CTA loads 128/CS rows
// of X and multicasts them, so L2->SM traffic for X drops by CS).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_x_probe tools/tma_x_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2504_18154_b200/csrc/common.cuh"

using namespace eco;

__device__ __forceinline__ void tma_mc_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                          uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void arrive_remote(uint64_t* bar, uint32_t cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}

// MODE 0: W only; 1: W + X; 2: W + X multicast over the cluster (CS CTAs)
template <int S, int MODE, int CS>
__global__ void probe_kernel(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
                             int n_tiles_m, int kb_total, int* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int STAGE = MODE == 0 ? 16384 : 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
  uint64_t* empty = full + S;
  const uint32_t rank = CS > 1 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CS);
    }
    fence_barrier_init();
  }
  if (CS > 1) cluster_sync(); else __syncthreads();
  if (threadIdx.x == 0) {
    // cluster c walks tile groups g = c, c + n_clusters, ...; CTA rank r takes W tile g*CS + r
    const int n_clusters = gridDim.x / CS, cid = blockIdx.x / CS;
    const int groups = n_tiles_m / CS;
    const int per = ((groups - cid + n_clusters - 1) / n_clusters) * kb_total;  // iterations of this CTA
    auto issue = [&](int it, int s) {
      const int g = cid + (it / kb_total) * n_clusters, kb = it % kb_total;
      const int mt = g * CS + rank;
      mbar_arrive_expect_tx(&full[s], STAGE);
      tma_load_2d(smem + s * STAGE, &wmap, &full[s], kb * 64, mt * 128);
      if (MODE == 1) tma_load_2d(smem + s * STAGE + 16384, &xmap, &full[s], kb * 64, 0);
      if (MODE == 2)
        tma_mc_2d(smem + s * STAGE + 16384 + rank * (16384 / CS), &xmap, &full[s], kb * 64, rank * (128 / CS),
                  (uint16_t)((1u << CS) - 1));
    };
    int acc = 0;
    for (int it = 0; it < S && it < per; ++it) issue(it, it);
    for (int it = 0; it < per; ++it) {
      const int s = it % S;
      const uint32_t ph = (it / S) & 1;
      mbar_wait(&full[s], ph);
      acc += smem[s * STAGE + (it & 1023)];
      if (CS > 1) {
        for (int c = 0; c < CS; ++c) arrive_remote(&empty[s], c);
      } else {
        mbar_arrive(&empty[s]);
      }
      if (it + S < per) {
        mbar_wait(&empty[s], ph);
        issue(it + S, s);
      }
    }
    if (acc == 12345678) *sink = acc;
  }
  if (CS > 1) cluster_sync();
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int S, int MODE, int CS>
float run(const CUtensorMap& w, const CUtensorMap& x, int mt, int kb, int* sink, int grid = 148) {
  constexpr int STAGE = MODE == 0 ? 16384 : 32768;
  const int smem = S * STAGE + 2048;
  auto k = probe_kernel<S, MODE, CS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) cudaLaunchKernelEx(&cfg, k, w, x, mt, kb, sink);
  cudaEventRecord(a);
  const int reps = 10;
  for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, k, w, x, mt, kb, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms / reps;
}

int main() {
  const int N = 28672, K = 4096, B = 128;  // the Llama-3-8B gate/up projection, B = 128
  void *w, *x;
  cudaMalloc(&w, (size_t)N * K * 2);
  cudaMalloc(&x, (size_t)B * K * 2);
  cudaMemset(w, 1, (size_t)N * K * 2);
  cudaMemset(x, 1, (size_t)B * K * 2);
  int* sink;
  cudaMalloc(&sink, 4);
  auto e = enc();
  CUtensorMap wm, xm, xm2, xm4;
  auto mk = [&](CUtensorMap* m, void* p, int rows, int box_rows) {
    cuuint64_t d[2] = {(cuuint64_t)K, (cuuint64_t)rows}, st[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, es[2] = {1, 1};
    e(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, d, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  mk(&wm, w, N, 128);
  mk(&xm, x, B, 128);
  mk(&xm2, x, B, 64);
  mk(&xm4, x, B, 32);
  const int mt = N / 128, kb = K / 64;
  const double gb = (double)N * K * 2 / 1e9;
  for (int grid : {148, 112, 74})
    printf("{\"grid\": %d, \"w_x_s6\": %.1f}\n", grid, gb / run<6, 1, 1>(wm, xm, mt, kb, sink, grid) * 1e3);
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
