// Where does a decode GEMM's time go? Runs the engine's swap-AB decode GEMM
// (gemm_tc_kernel, linked from the product source) on the Llama-3-8B projection
// shapes at B = 128 with per-CTA %globaltimer marks (GemmEpi::trace):
//   0 CTA start, 1 prologue done, 2 first stage landed, 3 last MMA issued, 4 epilogue done.
// Weights rotate over 8 copies so every launch streams from HBM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gemm_trace tools/gemm_trace.cu \
//          paper_2504_18154_b200/csrc/gemm_sm100.cu -lcuda
#include <cuda_runtime.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "../paper_2504_18154_b200/csrc/kernels.h"

using namespace eco;

__global__ void fill_kernel(bf16* p, size_t n, uint32_t seed, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    p[i] = __float2bfloat16_rn(((h & 0xffff) / 32768.f - 1.f) * scale);
  }
}

struct Shape {
  const char* name;
  int m, k, mode;
};

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int B = 128, COPIES = 8;
  printf("{\"max_active_clusters\": {\"2\": %d, \"3\": %d, \"4\": %d}}\n", gemm_cluster_max_active(128, 2),
         gemm_cluster_max_active(128, 3), gemm_cluster_max_active(128, 4));
  Shape shapes[] = {{"qkv", 6144, 4096, EPI_SWAP_F32}, {"o", 4096, 4096, EPI_SWAP_F32},
                    {"gu", 28672, 4096, EPI_SWAP_SILU}, {"down", 4096, 14336, EPI_SWAP_F32}};
  bf16* x;
  cudaMalloc(&x, (size_t)B * 14336 * 2);
  fill_kernel<<<1024, 256>>>(x, (size_t)B * 14336, 7u, 1.f);
  float* part;
  cudaMalloc(&part, (size_t)8 * B * 28672 * 4);
  bf16* act;
  cudaMalloc(&act, (size_t)B * 14336 * 2);
  unsigned long long* trace;
  cudaMalloc(&trace, 16 * 1024 * 8);
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (const Shape& sh : shapes) {
    std::vector<bf16*> w(COPIES);
    std::vector<CUtensorMap> wm(COPIES);
    for (int c = 0; c < COPIES; ++c) {
      cudaMalloc(&w[c], (size_t)sh.m * sh.k * 2);
      fill_kernel<<<4096, 256>>>(w[c], (size_t)sh.m * sh.k, 11u + c, 0.03f);
      make_tmap_bf16(&wm[c], w[c], sh.m, sh.k, 128);
    }
    CUtensorMap xm;
    make_tmap_bf16(&xm, x, B, sh.k, 128);
    for (int splits_req : {0, 2, 3, 4}) {
      int splits = splits_req == 0 ? gemm_decode_splits(sh.m, sh.k, sms) : splits_req;
      if (sh.mode == EPI_SWAP_SILU && splits > 1) continue;
      GemmEpi e;
      memset(&e, 0, sizeof(e));
      e.mode = sh.mode;
      e.out = sh.mode == EPI_SWAP_F32 ? (void*)part : (void*)act;
      e.ldo = sh.mode == EPI_SWAP_F32 ? sh.m : sh.m / 2;
      e.indep = 1;
      auto launch = [&](int i, unsigned long long* tr) {
        e.trace = tr;
        return gemm_launch_r(&wm[i % COPIES], &xm, sh.m, B, sh.k, 128, 1, splits, e, sms, st);
      };
      if (sh.mode == EPI_SWAP_F32 && splits >= 2 && splits <= 4) {
        // the cluster split-K variant (DSMEM reduction + epilogue in one kernel), f32 store epilogue
        GemmEpi ec;
        memset(&ec, 0, sizeof(ec));
        ec.mode = EPI_SWAP_STORE;
        ec.resid = part;
        ec.ldr = sh.m;
        ec.indep = 1;
        const int eff = gemm_effective_splits(sh.k, splits);
        for (int i = 0; i < 8; ++i) gemm_cluster_launch(&wm[i % COPIES], &xm, sh.m, B, sh.k, 128, eff, ec, st);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
        for (int i = 0; i < 40; ++i) gemm_cluster_launch(&wm[i % COPIES], &xm, sh.m, B, sh.k, 128, eff, ec, st);
        cudaEventRecord(b, st);
        cudaError_t err = cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        // traced launch: epilogue phases of the cluster kernel
        cudaStreamSynchronize(st);
        cudaMemset(trace, 0, 16 * 1024 * 8);
        ec.trace = trace;
        gemm_cluster_launch(&wm[3], &xm, sh.m, B, sh.k, 128, eff, ec, st);
        ec.trace = nullptr;
        cudaStreamSynchronize(st);
        const int cgrid = ((sh.m + 127) / 128) * eff;
        std::vector<unsigned long long> tc(cgrid * 16);
        cudaMemcpy(tc.data(), trace, cgrid * 16 * 8, cudaMemcpyDeviceToHost);
        unsigned long long T0 = ~0ull, T1 = 0;
        double mma = 0, epi = 0, first = 0;
        for (int c = 0; c < cgrid; ++c) {
          T0 = std::min(T0, tc[c * 16]);
          T1 = std::max(T1, tc[c * 16 + 4]);
        }
        double last_start = 0;
        for (int c = 0; c < cgrid; ++c) {
          const unsigned long long* r = &tc[c * 16];
          first += (double)(r[2] - r[0]);
          mma += (double)(r[3] - r[2]);
          epi += (double)(r[4] - r[5]);
          last_start = std::max(last_start, (double)(r[0] - T0));
        }
        printf("{\"op\": \"%s\", \"variant\": \"cluster\", \"splits\": %d, \"us_stream\": %.2f, \"gbs_stream\": %.0f, "
               "\"span_us\": %.2f, \"last_cta_start_us\": %.2f, \"avg_first_us\": %.2f, \"avg_mma_us\": %.2f, \"avg_epi_us\": %.2f, \"err\": \"%s\"}\n",
               sh.name, eff, ms * 1e3 / 40, (double)sh.m * sh.k * 2 / 1e9 / (ms / 40) * 1e3, (T1 - T0) / 1e3,
               last_start / 1e3, first / cgrid / 1e3, mma / cgrid / 1e3, epi / cgrid / 1e3, cudaGetErrorString(err));
      }
      for (int i = 0; i < 8; ++i) launch(i, nullptr);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      const int reps = 40;
      cudaEventRecord(a, st);
      for (int i = 0; i < reps; ++i) launch(i, nullptr);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      // one traced launch, isolated (previous work drained)
      cudaStreamSynchronize(st);
      cudaMemset(trace, 0, 16 * 1024 * 8);
      launch(3, trace);
      cudaError_t err = cudaStreamSynchronize(st);
      const int tiles = (sh.m + 127) / 128;
      const int grid = std::min(tiles * gemm_effective_splits(sh.k, splits), sms);
      std::vector<unsigned long long> t(grid * 16);
      cudaMemcpy(t.data(), trace, grid * 16 * 8, cudaMemcpyDeviceToHost);
      unsigned long long T0 = ~0ull, Tend = 0;
      double s_pro = 0, s_first = 0, s_mma = 0, s_epi = 0, m_start = 0, m_first = 0, s_acc = 0, s_ep = 0, s_ld = 0;
      for (int c = 0; c < grid; ++c) {
        T0 = std::min(T0, t[c * 16 + 0]);
        Tend = std::max(Tend, t[c * 16 + 4]);
      }
      double s_c[4] = {0, 0, 0, 0};
      for (int c = 0; c < grid; ++c) {
        const unsigned long long* r = &t[c * 16];
        s_pro += (double)(r[1] - r[0]);
        s_first += (double)(r[2] - r[1]);
        s_mma += (double)(r[3] - r[2]);
        s_epi += (double)(r[4] - r[3]);
        s_acc += (double)(r[5] - r[3]);   // last MMA issued -> (last) accumulator ready
        s_ep += (double)(r[4] - r[5]);    // (last) epilogue work
        s_ld += (double)(r[3] - r[6]);    // last load issued -> last MMA issued
        s_c[0] += r[8]; s_c[1] += r[9]; s_c[2] += r[10]; s_c[3] += r[11];
        m_start = std::max(m_start, (double)(r[0] - T0));
        m_first = std::max(m_first, (double)(r[2] - T0));
      }
      const double gb = (double)sh.m * sh.k * 2 / 1e9;
      printf("{\"op\": \"%s\", \"splits\": %d, \"grid\": %d, \"us_stream\": %.2f, \"gbs_stream\": %.0f, "
             "\"traced_span_us\": %.2f, \"last_cta_start_us\": %.2f, \"avg_prologue_us\": %.2f, "
             "\"avg_first_data_us\": %.2f, \"last_first_data_us\": %.2f, \"avg_mma_span_us\": %.2f, "
             "\"avg_epilogue_tail_us\": %.2f, \"avg_acc_ready_us\": %.2f, \"avg_epi_work_us\": %.2f, \"avg_lastload_to_lastmma_us\": %.2f, \"err\": \"%s\"}\n",
             sh.name, splits, grid, ms * 1e3 / reps, gb / (ms / reps) * 1e3, (Tend - T0) / 1e3, m_start / 1e3,
             s_pro / grid / 1e3, s_first / grid / 1e3, m_first / 1e3, s_mma / grid / 1e3, s_epi / grid / 1e3,
             s_acc / grid / 1e3, s_ep / grid / 1e3, s_ld / grid / 1e3, cudaGetErrorString(err));
      printf("  epilogue cycles (thread 64, last tile): wait_staging %.0f tmem_ld %.0f math+sts %.0f bar+bulk %.0f\n",
             s_c[0] / grid, s_c[1] / grid, s_c[2] / grid, s_c[3] / grid);
      fflush(stdout);
    }
    for (int c = 0; c < COPIES; ++c) cudaFree(w[c]);
  }
  return 0;
}
