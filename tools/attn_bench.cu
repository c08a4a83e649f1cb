// Prefill-attention kernel timing without host work in the loop: the tcgen05 kernel
// (attention_tc.cu) and the mma.sync FA2 kernel (attention.cu) on the Llama-3-8B head
// layout (M=32, Mkv=8, D=128) over a paged single-layer pool, configs[1]-like batches.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/attn_bench tools/attn_bench.cu \
//          paper_2504_18154_b200/csrc/attention_tc.cu paper_2504_18154_b200/csrc/attention.cu \
//          paper_2504_18154_b200/csrc/gemm_sm100.cu -lcuda
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

#include "../paper_2504_18154_b200/csrc/kernels.h"

using namespace eco;

__global__ void fill(bf16* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    p[i] = __float2bfloat16_rn(((h & 0xffff) / 32768.f - 1.f) * 1.7f);
  }
}

int main(int argc, char** argv) {
  const int M = 32, Mkv = 8, D = 128;
  // optional: the engine's block-major multi-layer pool [blk][L][2][Mkv][64][D], layer L/2
  const int L = argc > 1 ? atoi(argv[1]) : 1, layer = L / 2;
  std::mt19937 rng(0);
  std::vector<std::vector<int>> cfgs = {std::vector<int>(16, 512), {}, std::vector<int>(4, 2048), {8192}};
  for (int i = 0; i < 8; ++i) cfgs[1].push_back(512 + (int)(rng() % 1537));
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (auto& lens : cfgs) {
    const int n = (int)lens.size();
    std::vector<int> cu(n + 1, 0), nb(n);
    for (int i = 0; i < n; ++i) {
      cu[i + 1] = cu[i] + lens[i];
      nb[i] = (lens[i] + 63) / 64;
    }
    const int T = cu[n];
    int n_blocks = 8;
    int bt_ld = 0;
    for (int b : nb) { n_blocks += b; bt_ld = std::max(bt_ld, b); }
    std::vector<int> perm(n_blocks);
    for (int i = 0; i < n_blocks; ++i) perm[i] = i;
    std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<int> bt(n * bt_ld, 0), tiles;
    for (int i = 0, k = 0; i < n; ++i)
      for (int b = 0; b < nb[i]; ++b) bt[i * bt_ld + b] = perm[k++];
    for (int i = 0; i < n; ++i)
      for (int q = 0; q < lens[i]; q += 128) { tiles.push_back(i); tiles.push_back(q); }
    const int n_tiles = (int)tiles.size() / 2;
    bf16 *q, *pool, *out;
    const size_t pool_elems = (size_t)n_blocks * L * 2 * Mkv * 64 * D;
    cudaMalloc(&q, (size_t)T * M * D * 2);
    cudaMalloc(&pool, pool_elems * 2);
    cudaMalloc(&out, (size_t)T * M * D * 2);
    fill<<<1024, 256>>>(q, (size_t)T * M * D, 1);
    fill<<<1024, 256>>>(pool, pool_elems, 2);
    int *d_cu, *d_bt, *d_tiles;
    cudaMalloc(&d_cu, 4 * (n + 1));
    cudaMalloc(&d_bt, 4 * bt.size());
    cudaMalloc(&d_tiles, 4 * tiles.size());
    cudaMemcpy(d_cu, cu.data(), 4 * (n + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(d_bt, bt.data(), 4 * bt.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_tiles, tiles.data(), 4 * tiles.size(), cudaMemcpyHostToDevice);
    CUtensorMap qm, km;
    make_attn_tc_maps(&qm, &km, q, T, M, pool, (int64_t)n_blocks * L * 2 * Mkv * 64);
    PrefillAttnArgs a;
    a.q = q;
    a.k_cache = pool + (size_t)layer * 2 * Mkv * 64 * D;
    a.v_cache = a.k_cache + (size_t)Mkv * 64 * D;
    a.blk_stride = (int64_t)L * 2 * Mkv * 64 * D;
    a.cu_seqlens = d_cu;
    a.block_tables = d_bt;
    a.bt_ld = bt_ld;
    a.tiles = d_tiles;
    a.ctx_off = nullptr;
    a.n_tiles = n_tiles;
    a.out = out;
    a.n_heads = M;
    a.n_kv = Mkv;
    a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
    auto run_tc = [&]() {
      return attn_prefill_tc_launch(&qm, &km, d_cu, d_bt, bt_ld, d_tiles, n_tiles, out, M, Mkv, layer, L, st);
    };
    auto run_mma = [&]() { return attn_prefill_launch(a, D, st); };
    auto time = [&](auto fn) {
      for (int i = 0; i < 3; ++i) fn();
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        for (int i = 0; i < 10; ++i) fn();
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms / 10);
      }
      return best * 1e3f;
    };
    const float t_tc = time(run_tc), t_mma = time(run_mma);
    if (getenv("ATTN_TRACE") && n == 1) {   // per-block clock64 stamps of one 64-block CTA (tile 31)
      long long* d_tr;
      cudaMalloc(&d_tr, 20 * 64 * sizeof(long long));
      cudaMemset(d_tr, 0, 20 * 64 * sizeof(long long));
      attn_tc_set_trace(d_tr, 31);
      run_tc();
      cudaStreamSynchronize(st);
      attn_tc_set_trace(nullptr, 0);
      long long h[20 * 64];
      cudaMemcpy(h, d_tr, sizeof(h), cudaMemcpyDeviceToHost);
      const long long t0 = h[8 * 64];
      printf("# j: P stored by softmax warps 2..9 | S seen by warps 2..9 | P0, P1 seen by issuer | S(j+2) 0, 1 issued (cycles)\n");
      for (int j = 0; j < 64; ++j) {
        printf("%2d", j);
        for (int r = 0; r < 20; ++r) printf(" %7lld", h[r * 64 + j] ? h[r * 64 + j] - t0 : -1);
        printf("\n");
      }
      cudaFree(d_tr);
    }
    double flop = 0;
    for (int s : lens) flop += 2.0 * M * D * (double)s * (s + 1);  // causal QK^T + PV
    cudaError_t err = cudaStreamSynchronize(st);
    printf("{\"L\": %d, \"tokens\": %d, \"n_seq\": %d, \"tc_us\": %.1f, \"tc_tflops\": %.1f, \"mma_us\": %.1f, \"mma_tflops\": %.1f, "
           "\"err\": \"%s\"}\n",
           L, T, n, t_tc, flop / t_tc / 1e6, t_mma, flop / t_mma / 1e6, cudaGetErrorString(err));
    cudaFree(q); cudaFree(pool); cudaFree(out); cudaFree(d_cu); cudaFree(d_bt); cudaFree(d_tiles);
  }
  return 0;
}
