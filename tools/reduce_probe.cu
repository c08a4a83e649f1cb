// Probe: time the decode-flow O-tile reduction pattern in isolation (32 CTAs x 128
// threads; each CTA sums 5 contributor slots [128 tok][128 f32] + x and writes x, h),
// scalar per-feature loads (the flow kernel's mapping) vs float4 loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/reduce_probe tools/reduce_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void red_scalar(const float* slots, float* x, __nv_bfloat16* h, int H, int B, int nc) {
  const int t = blockIdx.x, row = threadIdx.x;
  const int feat = t * 128 + row;
  for (int c0 = 0; c0 < B; c0 += 32) {
    float f[32], xv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) f[i] = 0.f;
    for (int c = 0; c < nc; ++c) {
      const float* sl = slots + ((size_t)(t * 8 + c)) * 128 * 128;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (c0 + i < B) f[i] += sl[(c0 + i) * 128 + row];
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) xv[i] = (c0 + i < B) ? x[(size_t)(c0 + i) * H + feat] : 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (c0 + i < B) {
        x[(size_t)(c0 + i) * H + feat] = xv[i] + f[i];
        h[(size_t)(c0 + i) * H + feat] = __float2bfloat16_rn(xv[i] + f[i]);
      }
  }
}

__global__ void red_vec4(const float* slots, float* x, __nv_bfloat16* h, int H, int B, int nc) {
  const int t = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f0 = lane * 4;
  for (int tok = w; tok < B; tok += 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = 0; c < nc; ++c) {
      const float4 v = *reinterpret_cast<const float4*>(slots + ((size_t)(t * 8 + c)) * 128 * 128 + tok * 128 + f0);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    float4* xp = reinterpret_cast<float4*>(x + (size_t)tok * H + t * 128 + f0);
    float4 xv = *xp;
    xv.x += acc.x; xv.y += acc.y; xv.z += acc.z; xv.w += acc.w;
    *xp = xv;
  }
}

int main() {
  const int H = 4096, B = 128, T = 32, NC = 5;
  float *slots, *x;
  __nv_bfloat16* h;
  cudaMalloc(&slots, sizeof(float) * T * 8 * 128 * 128);
  cudaMalloc(&x, sizeof(float) * B * H);
  cudaMalloc(&h, 2 * B * H);
  cudaMemset(slots, 0, sizeof(float) * T * 8 * 128 * 128);
  cudaMemset(x, 0, sizeof(float) * B * H);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int k = 0; k < 3; ++k) {
    float ms;
    cudaEventRecord(a);
    red_scalar<<<T, 128>>>(slots, x, h, H, B, NC);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("scalar: %.2f us\n", ms * 1e3);
    cudaEventRecord(a);
    red_vec4<<<T, 128>>>(slots, x, h, H, B, NC);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("vec4:   %.2f us\n", ms * 1e3);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
