#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void fma2(float2& d, float2 a, float2 b) {
  unsigned long long dd, aa, bb;
  aa = *reinterpret_cast<unsigned long long*>(&a); bb = *reinterpret_cast<unsigned long long*>(&b);
  dd = *reinterpret_cast<unsigned long long*>(&d);
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(dd) : "l"(aa), "l"(bb));
  d = *reinterpret_cast<float2*>(&dd);
}
__global__ void k2(float* out, int iters, float s) {
  float2 a[8], x = make_float2(threadIdx.x * 1e-3f, s), y = make_float2(s, threadIdx.x * 2e-3f);
  for (int j = 0; j < 8; ++j) a[j] = make_float2(j, -j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) fma2(a[j], x, y);
  }
  float t = 0; for (int j = 0; j < 8; ++j) t += a[j].x + a[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k1(float* out, int iters, float s) {
  float a[16], x = threadIdx.x * 1e-3f, y = s;
  for (int j = 0; j < 16; ++j) a[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], x, y + 0.f * j);
  }
  float t = 0; for (int j = 0; j < 16; ++j) t += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int it = 1 << 14;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k2<<<148 * 4, 256>>>(d, it, 1.0001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("f32x2: %.1f TFLOP/s\n", 2.0 * 16 * it * 148.0 * 4 * 256 / ms / 1e9);
    cudaEventRecord(e0); k1<<<148 * 4, 256>>>(d, it, 1.0001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ffma 3-reg: %.1f TFLOP/s\n", 2.0 * 16 * it * 148.0 * 4 * 256 / ms / 1e9);
  }
  return 0;
}
