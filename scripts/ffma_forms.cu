// FFMA throughput by operand form on B200: uniform-register operand (as the
// bench's vm_ffma_peak probe compiles) vs all-vector-register operands (the
// form KF's micro-GEMMs use).
#include <cstdio>
__global__ void uform(float* out, int iters, float a, float b) {
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5f) out[0] = s;
}
__global__ void vform(float* out, int iters, const float* ab) {
  float a[8], b[8], x[8];
  for (int j = 0; j < 8; ++j) { a[j] = ab[(threadIdx.x + j) & 63]; b[j] = ab[64 + ((threadIdx.x * 3 + j) & 63)]; x[j] = threadIdx.x * 1e-3f + j; }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fmaf(a[j], b[(j + 1) & 7], x[j]);
  float s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  float *o, *ab; cudaMalloc(&o, 4); cudaMalloc(&ab, 512);
  cudaMemset(ab, 0, 512);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, it = 16384;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  uform<<<blocks, threads>>>(o, 64, 0.999f, 0.001f);
  cudaEventRecord(e0); uform<<<blocks, threads>>>(o, it, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("uniform-operand FFMA: %.1f TFLOP/s\n", 16.0 * it * blocks * threads / (ms * 1e9));
  vform<<<blocks, threads>>>(o, 64, ab);
  cudaEventRecord(e0); vform<<<blocks, threads>>>(o, it, ab); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); printf("vector-register FFMA: %.1f TFLOP/s\n", 16.0 * it * blocks * threads / (ms * 1e9));
}
