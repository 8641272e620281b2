// Throughput probe: legacy warp-level mma.sync (HMMA) tf32 m16n8k8 and bf16
// m16n8k16 on sm_100a, vs FFMA.  Decides whether the hidden-32 object MLPs
// should move off FFMA (north star: "warp-level mma ... only if it pays off").
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tf32_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void bf16_loop(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 64 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 4; w <= 16; w *= 2) {
    int it = 4096;
    tf32_loop<<<148 * 2, w * 32>>>(d, 16);
    cudaEventRecord(e0); tf32_loop<<<148 * 2, w * 32>>>(d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 8 * 8.0 * it * (148 * 2) * w;
    printf("tf32 m16n8k8  warps/CTA %2d: %.1f TFLOP/s\n", w, fl / ms / 1e9);
    cudaEventRecord(e0); bf16_loop<<<148 * 2, w * 32>>>(d, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 8.0 * it * (148 * 2) * w;
    printf("bf16 m16n8k16 warps/CTA %2d: %.1f TFLOP/s\n", w, fl / ms / 1e9);
  }
  return 0;
}
