// Fingerprint the operand address pattern of an MN-major tf32 descriptor:
// A smem holds its own float index; B (K-major, known-good) is one-hot so
// D[m][k] = the smem index the tensor core read for logical A(m, k).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "vm_tc.cuh"
using namespace vm::tc;
__global__ void fp(float* D, uint32_t lbo, uint32_t sbo, int a_mn, int pass) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* sA = reinterpret_cast<float*>(sm);
  float* sB = sA + 48 * 1024;
  for (int i = tid; i < 48 * 1024; i += 128) sA[i] = pass ? float(i >> 10) : float(i & 1023);
  for (int i = tid; i < 16 * 8; i += 128) { int n = i / 8, k = i % 8; sB[ilv_off(n, k, 8) / 4] = (n == k) ? 1.f : 0.f; }
  if (warp == 0) tmem_alloc(&tbase, 32);
  if (tid == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  fence_async_smem(); fence_before_sync(); __syncthreads(); fence_after_sync();
  if (tid == 0) {
    mma_tf32(tbase, sdesc(smem_u32(sA), lbo, sbo), sdesc(smem_u32(sB), 128, 256), idesc_tf32(128, 16, a_mn, false), 0);
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  fence_after_sync();
  float v[16];
  tmem_ld16(tbase + (uint32_t(32 * warp) << 16), v);
  for (int j = 0; j < 8; ++j) D[(32 * warp + lane) * 8 + j] = v[j];
  fence_before_sync(); __syncthreads();
  if (warp == 0) tmem_free(tbase, 32);
}
int main() {
  float* d; cudaMalloc(&d, 128 * 8 * 4);
  float h[128 * 8], h2[128 * 8];
  const int SM = 48 * 1024 * 4 + 1024;
  cudaFuncSetAttribute(fp, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
  struct { uint32_t lbo, sbo; int mn; } cs[] = {{128, 256, 0}, {4096, 128, 1}, {128, 4096, 1}, {256, 512, 1}, {512, 256, 1}};
  for (auto c : cs) {
    fp<<<1, 128, SM>>>(d, c.lbo, c.sbo, c.mn, 1);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h2, d, 4096, cudaMemcpyDeviceToHost);
    fp<<<1, 128, SM>>>(d, c.lbo, c.sbo, c.mn, 0);
    e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 4096, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 1024; ++i) h[i] += 1024 * h2[i];
    printf("a_mn=%d lbo=%u sbo=%u err=%s\n", c.mn, c.lbo, c.sbo, cudaGetErrorString(e));
    for (int m : {0, 1, 2, 3, 4, 5, 7, 8, 15, 16, 31, 32, 64, 127}) {
      printf("  m=%3d:", m);
      for (int k = 0; k < 8; ++k) printf(" %6.0f", h[m * 8 + k]);
      printf("\n");
    }
  }
}
