// Probe for the tcgen05 kind::tf32 path on B200: descriptor/major-ness
// correctness against an fp64 host GEMM (plain TF32 and 3xTF32), the M=64
// TMEM row placement, and single-CTA MMA throughput; plus the legacy
// mma.sync m16n8k8 TF32 rate for comparison.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2302_01838_b200/csrc \
//        scripts/tc_probe.cu -o /tmp/tc_probe && /tmp/tc_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "vm_tc.cuh"

using namespace vm::tc;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

// D[M][N] = A[M][K] * B[N][K]^T.  a_mn / b_mn select MN-major storage.
__global__ void gemm_probe(const float* A, const float* B, float* D, int M, int N, int K, int a_mn, int b_mn,
                           int split, int dump_lanes, int swap) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Mt = 128;  // storage rows for A are padded to 128 so M=64 reads valid smem
  uint8_t* sAh = sm;
  uint8_t* sAl = sAh + Mt * K * 4;
  uint8_t* sBh = sAl + Mt * K * 4;
  uint8_t* sBl = sBh + N * K * 4;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tbase;
  for (int i = tid; i < Mt * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const float x = m < M ? A[m * K + k] : 0.f;
    float hi, lo;
    if (split) split3(x, hi, lo); else { hi = x; lo = 0.f; }
    const uint32_t off = a_mn == 3 ? uint32_t((m >> 5) * (K * 128) + (k >> 2) * 512 + (k & 3) * 128 + ((((m & 31) >> 3) ^ (k & 3)) << 5) + (m & 7) * 4)
                       : a_mn == 2 ? uint32_t(m * 128 + (((k >> 2) ^ (m & 7)) << 4) + (k & 3) * 4) : a_mn ? ilv_off(k, m, Mt) : ilv_off(m, k, K);
    *reinterpret_cast<float*>(sAh + off) = hi;
    *reinterpret_cast<float*>(sAl + off) = lo;
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    float hi, lo;
    if (split) split3(B[i], hi, lo); else { hi = B[i]; lo = 0.f; }
    const uint32_t off = b_mn == 3 ? uint32_t((n >> 5) * (K * 128) + (k >> 2) * 512 + (k & 3) * 128 + ((((n & 31) >> 3) ^ (k & 3)) << 5) + (n & 7) * 4)
                       : b_mn == 2 ? uint32_t(n * 128 + (((k >> 2) ^ (n & 7)) << 4) + (k & 3) * 4) : b_mn ? ilv_off(k, n, N) : ilv_off(n, k, K);
    *reinterpret_cast<float*>(sBh + off) = hi;
    *reinterpret_cast<float*>(sBl + off) = lo;
  }
  fence_async_smem();
  __syncthreads();
  if (tid == 0) {
    fence_after_sync();
    const uint32_t idesc = idesc_tf32(M, N, a_mn == 1 || a_mn == 3, b_mn == 1 || b_mn == 3);
    // K-major: LBO = 128 (k group), SBO = cols*32 (row group); step 8 k = 256 B
    // MN-major: LBO = cols*32 (8 K-rows), SBO = 128 (4 MN); step 8 k = cols*32
    uint32_t a_lbo = a_mn ? Mt * 32 : 128, a_sbo = a_mn ? 128 : K * 32, a_step = a_mn ? Mt * 32 : 256;
    uint32_t b_lbo = b_mn ? N * 32 : 128, b_sbo = b_mn ? 128 : K * 32, b_step = b_mn ? N * 32 : 256;
    if (swap && a_mn) { uint32_t t = a_lbo; a_lbo = a_sbo; a_sbo = t; }
    if (swap && b_mn) { uint32_t t = b_lbo; b_lbo = b_sbo; b_sbo = t; }
    uint32_t acc = 0;
    const uint64_t a_sw = a_mn == 2 ? (uint64_t(2) << 61) : a_mn == 3 ? (uint64_t(1) << 61) : 0;
    const uint64_t b_sw = b_mn == 2 ? (uint64_t(2) << 61) : b_mn == 3 ? (uint64_t(1) << 61) : 0;
    if (a_mn == 3) { a_lbo = K * 128; a_sbo = 512; a_step = 1024; }
    if (b_mn == 3) { b_lbo = K * 128; b_sbo = 512; b_step = 1024; }
    if (a_mn == 2) { a_lbo = 16; a_sbo = 1024; a_step = 32; }
    if (b_mn == 2) { b_lbo = 16; b_sbo = 1024; b_step = 32; }
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t ah = sdesc(smem_u32(sAh) + ks * a_step, a_lbo, a_sbo) | a_sw;
      const uint64_t al = sdesc(smem_u32(sAl) + ks * a_step, a_lbo, a_sbo) | a_sw;
      const uint64_t bh = sdesc(smem_u32(sBh) + ks * b_step, b_lbo, b_sbo) | b_sw;
      const uint64_t bl = sdesc(smem_u32(sBl) + ks * b_step, b_lbo, b_sbo) | b_sw;
      if (split) {
        mma_tf32(tm, al, bh, idesc, acc); acc = 1;
        mma_tf32(tm, ah, bl, idesc, 1);
      }
      mma_tf32(tm, ah, bh, idesc, acc);
      acc = 1;
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  fence_after_sync();
  const int rows = dump_lanes ? 128 : M;
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tm + (uint32_t(32 * warp) << 16) + c, v);
    const int r = 32 * warp + lane;
    if (r < rows)
      for (int j = 0; j < 16; ++j) D[r * N + c + j] = v[j];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free(tm, 512);
}

// Back-to-back MMAs from one thread; returns cycles per instruction.
__global__ void mma_rate(long long* out, int N, int iters, int sw) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 32 + N * 32; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i % 7);
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, N, false, false);
    uint64_t a = sdesc(smem_u32(sm), 128, 32 * 32);
    uint64_t b = sdesc(smem_u32(sm) + 128 * 32 * 4, 128, 32 * 32);
    uint64_t step = 16;
    if (sw) {
      a = sdesc(smem_u32(sm), 16, 1024) | (uint64_t(2) << 61);
      b = sdesc(smem_u32(sm) + 128 * 32 * 4, 16, 1024) | (uint64_t(2) << 61);
      step = 2;
    }
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) mma_tf32(tbase, a + (i & 3) * step, b + (i & 3) * step, idesc, i > 0);
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free(tbase, 512);
}

__global__ void mmasync_rate(float* out, int iters) {
  uint32_t a0 = __float_as_uint(1.0f + threadIdx.x), a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  uint32_t b0 = __float_as_uint(0.5f), b1 = b0;
  float c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static int g_swap = 0;
static bool run_case(int M, int N, int K, int a_mn, int b_mn, int split) {
  std::vector<float> A(M * K), B(N * K), D(128 * N, 0.f);
  srand(1234 + M + N + a_mn * 3 + b_mn * 5);
  for (auto& x : A) x = (rand() / float(RAND_MAX) - 0.5f) * 2.f;
  for (auto& x : B) x = (rand() / float(RAND_MAX) - 0.5f) * 2.f;
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, D.size() * 4));
  const int smem = (2 * 128 * K + 2 * N * K) * 4;
  CK(cudaFuncSetAttribute(gemm_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  gemm_probe<<<1, 128, smem>>>(dA, dB, dD, M, N, K, a_mn, b_mn, split, 0, g_swap);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double max_rel = 0.0, max_abs = 0.0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0.0, mag = 0.0;
      for (int k = 0; k < K; ++k) {
        ref += double(A[m * K + k]) * double(B[n * K + k]);
        mag += fabs(double(A[m * K + k]) * double(B[n * K + k]));
      }
      const double err = fabs(double(D[m * N + n]) - ref);
      max_abs = fmax(max_abs, err);
      max_rel = fmax(max_rel, err / (mag + 1e-30));
    }
  const double tol = split ? 1e-6 : 5e-3;
  const bool ok = max_rel < tol;
  printf("swap=%d case M=", g_swap); printf("%d N=%d K=%d a_mn=%d b_mn=%d split=%d: max_abs=%.3e max_rel(vs sum|ab|)=%.3e %s\n", M, N, K, a_mn,
         b_mn, split, max_abs, max_rel, ok ? "OK" : "FAIL");
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return ok;
}

static void m64_layout(int N) {
  // identity-ish A so D row m = B row (m % N)... use A[m][k] = (k == m % 8) * (m + 1)
  const int M = 64, K = 8;
  std::vector<float> A(M * K, 0.f), B(N * K, 0.f), D(128 * N, 0.f);
  for (int m = 0; m < M; ++m) A[m * K + 0] = float(m + 1);
  for (int n = 0; n < N; ++n) B[n * K + 0] = float(1000 * (n + 1));
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, D.size() * 4));
  const int smem = (2 * 128 * K + 2 * N * K) * 4;
  gemm_probe<<<1, 128, smem>>>(dA, dB, dD, M, N, K, 0, 0, 0, 1, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  printf("M=64 N=%d TMEM placement: lane -> (m, n of col0) [value/1000 = (m+1)(n+1)]\n", N);
  for (int l = 0; l < 128; ++l) {
    printf("  lane %3d:", l);
    for (int c = 0; c < N && c < 8; ++c) printf(" %8.0f", D[l * N + c]);
    printf("\n");
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
}

int main() {
  bool ok = true;
  for (int split = 0; split < 2; ++split)
    for (int amn = 0; amn < 3; amn += 2)
      for (int bmn = 0; bmn < 3; bmn += 2) ok &= run_case(128, 128, 32, amn, bmn, split);
  ok &= run_case(128, 16, 40, 0, 0, 1);
  ok &= run_case(128, 128, 32, 3, 3, 1);
  ok &= run_case(128, 128, 32, 3, 3, 0);
  ok &= run_case(128, 48, 32, 3, 3, 1);
  ok &= run_case(128, 16, 32, 3, 3, 1);
  ok &= run_case(128, 128, 32, 0, 3, 1);
  ok &= run_case(128, 16, 32, 2, 2, 1);
  ok &= run_case(128, 256, 16, 0, 0, 1);
  if (getenv("M64")) m64_layout(16);
  long long* dout;
  CK(cudaMalloc(&dout, 8));
  const int smem = (128 * 32 + 256 * 32) * 4;
  CK(cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int sw = 0; sw < 2; ++sw)
  for (int N : {16, 32, 48, 64, 128, 256}) {
    const int iters = 4096;
    mma_rate<<<1, 128, smem>>>(dout, N, iters, sw);
    CK(cudaDeviceSynchronize());
    long long cyc;
    CK(cudaMemcpy(&cyc, dout, 8, cudaMemcpyDeviceToHost));
    printf("sw=%d tcgen05 tf32 M=128 N=%3d K=8: %.1f cycles/MMA -> %.0f MAC/cycle/SM\n", sw, N, double(cyc) / iters,
           128.0 * N * 8 * iters / double(cyc));
  }
  // mma.sync rate: full chip, 148*4 CTAs of 256 threads
  float* dummy;
  CK(cudaMalloc(&dummy, 148 * 4 * 256 * 4));
  const int it = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mmasync_rate<<<148 * 4, 256>>>(dummy, 100);
  cudaEventRecord(e0);
  mmasync_rate<<<148 * 4, 256>>>(dummy, it);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 16 * 8 * 8 * 4.0 * it * (148 * 4 * 256 / 32);
  printf("mma.sync m16n8k8 tf32 full chip: %.1f TFLOP/s\n", flops / ms / 1e9);
  printf(ok ? "ALL OK\n" : "SOME FAILED\n");
  return ok ? 0 : 1;
}
