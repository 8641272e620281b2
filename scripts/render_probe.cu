// Times the per-ray render chain (vm_render.cuh) for one ray in isolation.
#include <cstdio>
#include "vm_render.cuh"
using namespace vm;
__global__ void k(const float* in, float* out, long long* cyc, int S, int mode) {
  __shared__ float sO[4][32], sT[32], sTr[32];
  for (int i = threadIdx.x; i < 32; i += blockDim.x) {
    for (int c = 0; c < 4; ++c) sO[c][i] = in[c * 32 + i];
    sT[i] = in[128 + i];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  RayTargets tg{1.5f, {0.2f, 0.4f, 0.6f}, true, true, true};
  long long t0 = clock64();
  RayLossGrad lg;
  if (mode == 0) {
    float o[10], cl[3][10], tv[10];
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      o[i] = sO[0][i];
      tv[i] = sT[i];
#pragma unroll
      for (int c = 0; c < 3; ++c) cl[c][i] = sO[1 + c][i];
    }
    lg = render_ray_fixed<10>(o, cl, tv, tg, 5.f, 10.f);
#pragma unroll
    for (int i = 0; i < 10; ++i) { sO[0][i] = o[i]; for (int c = 0; c < 3; ++c) sO[1 + c][i] = cl[c][i]; }
  } else {
    auto occ = [&](int i) { return sO[0][i]; };
    auto col = [&](int i, int c) { return sO[1 + c][i]; };
    auto tt = [&](int i) { return sT[i]; };
    render_ray_forward(S, occ, col, tt, [&](int i, float v) { sTr[i] = v; });
    const RayFwd f = render_ray_sums(S, occ, col, tt, [&](int i) { return sTr[i]; });
    lg = ray_loss_grad(f, tg, 5.f, 10.f);
    render_ray_backward(S, occ, col, tt, [&](int i) { return sTr[i]; }, lg.dO, lg.dD, lg.dC,
                        [&](int i, float d_occ, const float* d_col) {
                          const float o = sO[0][i];
                          sO[0][i] = __fmul_rn(__fmul_rn(d_occ, o), __fsub_rn(1.0f, o));
                          for (int c = 0; c < 3; ++c) {
                            const float cv = sO[1 + c][i];
                            sO[1 + c][i] = __fmul_rn(__fmul_rn(d_col[c], cv), __fsub_rn(1.0f, cv));
                          }
                        });
  }
  __syncwarp(1);
  long long t1 = clock64();
  cyc[mode] = t1 - t0;
  for (int i = 0; i < S; ++i) out[mode * 64 + i] = sO[0][i] + sO[1][i];
  out[mode * 64 + 40] = lg.l_depth;
}
int main() {
  float h[160];
  for (int i = 0; i < 160; ++i) h[i] = 0.1f + 0.8f * ((i * 37) % 101) / 101.f;
  for (int i = 0; i < 32; ++i) h[128 + i] = 0.2f * i;
  float *din, *dout; long long* dc;
  cudaMalloc(&din, 640); cudaMalloc(&dout, 4096); cudaMalloc(&dc, 16);
  cudaMemcpy(din, h, 640, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep)
    for (int mode = 0; mode < 2; ++mode) k<<<1, 32>>>(din, dout, dc, 10, mode);
  cudaDeviceSynchronize();
  long long c[2]; float o[128];
  cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
  cudaMemcpy(o, dout, 512, cudaMemcpyDeviceToHost);
  printf("regs render: %lld cycles, smem render: %lld cycles, same=%d\n", c[0], c[1],
         (int)(memcmp(o, o + 64, 11 * 4) == 0));
}
