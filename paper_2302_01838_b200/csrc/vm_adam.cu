// Standalone Adam entry point (models.py:401-467 adam_step).
#include "vm_adam.cuh"

namespace vm {
namespace {

// Pass 1: first active model with a non-finite gradient (models.py:423-428).
__global__ void adam_check_kernel(int K, int64_t block, const float* __restrict__ G,
                                  const uint8_t* __restrict__ frozen, const uint8_t* __restrict__ mask,
                                  int32_t* __restrict__ status) {
  const int k = blockIdx.y;
  if (frozen[k] || (mask && !mask[k])) return;
  const float* g = G + int64_t(k) * block;
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < block; i += int64_t(gridDim.x) * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMin(status, k);
}

// Pass 2: update every active model unless pass 1 found a bad one.
__global__ void adam_apply_kernel(int K, int64_t block, float* __restrict__ P, float* __restrict__ M,
                                  float* __restrict__ V, const float* __restrict__ G,
                                  const int64_t* __restrict__ step, const uint8_t* __restrict__ frozen,
                                  const uint8_t* __restrict__ mask, const int32_t* __restrict__ status,
                                  AdamConsts a) {
  if (*status != INT32_MAX) return;
  const int k = blockIdx.y;
  if (frozen[k] || (mask && !mask[k])) return;
  float c1, c2;
  adam_corr(a, step[k], c1, c2);
  const int64_t base = int64_t(k) * block;
  for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * 4; i < block;
       i += int64_t(gridDim.x) * blockDim.x * 4)
    adam_vec4(P + base, M + base, V + base, G + base, i, c1, c2, a);
}

__global__ void adam_finish_kernel(int K, int64_t* __restrict__ step, const uint8_t* __restrict__ frozen,
                                   const uint8_t* __restrict__ mask, int32_t* __restrict__ status) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = *status == INT32_MAX;
  if (k < K && ok && !frozen[k] && !(mask && !mask[k])) step[k] += 1;
}

__global__ void set_i32(int32_t* p, int32_t v) { *p = v; }
__global__ void status_to_public(int32_t* p) {
  if (*p == INT32_MAX) *p = -1;
}

}  // namespace
}  // namespace vm

using namespace vm;

extern "C" int vm_adam(const VmStack* st, const float* grads, const uint8_t* update_mask, int32_t* status,
                       void* stream) {
  VM_REQUIRE(st && grads && status, "vm_adam: null argument");
  VmLayout L;
  int rc = compute_layout(st->arch, L);
  if (rc) {
    set_error("vm_adam: unsupported arch");
    return rc;
  }
  cudaStream_t s = cudaStream_t(stream);
  set_i32<<<1, 1, 0, s>>>(status, INT32_MAX);
  const int K = st->count;
  if (K > 0) {
    const int bx = int((L.block / 4 + 255) / 256);
    dim3 grid(bx < 1 ? 1 : bx, K);
    adam_check_kernel<<<grid, 256, 0, s>>>(K, L.block, grads, st->frozen, update_mask, status);
    adam_apply_kernel<<<grid, 256, 0, s>>>(K, L.block, st->params, st->m, st->v, grads, st->step, st->frozen,
                                           update_mask, status, adam_consts(*st));
    adam_finish_kernel<<<(K + 255) / 256, 256, 0, s>>>(K, st->step, st->frozen, update_mask, status);
  }
  status_to_public<<<1, 1, 0, s>>>(status);
  VM_CUDA(cudaGetLastError());
  return VM_OK;
}
