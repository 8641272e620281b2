// Shared device/host helpers for the vMAP B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/vmap_b200.h"

namespace vm {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int cuda_check(cudaError_t e, const char* what);

#define VM_CUDA(call)                                          \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return ::vm::cuda_check(_e, #call); \
  } while (0)

#define VM_REQUIRE(cond, msg)        \
  do {                               \
    if (!(cond)) {                   \
      ::vm::set_error(msg);          \
      return VM_ERR_SHAPE;           \
    }                                \
  } while (0)

// ---------------------------------------------------------------- layout
inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

inline int hidden_pad_of(int hidden) {
  if (hidden <= 32) return 32;
  if (hidden <= 64) return 64;
  if (hidden <= 128) return 128;
  if (hidden <= (1 << 16)) return round_up(hidden, 32);  // layered path only (vm_layered.cu)
  return -1;
}

// models.py:50-55 layer_dims, padded for the kernels: layer 0 fan-in to a
// multiple of 4 floats (16 B rows), hidden widths to 32/64/128 (wider: a
// multiple of 32, trained by the layered path).
inline int compute_layout(const VmArch& a, VmLayout& L) {
  if (a.n_layers < 2 || a.n_layers > VM_MAX_LAYERS || a.hidden < 1 || a.input_dim < 1) return VM_ERR_SHAPE;
  const int hp = hidden_pad_of(a.hidden);
  if (hp < 0) return VM_ERR_UNSUPPORTED;
  L = VmLayout{};
  L.n_layers = a.n_layers;
  L.hidden_pad = hp;
  int64_t off = 0, n = 0;
  for (int l = 0; l < a.n_layers; ++l) {
    const bool last = l == a.n_layers - 1;
    L.fo[l] = last ? 4 : a.hidden;
    L.fi[l] = l == 0 ? a.input_dim : a.hidden;
    L.fo_pad[l] = last ? 4 : hp;
    L.fi_pad[l] = l == 0 ? round_up(a.input_dim, 4) : hp;
    L.w_off[l] = off;
    off += int64_t(L.fo_pad[l]) * L.fi_pad[l];
    L.b_off[l] = off;
    off += L.fo_pad[l];
    n += int64_t(L.fo[l]) * L.fi[l] + L.fo[l];
  }
  L.block = off;
  L.n_params = n;
  return VM_OK;
}

// ---------------------------------------------------------------- forward-only evaluation (vm_mlp.cu)
// bytes of the tensor-core forward's weight image for `a` (0: FFMA forward)
size_t fwd_image_bytes(const VmArch& a);
// vm_forward with the caller's scratch for that image (nullptr: stream-ordered temporary)
int forward_ws(const VmStack* st, const float* encoded, int64_t n_samples, float* occ, float* col, float* img,
               cudaStream_t s);

// ---------------------------------------------------------------- layered path (vm_layered.cu)
// Architectures / batches without a fused kernel: one kernel sequence per layer.
bool layered_forced();
size_t layered_train_bytes(const VmStack* stacks, const VmBatch* batches, int n, int first);
int train_layered(const VmStack* stacks, const VmBatch* batches, int n, int first, VmLossWeights w, float* losses,
                  int32_t* status, void* workspace, size_t workspace_bytes, cudaStream_t s);
int layered_fwd_bwd(const VmStack& st, const float* enc, int64_t n_samples, const float* gocc, const float* gcol,
                    float* occ, float* col, float* grads, bool backward, cudaStream_t s);

// ---------------------------------------------------------------- schedule tracing (VM_TRACE=1)
unsigned long long* trace_ptr();  // host: VM_TRACE buffer or null (vm_mlp.cu)

__device__ __forceinline__ unsigned long long vm_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned vm_smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
// one schedule record (kind, SM, start ns, end ns); called by one thread
__device__ __forceinline__ void vm_trace_rec(unsigned long long* tr, int kind, unsigned long long t0) {
  if (!tr) return;
  const unsigned slot = atomicAdd(reinterpret_cast<unsigned*>(tr), 1u);
  if (slot >= (1u << 16)) return;
  unsigned long long* r = tr + 1 + 4ull * slot;
  r[0] = kind;
  r[1] = vm_smid();
  r[2] = t0;
  r[3] = vm_gtime();
}

// ---------------------------------------------------------------- device
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// numpy pairwise summation for float32 (loops_utils.h.src pairwise_sum),
// the order `arr.sum(axis=-1)` uses on a contiguous axis.  `get(i)` yields
// element i.  n < 8: sequential from -0.0; n <= 128: 8 strided accumulators
// combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail; larger n
// recurses on halves rounded down to a multiple of 8.
template <typename F>
__device__ float pairwise_sum_leaf(const F& get, int64_t i0, int64_t n) {
  if (n < 8) {
    float res = -0.0f;
    for (int64_t i = 0; i < n; ++i) res = __fadd_rn(res, get(i0 + i));
    return res;
  }
  float r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = get(i0 + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], get(i0 + i + j));
  }
  float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                        __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __fadd_rn(res, get(i0 + i));
  return res;
}

// pairwise_sum_leaf for a compile-time n <= 128: every index is a constant,
// so register arrays behind `get` stay in registers (same order, same bits).
template <int N, typename F>
__device__ __forceinline__ float pairwise_sum_fixed(const F& get) {
  static_assert(N <= 128, "one pairwise leaf");
  if constexpr (N < 8) {
    float res = -0.0f;
#pragma unroll
    for (int i = 0; i < N; ++i) res = __fadd_rn(res, get(i));
    return res;
  } else {
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = get(j);
#pragma unroll
    for (int i = 8; i < N - (N % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], get(i + j));
    }
    float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                          __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
#pragma unroll
    for (int i = N - (N % 8); i < N; ++i) res = __fadd_rn(res, get(i));
    return res;
  }
}

// Recursive split for n > 128 (depth <= log2(n/128)).
template <typename F>
__device__ float pairwise_sum_rec(const F& get, int64_t i0, int64_t n) {
  if (n <= 128) return pairwise_sum_leaf(get, i0, n);
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __fadd_rn(pairwise_sum_rec(get, i0, n2), pairwise_sum_rec(get, i0 + n2, n - n2));
}

template <typename F>
__device__ float pairwise_sum(const F& get, int64_t n) {
  return pairwise_sum_rec(get, 0, n);
}

// The leaves (n <= 128 blocks) of pairwise_sum_rec's recursion for n
// elements, in depth-first order; returns their count (only the first
// max_leaves are stored).  Lets a CTA sum the leaves in parallel and combine
// them with pairwise_combine in exactly the recursive order.
__host__ __device__ inline int pairwise_leaves(int64_t n, int64_t* start, int* len, int max_leaves) {
  int64_t si[24], sn[24];  // depth <= log2(n / 128) + 1 <= 24 for any int32 row count
  int sp = 0, cnt = 0;
  si[sp] = 0;
  sn[sp++] = n;
  while (sp > 0) {
    --sp;
    const int64_t i0 = si[sp], m = sn[sp];
    if (m <= 128) {
      if (cnt < max_leaves) {
        start[cnt] = i0;
        len[cnt] = int(m);
      }
      ++cnt;
    } else {
      int64_t m2 = m / 2;
      m2 -= m2 % 8;
      si[sp] = i0 + m2;  // right half, popped after the left one
      sn[sp++] = m - m2;
      si[sp] = i0;
      sn[sp++] = m2;
    }
  }
  return cnt;
}

// Adds per-leaf sums (depth-first order) the way pairwise_sum_rec adds halves.
__device__ inline float pairwise_combine(int64_t n, const float* leaf, int& next) {
  if (n <= 128) return leaf[next++];
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const float a = pairwise_combine(n2, leaf, next);
  const float b = pairwise_combine(n - n2, leaf, next);
  return __fadd_rn(a, b);
}

// np.sign for float32: +1, -1, 0 for +-0, NaN for NaN.
__device__ __forceinline__ float np_sign(float x) {
  return x > 0.f ? 1.f : (x < 0.f ? -1.f : (x == 0.f ? 0.f : x));
}
// np.maximum (propagates NaN from either side).
__device__ __forceinline__ float np_maximum(float a, float b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}

}  // namespace vm
