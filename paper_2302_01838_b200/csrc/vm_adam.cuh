// Batched Adam over the stacked model arena (models.py:401-467).
//
// Bit-exact with the reference given identical gradients: f32 op sequence of
// models.py:444-461 with no FMA contraction, bias corrections precomputed on
// the host in f64 exactly like models.py:434-436, IEEE sqrt/div.
#pragma once

#include "vm_common.cuh"

namespace vm {

struct AdamConsts {
  float b1, omb1, b2, omb2, eps, lr;
  const float* corr1;
  const float* corr2;
  int corr_len;
  double beta1, beta2;
};

// f32(1 - beta^t) for t = step + 1 (models.py:434-436): the host's f64 table
// for t <= corr_len, else the same f64 expression on the device.
__device__ __forceinline__ float2 bias_corrections(const float* corr1, const float* corr2, int corr_len, double b1,
                                                   double b2, int64_t step) {
  const int64_t t = step + 1;
  if (t <= corr_len) return make_float2(corr1[t - 1], corr2[t - 1]);
  return make_float2(float(1.0 - pow(b1, double(t))), float(1.0 - pow(b2, double(t))));
}

__device__ __forceinline__ void adam_elem(float& p, float& m, float& v, float g, float c1, float c2,
                                          const AdamConsts& a) {
  m = __fmul_rn(m, a.b1);
  m = __fadd_rn(m, __fmul_rn(a.omb1, g));
  float gg = __fmul_rn(g, g);
  gg = __fmul_rn(gg, a.omb2);
  v = __fmul_rn(v, a.b2);
  v = __fadd_rn(v, gg);
  const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(v, c2)), a.eps);
  float upd = __fdiv_rn(m, c1);
  upd = __fdiv_rn(upd, den);
  upd = __fmul_rn(upd, a.lr);
  p = __fsub_rn(p, upd);
}

__device__ __forceinline__ void adam_corr(const AdamConsts& a, int64_t step, float& c1, float& c2) {
  const float2 c = bias_corrections(a.corr1, a.corr2, a.corr_len, a.beta1, a.beta2, step);
  c1 = c.x;
  c2 = c.y;
}

// One float4 of model `k`'s block.  Caller guarantees the model is active.
__device__ __forceinline__ void adam_vec4(float* __restrict__ P, float* __restrict__ M, float* __restrict__ V,
                                          const float* __restrict__ G, int64_t idx, float c1, float c2,
                                          const AdamConsts& a) {
  float4 p = ld4(P + idx), m = ld4(M + idx), v = ld4(V + idx);
  const float4 g = ld4(G + idx);
  adam_elem(p.x, m.x, v.x, g.x, c1, c2, a);
  adam_elem(p.y, m.y, v.y, g.y, c1, c2, a);
  adam_elem(p.z, m.z, v.z, g.z, c1, c2, a);
  adam_elem(p.w, m.w, v.w, g.w, c1, c2, a);
  st4(P + idx, p);
  st4(M + idx, m);
  st4(V + idx, v);
}

inline AdamConsts adam_consts(const VmStack& s) {
  return AdamConsts{s.beta1f, s.omb1, s.beta2f, s.omb2, s.eps, s.lr, s.corr1, s.corr2, s.corr_len, s.beta1, s.beta2};
}

}  // namespace vm
