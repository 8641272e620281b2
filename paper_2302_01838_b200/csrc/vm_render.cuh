// Per-ray occupancy rendering, L1 losses and their gradients.
//
// Restates render.py:230-333 with numpy's float32 operation order so that,
// given bit-identical per-sample occupancy/colour, the results are
// bit-identical too (every op is an explicit _rn intrinsic: no FMA
// contraction).  Used by the standalone parity kernels (vm_render.cu) and by
// the fused training kernel (vm_mlp.cu).
#pragma once

#include "vm_common.cuh"

namespace vm {

// Accessor-based so callers can keep samples in smem or global memory.
// OCC(i), COL(i,c), TT(i) read sample i of the ray; TRANS is scratch with
// room for S floats (written: T_i).
struct RayFwd {
  float opacity, depth, colour[3];
};

template <typename Occ, typename Col, typename Tt, typename Tw>
__device__ __forceinline__ RayFwd render_ray_forward(int S, const Occ& occ, const Col& col, const Tt& tt,
                                                     const Tw& trans_store) {
  // trans[0] = 1, trans[i] = cumprod(1 - o)[i-1]   (render.py:238-241)
  float T = 1.0f;
  for (int i = 0; i < S; ++i) {
    trans_store(i, T);
    T = (i == 0) ? __fsub_rn(1.0f, occ(0)) : __fmul_rn(T, __fsub_rn(1.0f, occ(i)));
  }
  return RayFwd{};
}

// Full forward given stored transmittance: weights = o*T; O = pw(w);
// D = pw(w*t); C = sequential over samples of w*c (render.py:242-245).
template <typename Occ, typename Col, typename Tt, typename Tr>
__device__ __forceinline__ RayFwd render_ray_sums(int S, const Occ& occ, const Col& col, const Tt& tt,
                                                  const Tr& trans) {
  RayFwd r;
  auto w = [&](int64_t i) { return __fmul_rn(occ(int(i)), trans(int(i))); };
  r.opacity = pairwise_sum_leaf(w, 0, S);
  r.depth = pairwise_sum_leaf([&](int64_t i) { return __fmul_rn(w(i), tt(int(i))); }, 0, S);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float acc = __fmul_rn(w(0), col(0, c));
    for (int i = 1; i < S; ++i) acc = __fadd_rn(acc, __fmul_rn(w(i), col(i, c)));
    r.colour[c] = acc;
  }
  return r;
}

struct RayTargets {
  float depth, colour[3];
  bool mask, valid, ok;
};

struct RayLossGrad {
  float l_depth, l_colour, l_occ;  // per-ray terms (before the sum over rays)
  float dO, dD, dC[3];
};

// compute_losses / loss_output_grads per ray (render.py:284-333).
__device__ __forceinline__ RayLossGrad ray_loss_grad(const RayFwd& f, const RayTargets& tg, float w_colour,
                                                     float w_occ) {
  const bool m_ok = tg.mask && tg.ok;
  const float m_ind = tg.mask ? 1.0f : 0.0f;
  const float wd = (m_ok && tg.valid) ? 1.0f : 0.0f;
  const float wc = m_ok ? 1.0f : 0.0f;
  const float wo = tg.ok ? 1.0f : 0.0f;
  RayLossGrad o;
  o.l_depth = __fmul_rn(wd, fabsf(__fsub_rn(f.depth, tg.depth)));
  float cs = fabsf(__fsub_rn(f.colour[0], tg.colour[0]));
  cs = __fadd_rn(cs, fabsf(__fsub_rn(f.colour[1], tg.colour[1])));
  cs = __fadd_rn(cs, fabsf(__fsub_rn(f.colour[2], tg.colour[2])));
  o.l_colour = __fmul_rn(wc, cs);
  o.l_occ = __fmul_rn(wo, fabsf(__fsub_rn(f.opacity, m_ind)));
  o.dD = __fmul_rn(wd, np_sign(__fsub_rn(f.depth, tg.depth)));
  const float wcc = __fmul_rn(w_colour, wc);
#pragma unroll
  for (int c = 0; c < 3; ++c) o.dC[c] = __fmul_rn(wcc, np_sign(__fsub_rn(f.colour[c], tg.colour[c])));
  o.dO = __fmul_rn(__fmul_rn(w_occ, wo), np_sign(__fsub_rn(f.opacity, m_ind)));
  return o;
}

// render_backward per ray (render.py:249-281).  Emits (i, d_occ_i, d_col_i)
// through `emit`, from the last sample to the first.
template <typename Occ, typename Col, typename Tt, typename Tr, typename Emit>
__device__ __forceinline__ void render_ray_backward(int S, const Occ& occ, const Col& col, const Tt& tt,
                                                    const Tr& trans, float dO, float dD, const float dC[3],
                                                    const Emit& emit) {
  float rev = 0.0f;
  for (int i = S - 1; i >= 0; --i) {
    const float o = occ(i);
    const float T = trans(i);
    const float w = __fmul_rn(o, T);
    float cs = __fmul_rn(dC[0], col(i, 0));
    cs = __fadd_rn(cs, __fmul_rn(dC[1], col(i, 1)));
    cs = __fadd_rn(cs, __fmul_rn(dC[2], col(i, 2)));
    const float g = __fadd_rn(__fadd_rn(dO, __fmul_rn(dD, tt(i))), cs);
    const float gw = __fmul_rn(g, w);
    rev = (i == S - 1) ? gw : __fadd_rn(rev, gw);
    const float suffix = __fsub_rn(rev, gw);
    const float denom = np_maximum(__fsub_rn(1.0f, o), 1e-7f);
    const float d_occ = __fsub_rn(__fmul_rn(g, T), __fdiv_rn(suffix, denom));
    float d_col[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) d_col[c] = __fmul_rn(w, dC[c]);
    emit(i, d_occ, d_col);
  }
}

// Register-resident variant of the whole per-ray chain for a compile-time
// sample count NS (render_ray_forward + render_ray_sums + ray_loss_grad +
// render_ray_backward with identical operation order).  With NS known every
// loop is straight-line code, so the independent per-sample work of the sums
// and of the backward pass overlaps instead of running as one predicated
// chain.  On return o[] / c[][] hold the sigmoid-input gradients dz.
template <int NS>
__device__ __forceinline__ RayLossGrad render_ray_fixed(float (&o)[NS], float (&c)[3][NS], const float (&t)[NS],
                                                        const RayTargets& tg, float w_colour, float w_occ) {
  float T[NS], w[NS];
  float Tc = 1.0f;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    T[i] = Tc;
    Tc = (i == 0) ? __fsub_rn(1.0f, o[0]) : __fmul_rn(Tc, __fsub_rn(1.0f, o[i]));
    w[i] = __fmul_rn(o[i], T[i]);
  }
  // pairwise_sum_leaf (loops_utils.h.src order) for n = NS <= 128
  auto psum = [&](auto&& get) -> float {
    if constexpr (NS < 8) {
      float res = -0.0f;
#pragma unroll
      for (int i = 0; i < NS; ++i) res = __fadd_rn(res, get(i));
      return res;
    } else {
      float r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = get(j);
      constexpr int full = NS - (NS % 8);
#pragma unroll
      for (int i = 8; i < full; i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], get(i + j));
      float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                            __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
#pragma unroll
      for (int i = full; i < NS; ++i) res = __fadd_rn(res, get(i));
      return res;
    }
  };
  RayFwd f;
  f.opacity = psum([&](int i) { return w[i]; });
  f.depth = psum([&](int i) { return __fmul_rn(w[i], t[i]); });
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    float acc = __fmul_rn(w[0], c[ch][0]);
#pragma unroll
    for (int i = 1; i < NS; ++i) acc = __fadd_rn(acc, __fmul_rn(w[i], c[ch][i]));
    f.colour[ch] = acc;
  }
  const RayLossGrad lg = ray_loss_grad(f, tg, w_colour, w_occ);
  float g[NS], gw[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    float cs = __fmul_rn(lg.dC[0], c[0][i]);
    cs = __fadd_rn(cs, __fmul_rn(lg.dC[1], c[1][i]));
    cs = __fadd_rn(cs, __fmul_rn(lg.dC[2], c[2][i]));
    g[i] = __fadd_rn(__fadd_rn(lg.dO, __fmul_rn(lg.dD, t[i])), cs);
    gw[i] = __fmul_rn(g[i], w[i]);
  }
  float rev = 0.0f;
#pragma unroll
  for (int i = NS - 1; i >= 0; --i) {
    rev = (i == NS - 1) ? gw[i] : __fadd_rn(rev, gw[i]);
    const float suffix = __fsub_rn(rev, gw[i]);
    const float denom = np_maximum(__fsub_rn(1.0f, o[i]), 1e-7f);
    const float d_occ = __fsub_rn(__fmul_rn(g[i], T[i]), __fdiv_rn(suffix, denom));
    const float oi = o[i];
    o[i] = __fmul_rn(__fmul_rn(d_occ, oi), __fsub_rn(1.0f, oi));
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float cv = c[ch][i];
      c[ch][i] = __fmul_rn(__fmul_rn(__fmul_rn(w[i], lg.dC[ch]), cv), __fsub_rn(1.0f, cv));
    }
  }
  return lg;
}

// Register-light render chain for one ray (render_ray_fixed's operation
// order): occupancy/colour/t are read from smem (feature-major rows of LD
// floats: occupancy, r, g, b), the 2*NS transmittance and
// weight values stay in registers; writes dz (sigmoid'd gradients) in place.
template <int NS, int LD>
__device__ __forceinline__ RayLossGrad render_ray_smem(float* __restrict__ O, const float* __restrict__ tS, int sb,
                                                       const RayTargets& tg, float w_colour, float w_occ) {
  float Tr[NS], w[NS];
  float Tc = 1.0f;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const float o = O[sb + i];
    Tr[i] = Tc;
    Tc = (i == 0) ? __fsub_rn(1.0f, o) : __fmul_rn(Tc, __fsub_rn(1.0f, o));
    w[i] = __fmul_rn(o, Tr[i]);
  }
  RayFwd f;
  f.opacity = pairwise_sum_fixed<NS>([&](int i) { return w[i]; });
  f.depth = pairwise_sum_fixed<NS>([&](int i) { return __fmul_rn(w[i], tS[sb + i]); });
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const float* c = O + (1 + ch) * LD + sb;
    float acc = __fmul_rn(w[0], c[0]);
#pragma unroll
    for (int i = 1; i < NS; ++i) acc = __fadd_rn(acc, __fmul_rn(w[i], c[i]));
    f.colour[ch] = acc;
  }
  const RayLossGrad lg = ray_loss_grad(f, tg, w_colour, w_occ);
  float rev = 0.0f;
#pragma unroll
  for (int i = NS - 1; i >= 0; --i) {
    float cl[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) cl[ch] = O[(1 + ch) * LD + sb + i];
    float cs = __fmul_rn(lg.dC[0], cl[0]);
    cs = __fadd_rn(cs, __fmul_rn(lg.dC[1], cl[1]));
    cs = __fadd_rn(cs, __fmul_rn(lg.dC[2], cl[2]));
    const float g = __fadd_rn(__fadd_rn(lg.dO, __fmul_rn(lg.dD, tS[sb + i])), cs);
    const float gw = __fmul_rn(g, w[i]);
    rev = (i == NS - 1) ? gw : __fadd_rn(rev, gw);
    const float suffix = __fsub_rn(rev, gw);
    const float oi = O[sb + i];
    const float denom = np_maximum(__fsub_rn(1.0f, oi), 1e-7f);
    const float d_occ = __fsub_rn(__fmul_rn(g, Tr[i]), __fdiv_rn(suffix, denom));
    O[sb + i] = __fmul_rn(__fmul_rn(d_occ, oi), __fsub_rn(1.0f, oi));
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
      O[(1 + ch) * LD + sb + i] = __fmul_rn(__fmul_rn(__fmul_rn(w[i], lg.dC[ch]), cl[ch]), __fsub_rn(1.0f, cl[ch]));
  }
  return lg;
}

}  // namespace vm
