// KH32: the fused train step for the reference's object model (hidden 32,
// 4 layers, models.py:19-55; trainer.py:70-71) on the warp-level tensor path
// (mma.sync m16n8k8 TF32 -> HMMA), 3xTF32 so products keep ~FP32 accuracy.
//
// Why the tensor path: the per-object GEMMs are 32 wide, too small for
// tcgen05 tiles, but a B200 sustains 277 TFLOP/s of dense TF32 on mma.sync
// (scripts/hmma_probe.cu) against 71 TFLOP/s of FP32 FFMA; with three
// products per multiply (lo.hi + hi.lo + hi.hi) the tensor path still beats
// the FFMA roofline and issues ~10x fewer math instructions than KF32.
//
// Math: models.py:311-398 (forward/backward), render.py:230-333 (render,
// losses, grads), trainer.py:480-506 (the train_on_batch chain); the render
// and losses are the bit-exact register chain shared with KF32
// (render_ray_smem).
//
// Execution (B200, sm_100a):
//  * CTA = 8 warps, one CTA per SM (~212 KB smem).  Work item (one CTA) =
//    (model, chunk of VM_KF_CHUNK = 8 consecutive 32-sample blocks), the
//    same K-independent chunking as KF32, so vectorised == sequential.
//  * Warp w owns block w of the chunk (floor(32/S) whole rays).  Forward:
//    M = samples (2 m-tiles), N = outputs (4 n-tiles), K = inputs; each
//    layer's accumulator fragments become the next layer's A fragments in
//    registers (the next layer's K index is permuted to the accumulator's
//    column order: k-slot t <-> column 2t, k-slot t+4 <-> column 2t+1, and
//    the weight B fragments are read with the same permutation), so hidden
//    activations never round-trip through shared memory on the way forward.
//    ReLU masks are kept as bits (one register per layer).
//  * The activations a weight gradient needs are also written feature-major
//    ([feature][sample], stride 40 floats) to the warp's smem; the backward
//    dx GEMMs again chain in registers, and dW_l = dZ_l^T X_{l-1} runs as an
//    MMA with K = the block's 32 samples from smem (dZ staged feature-major in
//    the slot X_3 vacated).  Every weight-gradient tile is written into the
//    activation slot its layer no longer needs.
//  * End of item: the 8 warps' gradients are summed in warp order (fixed:
//    deterministic), then, as in KF32, the last chunk of a model (atomic
//    ticket) sums the chunk partials in order and finalises the model.
#include "vm_mlp.cuh"

namespace vm {
namespace kh32 {

constexpr int H = 32, NW = 8, NTHR = NW * 32;
constexpr int WS = 40;   // row stride (floats) of weights and feature-major activations: == 8 mod 32
constexpr int D0 = 40;   // layer-0 fan-in padded to 5 k-chunks of 8
constexpr int kOL = 40;  // render/output rows (occupancy, r, g, b), feature-major
// weight image (floats): W0..W2 [32][WS], W3 [8][WS] (rows 4..7 zero), then
// the transposed copies the dx GEMMs read: W1T, W2T [32][WS], W3T [32][8]
constexpr int oW0 = 0, oW1 = oW0 + H * WS, oW2 = oW1 + H * WS, oW3 = oW2 + H * WS, oW1T = oW3 + 8 * WS,
              oW2T = oW1T + H * WS, oW3T = oW2T + H * WS, oB0 = oW3T + H * 8, oB1 = oB0 + H, oB2 = oB1 + H,
              oB3 = oB2 + H, kWFloats = oB3 + 8;
// per-warp region (floats)
constexpr int rET = 0, rX1 = rET + D0 * WS, rX2 = rX1 + H * WS, rX3 = rX2 + H * WS, rO = rX3 + H * WS,
              rTs = rO + 4 * kOL, rTg = rTs + kSB, rDb = rTg + kSB, kWarpFloats = rDb + 3 * H + 4;
constexpr int kTgt = 8;
constexpr size_t kSmem = size_t(kWFloats + NW * kWarpFloats) * 4 + 64;
static_assert(kSmem + 1600 <= 227 * 1024, "KH32 exceeds the per-CTA shared-memory limit");
static_assert(kWarpFloats % 4 == 0 && kWFloats % 4 == 0, "16-B alignment of the regions");

// x = hi + lo with hi = x rounded to TF32 (ties away from zero in magnitude:
// two integer ops, where cvt.rna.tf32 lowers to a ~6-instruction sequence);
// lo = x - hi exactly, and the MMA reads lo's leading TF32 bits
__device__ __forceinline__ void split(float x, uint32_t& hi, uint32_t& lo) {
  hi = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
  lo = __float_as_uint(__fsub_rn(x, __uint_as_float(hi)));
}
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void split4(const float (&x)[4], uint32_t (&h)[4], uint32_t (&l)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) split(x[i], h[i], l[i]);
}
__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ float relu(float z) {
  float r;
  asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(z));  // np.maximum(z, 0): NaN propagates
  return r;
}

// One k-chunk of 3xTF32 MMAs over MT x NT accumulator tiles: the B fragments
// (from `bfrag(nt)`) are split first, then the three passes run over every
// tile in turn, so consecutive MMAs never share an accumulator (the tensor
// pipe is not stalled on the accumulator dependency).
template <int MT, int NT, typename BF>
__device__ __forceinline__ void mma_passes(float (&d)[MT][NT][4], const uint32_t (&ah)[MT][4],
                                           const uint32_t (&al)[MT][4], const BF& bfrag) {
  uint32_t bh[NT][2], bl[NT][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const float2 w = bfrag(nt);
    split(w.x, bh[nt][0], bl[nt][0]);
    split(w.y, bh[nt][1], bl[nt][1]);
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) mma(d[mt][nt], al[mt], bh[nt][0], bh[nt][1]);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) mma(d[mt][nt], ah[mt], bl[nt][0], bl[nt][1]);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) mma(d[mt][nt], ah[mt], bh[nt][0], bh[nt][1]);
}

// A fragment (16 x 8, row) of k-chunk j from accumulator fragments c[j] of
// the previous GEMM (same rows): k-slot t <-> column 2t, t+4 <-> 2t+1.
__device__ __forceinline__ void a_from_c(const float (&c)[4], float (&a)[4]) {
  a[0] = c[0];
  a[1] = c[2];
  a[2] = c[1];
  a[3] = c[3];
}

// Y[s][o] = X[s][:] . W[o][:] for the warp's 32 samples x 32 outputs with X
// as accumulator fragments x[mt][j] (K = 32) and W rows of stride WS read
// with the permuted k order: b0 = W[8nt+g][8j+2t], b1 = W[8nt+g][8j+2t+1].
template <int NT>
__device__ __forceinline__ void gemm_rr(float (&y)[2][NT][4], const float (&x)[2][4][4], const float* __restrict__ wg) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) y[mt][nt][0] = y[mt][nt][1] = y[mt][nt][2] = y[mt][nt][3] = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t ah[2][4], al[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      float a[4];
      a_from_c(x[mt][j], a);
      split4(a, ah[mt], al[mt]);
    }
    mma_passes<2, NT>(y, ah, al, [&](int nt) { return ld2(wg + nt * 8 * WS + 8 * j); });
  }
}

// D[m][n] = sum_s A^T[s][m] B^T[s][n] over the block's 32 samples, with both
// operands feature-major in smem (rows of stride WS): a0 = AT[16mt+g][8j+2t],
// a2 = AT[16mt+g][8j+2t+1] (LDS.64), b likewise from BT rows 8nt+g.
template <int MT, int NT>
__device__ __forceinline__ void gemm_ss(float (&d)[MT][NT][4], const float* __restrict__ at,
                                        const float* __restrict__ bt, int g, int t) {
  at += g * WS + 2 * t;
  bt += g * WS + 2 * t;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) d[mt][nt][0] = d[mt][nt][1] = d[mt][nt][2] = d[mt][nt][3] = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t ah[MT][4], al[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const float2 u = ld2(at + mt * 16 * WS + 8 * j), v = ld2(at + (mt * 16 + 8) * WS + 8 * j);
      const float a[4] = {u.x, v.x, u.y, v.y};
      split4(a, ah[mt], al[mt]);
    }
    mma_passes<MT, NT>(d, ah, al, [&](int nt) { return ld2(bt + nt * 8 * WS + 8 * j); });
  }
}

// accumulator fragment element r of tile (mt, nt): row 16mt + g + 8(r>>1), column 8nt + 2t + (r&1)
__device__ __forceinline__ int frag_row(int mt, int r, int g) { return 16 * mt + g + 8 * (r >> 1); }
__device__ __forceinline__ int frag_col(int nt, int r, int t) { return 8 * nt + 2 * t + (r & 1); }

// feature-major store of a [32 samples][32 features] fragment set: XT[f][s]
__device__ __forceinline__ void store_t(float* __restrict__ xt, const float (&y)[2][4][4], int g, int t) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r) xt[frag_col(nt, r, t) * WS + frag_row(mt, r, g)] = y[mt][nt][r];
}

// bias + ReLU in place, ReLU mask bits (bit (mt*4+nt)*4+r)
__device__ __forceinline__ uint32_t bias_relu(float (&y)[2][4][4], const float* __restrict__ bias, int t) {
  uint32_t m = 0;
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const float2 bb = ld2(bias + 8 * nt + 2 * t);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float v = relu(y[mt][nt][r] + ((r & 1) ? bb.y : bb.x));
        y[mt][nt][r] = v;
        m |= uint32_t(v > 0.f) << ((mt * 4 + nt) * 4 + r);
      }
  }
  return m;
}
__device__ __forceinline__ void apply_mask(float (&y)[2][4][4], uint32_t m) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (!((m >> ((mt * 4 + nt) * 4 + r)) & 1u)) y[mt][nt][r] = 0.f;
}
// per-row sums of a feature-major [32][WS] tile (32 samples each): lane = row
__device__ __forceinline__ float row_sum32(const float* __restrict__ p) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kSB; k += 4) {
    const float4 v = ld4(p + k);
    s += (v.x + v.y) + (v.z + v.w);
  }
  return s;
}

__device__ __forceinline__ void cp_async4(float* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

template <int SFIX>
__global__ void __launch_bounds__(NTHR, 1) kh32_train_kernel(const __grid_constant__ KParams p) {
  static_assert(SFIX > 0 && SFIX <= kSB, "compile-time points per ray");
  extern __shared__ __align__(16) float smem[];
  int item = blockIdx.x, si = 0;
  if (p.n_stacks > 1 && item >= p.s[1].item_base) si = 1;
  const KStack& st = p.s[si];
  item -= st.item_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int k = st.items ? st.items[2 * item] : item / st.P;
  const int split_ = st.items ? st.items[2 * item + 1] : item % st.P;
  constexpr int S = SFIX, G = kSB / S;
  const int Rk = st.model_rays ? min(st.model_rays[k], st.R) : st.R;
  const int nblk = (Rk + G - 1) / G;
  const int Pk = max(1, (nblk + st.chunk - 1) / st.chunk);
  if (split_ >= Pk) return;
  const int bps = (nblk + Pk - 1) / Pk;
  const int blk0 = split_ * bps, blk1 = min(nblk, blk0 + bps);
  const int nact = blk1 - blk0;  // warps with a block (<= NW: chunk <= 8 blocks)
  const int blk = blk0 + warp;
  const bool has = warp < nact;
  const int D = st.D;

  float* sW = smem;
  float* wr = smem + kWFloats + warp * kWarpFloats;
  float* ET = wr + rET;
  float* O = wr + rO;
  float* tS = wr + rTs;
  float* sTg = wr + rTg;
  float* sDb = wr + rDb;
  const int r_begin = blk * G;
  const int nr = has ? min(G, Rk - r_begin) : 0;
  const int ns = nr * S;
  const int64_t r0 = int64_t(k) * st.R + r_begin, gs0 = r0 * S;

  // ---- this warp's encoded rows [ns][D] -> ET[f][s] (cp.async, overlaps the weight staging)
  if (has) {
    const float* src = st.enc + gs0 * D;
    const float invD = 1.0f / float(D);
    for (int idx = lane; idx < ns * D; idx += 32) {
      const int s = __float2int_rz((float(idx) + 0.5f) * invD), f = idx - s * D;
      cp_async4(ET + f * WS + s, src + idx);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // zero the rest of ET: feature rows >= D, sample columns >= ns
    for (int f = D; f < D0; ++f) ET[f * WS + lane] = 0.f;
    for (int f = 0; f < D; ++f)
      if (lane >= ns) ET[f * WS + lane] = 0.f;
    if (lane < ns) tS[lane] = st.t[gs0 + lane];
    else tS[lane] = 0.f;
    if (lane < nr) {
      float* t8 = sTg + lane * kTgt;
      const int64_t rg = r0 + lane;
      t8[0] = st.tdepth[rg];
      t8[1] = st.tcol[rg * 3 + 0];
      t8[2] = st.tcol[rg * 3 + 1];
      t8[3] = st.tcol[rg * 3 + 2];
      t8[4] = st.tmask[rg] != 0 ? 1.f : 0.f;
      t8[5] = st.valid[rg] != 0 ? 1.f : 0.f;
      t8[6] = st.ok[rg] != 0 ? 1.f : 0.f;
    }
  }

  // ---- stage the model's weights: natural rows by cp.async (forward), then
  // the transposed copies the dx GEMMs read, built from shared memory
  {
    const float* gp = st.params + int64_t(k) * st.block;
    const int fi0 = st.fi0;
    for (int i = tid; i < H * D0; i += NTHR) {
      const int o = i / D0, c = i % D0;
      if (c < fi0) cp_async4(sW + oW0 + o * WS + c, gp + st.w_off[0] + o * fi0 + c);
      else sW[oW0 + o * WS + c] = 0.f;
    }
    for (int i = tid; i < 2 * H * H; i += NTHR) {
      const int l = 1 + i / (H * H), r = i % (H * H), o = r / H, c = r % H;
      cp_async4(sW + (l == 1 ? oW1 : oW2) + o * WS + c, gp + st.w_off[l] + r);
    }
    for (int i = tid; i < 8 * H; i += NTHR) {
      const int o = i / H, c = i % H;
      if (o < 4) cp_async4(sW + oW3 + o * WS + c, gp + st.w_off[3] + o * H + c);
      else sW[oW3 + o * WS + c] = 0.f;
    }
    if (tid < H) {
      cp_async4(sW + oB0 + tid, gp + st.b_off[0] + tid);
      cp_async4(sW + oB1 + tid, gp + st.b_off[1] + tid);
      cp_async4(sW + oB2 + tid, gp + st.b_off[2] + tid);
    }
    if (tid < 8) {
      if (tid < 4) cp_async4(sW + oB3 + tid, gp + st.b_off[3] + tid);
      else sW[oB3 + tid] = 0.f;
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int i = tid; i < 2 * H * H; i += NTHR) {
      const int l = i / (H * H), r = i % (H * H), o = r / H, c = r % H;
      sW[(l == 0 ? oW1T : oW2T) + c * WS + o] = sW[(l == 0 ? oW1 : oW2) + o * WS + c];
    }
    for (int i = tid; i < 8 * H; i += NTHR) {
      const int o = i % 8, c = i / 8;
      sW[oW3T + c * 8 + o] = sW[oW3 + o * WS + c];
    }
  }
  __syncthreads();

  if (has) {
    // ---------------- forward ----------------
    float xa[2][4][4], xb[2][4][4];
    uint32_t m1, m2, m3;
    {  // layer 0: A from ET (feature-major), K = 40 (5 chunks)
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) xa[mt][nt][0] = xa[mt][nt][1] = xa[mt][nt][2] = xa[mt][nt][3] = 0.f;
      const float* wg = sW + oW0 + g * WS + 2 * t;
#pragma unroll
      for (int j = 0; j < D0 / 8; ++j) {
        uint32_t ah[2][4], al[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const float* e = ET + (8 * j + 2 * t) * WS + 16 * mt + g;
          const float a[4] = {e[0], e[8], e[WS], e[WS + 8]};
          split4(a, ah[mt], al[mt]);
        }
        mma_passes<2, 4>(xa, ah, al, [&](int nt) { return ld2(wg + nt * 8 * WS + 8 * j); });
      }
      m1 = bias_relu(xa, sW + oB0, t);
      store_t(wr + rX1, xa, g, t);
    }
    gemm_rr<4>(xb, xa, sW + oW1 + g * WS + 2 * t);  // layer 1
    m2 = bias_relu(xb, sW + oB1, t);
    store_t(wr + rX2, xb, g, t);
    gemm_rr<4>(xa, xb, sW + oW2 + g * WS + 2 * t);  // layer 2
    m3 = bias_relu(xa, sW + oB2, t);
    store_t(wr + rX3, xa, g, t);
    {  // output layer (4 logits, N padded to 8) -> sigmoid -> O[c][s]
      float z[2][1][4];
      gemm_rr<1>(z, xa, sW + oW3 + g * WS + 2 * t);
      if (t < 2) {
        const float2 bb = ld2(sW + oB3 + 2 * t);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int s = frag_row(mt, r, g), c = 2 * t + (r & 1);
            O[c * kOL + s] = s < ns ? sigmoid_f(z[mt][0][r] + ((r & 1) ? bb.y : bb.x)) : 0.f;
          }
      }
    }
    __syncwarp();

    // ---------------- render + L1 losses + loss grads + render backward ----------------
    if (lane < nr) {
      RayTargets tg;
      const float* t8 = sTg + lane * kTgt;
      tg.depth = t8[0];
      tg.colour[0] = t8[1];
      tg.colour[1] = t8[2];
      tg.colour[2] = t8[3];
      tg.mask = t8[4] != 0.f;
      tg.valid = t8[5] != 0.f;
      tg.ok = t8[6] != 0.f;
      const RayLossGrad lg = render_ray_smem<S, kOL>(O, tS, lane * S, tg, st.wc, st.wo);
      const int64_t rg = r0 + lane;
      st.ray_terms[rg * 3 + 0] = lg.l_depth;
      st.ray_terms[rg * 3 + 1] = lg.l_colour;
      st.ray_terms[rg * 3 + 2] = lg.l_occ;
    }
    __syncwarp();
    if (lane >= ns) {
#pragma unroll
      for (int c = 0; c < 4; ++c) O[c * kOL + lane] = 0.f;  // pad samples carry zero gradients
    }
    __syncwarp();

    // ---------------- backward ----------------
    float* R = wr + rX3;  // dZ staging (feature-major) once X3 is consumed
    {
      // output layer: dW3^T = X3^T dZ3 (M = inputs, N = outputs padded to 8)
      float d3[2][1][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) d3[mt][0][0] = d3[mt][0][1] = d3[mt][0][2] = d3[mt][0][3] = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t ah[2][4], al[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const float2 u = ld2(R + (16 * mt + g) * WS + 8 * j + 2 * t), v = ld2(R + (16 * mt + g + 8) * WS + 8 * j + 2 * t);
          const float a[4] = {u.x, v.x, u.y, v.y};
          split4(a, ah[mt], al[mt]);
        }
        mma_passes<2, 1>(d3, ah, al,
                         [&](int) { return g < 4 ? ld2(O + g * kOL + 8 * j + 2 * t) : make_float2(0.f, 0.f); });
      }
      // dX3 = dZ3 W3 (K = outputs padded to 8: one chunk)
      float dx[2][4][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dx[mt][nt][0] = dx[mt][nt][1] = dx[mt][nt][2] = dx[mt][nt][3] = 0.f;
      {
        uint32_t ah[2][4], al[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          float a[4] = {0.f, 0.f, 0.f, 0.f};
          if (t < 2) {
            const int s = 16 * mt + g;
            a[0] = O[(2 * t) * kOL + s];
            a[1] = O[(2 * t) * kOL + s + 8];
            a[2] = O[(2 * t + 1) * kOL + s];
            a[3] = O[(2 * t + 1) * kOL + s + 8];
          }
          split4(a, ah[mt], al[mt]);
        }
        mma_passes<2, 4>(dx, ah, al, [&](int nt) { return ld2(sW + oW3T + (8 * nt + g) * 8 + 2 * t); });
      }
      float db3 = 0.f;
      if (lane < 4) db3 = row_sum32(O + lane * kOL);
      apply_mask(dx, m3);  // dZ2
      __syncwarp();        // X3 and dZ3 consumed
      // dW3 -> O as [o][32 inputs]; db3 -> sDb[96..99]
      if (t < 2) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int r = 0; r < 4; ++r) O[(2 * t + (r & 1)) * H + frag_row(mt, r, g)] = d3[mt][0][r];
      }
      if (lane < 4) sDb[3 * H + lane] = db3;
      store_t(R, dx, g, t);
      __syncwarp();

      // layer 2: dW2 = dZ2^T X2, dX2 = dZ2 W2 -> dZ1
      float dw[2][4][4];
      gemm_ss<2, 4>(dw, R, wr + rX2, g, t);
      sDb[2 * H + lane] = row_sum32(R + lane * WS);
      gemm_rr<4>(xb, dx, sW + oW2T + g * WS + 2 * t);
      apply_mask(xb, m2);
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int r = 0; r < 4; ++r) wr[rX2 + frag_row(mt, r, g) * H + frag_col(nt, r, t)] = dw[mt][nt][r];
      store_t(R, xb, g, t);
      __syncwarp();

      // layer 1: dW1 = dZ1^T X1, dX1 = dZ1 W1 -> dZ0
      gemm_ss<2, 4>(dw, R, wr + rX1, g, t);
      sDb[H + lane] = row_sum32(R + lane * WS);
      gemm_rr<4>(dx, xb, sW + oW1T + g * WS + 2 * t);
      apply_mask(dx, m1);
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int r = 0; r < 4; ++r) wr[rX1 + frag_row(mt, r, g) * H + frag_col(nt, r, t)] = dw[mt][nt][r];
      store_t(R, dx, g, t);
      __syncwarp();

      // layer 0: dW0 = dZ0^T X0 (N = 40 input features), no dx into the input (models.py:394)
      float d0[2][5][4];
      gemm_ss<2, 5>(d0, R, ET, g, t);
      sDb[lane] = row_sum32(R + lane * WS);
      __syncwarp();
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 5; ++nt)
#pragma unroll
          for (int r = 0; r < 4; ++r) ET[frag_row(mt, r, g) * D0 + frag_col(nt, r, t)] = d0[mt][nt][r];
    }
  }

  // ---------------- gradient write-out: warps summed in warp order ----------------
  __syncthreads();
  const int k_block = st.block, fi0 = st.fi0;
  float* gdst = (Pk == 1) ? st.grads + int64_t(k) * k_block : st.partials + (int64_t(k) * st.P + split_) * k_block;
  const float* w0p = smem + kWFloats;
  auto wsum = [&](int off) {
    float v = w0p[off];
    for (int w = 1; w < nact; ++w) v += w0p[w * kWarpFloats + off];
    return v;
  };
  for (int i = tid; i < H * fi0; i += NTHR) gdst[st.w_off[0] + i] = wsum(rET + (i / fi0) * D0 + i % fi0);
  for (int i = tid; i < H * H; i += NTHR) {
    gdst[st.w_off[1] + i] = wsum(rX1 + i);
    gdst[st.w_off[2] + i] = wsum(rX2 + i);
  }
  for (int i = tid; i < 4 * H; i += NTHR) gdst[st.w_off[3] + i] = wsum(rO + i);
  if (tid < H) {
    gdst[st.b_off[0] + tid] = wsum(rDb + tid);
    gdst[st.b_off[1] + tid] = wsum(rDb + H + tid);
    gdst[st.b_off[2] + tid] = wsum(rDb + 2 * H + tid);
  }
  if (tid < 4) gdst[st.b_off[3] + tid] = wsum(rDb + 3 * H + tid);

  // ---------------- per-model finalisation (last chunk to finish) ---------
  bool finite = true;
  if (Pk > 1) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&st.counters[k], 1) == Pk - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float* pb = st.partials + int64_t(k) * st.P * k_block;
    float* gw = st.grads + int64_t(k) * k_block;
    for (int i = tid; i < k_block / 4; i += NTHR) {
      float4 v = __ldcg(reinterpret_cast<const float4*>(pb + 4 * i));
      for (int u = 1; u < Pk; ++u) {
        const float4 w = __ldcg(reinterpret_cast<const float4*>(pb + int64_t(u) * k_block + 4 * i));
        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
      }
      st4(gw + 4 * i, v);
      finite &= isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
    }
    if (tid == 0) st.counters[k] = 0;
  } else {
    __syncthreads();
    const float* gk = st.grads + int64_t(k) * k_block;
    for (int i = tid; i < k_block / 4; i += NTHR) {
      const float4 v = ld4(gk + 4 * i);
      finite &= isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
    }
  }
  const bool all_finite = __syncthreads_and(finite);
  finalize_model(st, k, all_finite, true, smem + kWFloats, NW * kWarpFloats);
}

}  // namespace kh32

// True when every stack of the launch fits the tensor-path kernel: hidden 32,
// 4 layers, encoded input (<= 40 features), 10 points per ray, and at most
// 8 ray blocks per work item.
bool kh32_supported(const KParams& p) {
  for (int i = 0; i < p.n_stacks; ++i) {
    const KStack& s = p.s[i];
    if (s.H != kh32::H || s.L != 4 || s.D > kh32::D0 || s.fi0 > kh32::D0 || s.tc || s.S != 10 || s.pts ||
        !s.enc || s.chunk > kh32::NW)
      return false;
  }
  return p.n_stacks > 0;
}

int launch_kh32(const KParams& p, int grid, cudaStream_t s) {
  const void* fn = reinterpret_cast<const void*>(kh32::kh32_train_kernel<10>);
  VM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kh32::kSmem)));
  void* args[] = {const_cast<KParams*>(&p)};
  VM_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kh32::NTHR), args, kh32::kSmem, s));
  return VM_OK;
}

}  // namespace vm
