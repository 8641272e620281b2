// KF32: the fused train step specialised for the reference's object model --
// hidden 32, 4 layers (trainer.py:70-71, models.py:19-55), input width <= 36
// -- with every dimension a compile-time constant, so each shared-memory
// operand of the FFMA micro-GEMMs is a per-lane base register plus an
// immediate offset (no per-access index arithmetic).
//
// Math: models.py:311-398 (forward/backward), render.py:230-333 (render,
// losses, grads), trainer.py:480-506 (the train_on_batch chain); identical
// to the generic kernel in vm_mlp.cu (same per-output summation order).
//
// Execution (B200, sm_100a):
//  * CTA = 8 warps = 4 teams of 2 warps; two CTAs per SM (128 registers,
//    ~95 KB smem each), so 16 warps share an SM's FFMA pipes.
//  * Work item (one CTA) = (model, chunk of VM_KF_CHUNK consecutive 32-sample
//    blocks).  The chunking depends only on the model's own ray count, so the
//    gradient summation order never depends on K (vectorised == sequential,
//    test_trainer.py:117-132) while a few hundred CTAs spread over the SMs.
//  * A team owns one 32-sample block (floor(32/S) whole rays) at a time; warp
//    wt computes outputs [16wt, 16wt+16) of every layer (forward, dx) and the
//    same rows of every weight gradient, accumulated in registers across the
//    team's blocks.  Activations are feature-major in smem (row stride 36
//    floats), weights are rows of stride 36 (bank-conflict free for both the
//    row reads of the forward and the column reads of dx).
//  * End of item: team partials summed in team order into the chunk partial;
//    the chunk that finishes last (atomic ticket) sums the partials in chunk
//    order and finalises the model (loss sums in numpy's pairwise order,
//    update mask, non-finite flags) -- no separate reduce kernel.
#include <algorithm>

#include "vm_mlp.cuh"

namespace vm {
namespace kf32 {

// partial unrolling keeps the per-block instruction stream (~2k
// instructions instead of ~11k straight-line) inside the instruction cache
#ifndef VM_KF_UNROLL_FWD
#define VM_KF_UNROLL_FWD 2
#endif
#ifndef VM_KF_UNROLL_DX
#define VM_KF_UNROLL_DX 4
#endif
#ifndef VM_KF_UNROLL_DW
#define VM_KF_UNROLL_DW 2
#endif
constexpr int kUnrollFwd = VM_KF_UNROLL_FWD, kUnrollDx = VM_KF_UNROLL_DX, kUnrollDw = VM_KF_UNROLL_DW;
constexpr int H = 32, L = 4, T = 2, OW = 16, NT = 4;  // hidden, layers, warps/team, outputs/warp, teams
constexpr int WS = 36;                                 // smem weight row stride (floats)
constexpr int D0 = 36;                                 // layer-0 input rows (fan-in padded)
constexpr int NW = NT * T, NTHR = NW * 32;
// smem weight image (floats): W0 [32][36] b0 [32] W1 [32][36] b1 W2 [32][36] b2 W3 [4][36] b3 [4]
constexpr int oW0 = 0, oB0 = oW0 + H * WS, oW1 = oB0 + H, oB1 = oW1 + H * WS, oW2 = oB1 + H, oB2 = oW2 + H * WS,
              oW3 = oB2 + H, oB3 = oW3 + 4 * WS, kWFloats = (oB3 + 4 + 31) / 32 * 32;
// per-team activation region (floats), rows of kLD = 36
constexpr int rE = 0, rA1 = rE + D0, rA2 = rA1 + H, rA3 = rA2 + H, rO = rA3 + H, kRows = rO + 4;
constexpr int kTgt = 8;  // per-ray targets staged in smem: depth, rgb, mask, valid, ok

// Per-team shared-memory layout (floats) for a compile-time S (SFIX > 0) or a
// runtime S (SFIX == 0).  With SFIX > 0 a block holds G = 32/S rays, and the
// team owns a staging area the next block's encoded rows, t, targets and
// flag words are copied into with cp.async while the current block computes
// (the enc input path): [G*S][D] raw rows | t [G*S] | targets [G][4] | flag
// words [3][kFw].
template <int SFIX>
struct Lay {
  static constexpr int G = SFIX > 0 ? kSB / SFIX : kSB;
  static constexpr int kTs = SFIX > 0 ? kSB : 2 * kSB;  // t (+ the runtime-S render scratch)
  static constexpr int kFw = SFIX > 0 ? (G + 3) / 4 + 1 : 0;  // 4-byte words covering G flag bytes
  static constexpr int kStEnc = SFIX > 0 ? G * SFIX * D0 : 0;
  static constexpr int kStT = SFIX > 0 ? G * SFIX : 0;
  static constexpr int kStTg = kStEnc + kStT, kStFl = kStTg + 4 * G;
  static constexpr int kStage = SFIX > 0 ? kStFl + 3 * kFw : 0;
  static constexpr int oTs = kRows * kLD, oDb = oTs + kTs, oTg = oDb + 3 * H + 4, oStage = oTg + G * kTgt;
  static constexpr int kTeam = oStage + kStage;
  static constexpr size_t kSmem = size_t(kWFloats + NT * kTeam) * 4 + 64;
};
// two CTAs per SM: 2 x (dynamic + ~1.6 KB static + 1 KB reserved) <= 228 KB
static_assert(Lay<10>::kSmem + 1600 + 1024 <= 228 * 1024 / 2, "KF32<10> no longer fits two CTAs per SM");

__device__ __forceinline__ void cp_async4(float* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ float relu(float z) {
  float r;
  asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(z));  // np.maximum(z, 0): NaN propagates
  return r;
}

// Y[o][4a..4a+3] = relu(b[o] + sum_k W[o][k] X[k][4a..]) for the warp's 16 outputs
// o = o0 + b + 4j.  xb = X + 4a, wb = W + (o0+b)*WS.
template <int K>
__device__ __forceinline__ void fwd16(const float* __restrict__ wb, const float* __restrict__ bias,
                                      const float* __restrict__ xb, float* __restrict__ yb) {
  float acc[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll(kUnrollFwd)
  for (int k = 0; k < K; k += 4) {
    const float4 x0 = ld4(xb + (k + 0) * kLD), x1 = ld4(xb + (k + 1) * kLD);
    const float4 x2 = ld4(xb + (k + 2) * kLD), x3 = ld4(xb + (k + 3) * kLD);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 w = ld4(wb + j * 4 * WS + k);
      acc[j][0] = fmaf(w.x, x0.x, acc[j][0]); acc[j][1] = fmaf(w.x, x0.y, acc[j][1]);
      acc[j][2] = fmaf(w.x, x0.z, acc[j][2]); acc[j][3] = fmaf(w.x, x0.w, acc[j][3]);
      acc[j][0] = fmaf(w.y, x1.x, acc[j][0]); acc[j][1] = fmaf(w.y, x1.y, acc[j][1]);
      acc[j][2] = fmaf(w.y, x1.z, acc[j][2]); acc[j][3] = fmaf(w.y, x1.w, acc[j][3]);
      acc[j][0] = fmaf(w.z, x2.x, acc[j][0]); acc[j][1] = fmaf(w.z, x2.y, acc[j][1]);
      acc[j][2] = fmaf(w.z, x2.z, acc[j][2]); acc[j][3] = fmaf(w.z, x2.w, acc[j][3]);
      acc[j][0] = fmaf(w.w, x3.x, acc[j][0]); acc[j][1] = fmaf(w.w, x3.y, acc[j][1]);
      acc[j][2] = fmaf(w.w, x3.z, acc[j][2]); acc[j][3] = fmaf(w.w, x3.w, acc[j][3]);
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float bb = bias[4 * j];
    st4(yb + j * 4 * kLD, make_float4(relu(acc[j][0] + bb), relu(acc[j][1] + bb), relu(acc[j][2] + bb),
                                      relu(acc[j][3] + bb)));
  }
}

// A[i][4a..] <- (sum_o W[o][i] G[o][4a..]) * (A > 0) for the warp's inputs
// i = i0 + 4b .. +3 (in place).  gb = G + 4a, wb = W + i0 + 4b, ab = A + (i0+4b)*kLD + 4a.
template <int K>
__device__ __forceinline__ void dx16(const float* __restrict__ wb, const float* __restrict__ gb,
                                     float* __restrict__ ab) {
  float acc[4][4];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.f;
#pragma unroll(kUnrollDx)
  for (int o = 0; o < K; ++o) {
    const float4 g = ld4(gb + o * kLD);
    const float4 w = ld4(wb + o * WS);
    acc[0][0] = fmaf(w.x, g.x, acc[0][0]); acc[0][1] = fmaf(w.x, g.y, acc[0][1]);
    acc[0][2] = fmaf(w.x, g.z, acc[0][2]); acc[0][3] = fmaf(w.x, g.w, acc[0][3]);
    acc[1][0] = fmaf(w.y, g.x, acc[1][0]); acc[1][1] = fmaf(w.y, g.y, acc[1][1]);
    acc[1][2] = fmaf(w.y, g.z, acc[1][2]); acc[1][3] = fmaf(w.y, g.w, acc[1][3]);
    acc[2][0] = fmaf(w.z, g.x, acc[2][0]); acc[2][1] = fmaf(w.z, g.y, acc[2][1]);
    acc[2][2] = fmaf(w.z, g.z, acc[2][2]); acc[2][3] = fmaf(w.z, g.w, acc[2][3]);
    acc[3][0] = fmaf(w.w, g.x, acc[3][0]); acc[3][1] = fmaf(w.w, g.y, acc[3][1]);
    acc[3][2] = fmaf(w.w, g.z, acc[3][2]); acc[3][3] = fmaf(w.w, g.w, acc[3][3]);
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float* p = ab + c * kLD;
    const float4 av = ld4(p);
    st4(p, make_float4(av.x > 0.f ? acc[c][0] : 0.f, av.y > 0.f ? acc[c][1] : 0.f, av.z > 0.f ? acc[c][2] : 0.f,
                       av.w > 0.f ? acc[c][3] : 0.f));
  }
}

// dW[o][i] += sum_s G[o][s] X[i][s] over the block's 32 samples for rows
// o = o0 + r + 4j (j < NJ) and columns i = c + 8q (q < NQ).
// gb = G + (o0+r)*kLD, xb = X + c*kLD.
template <int NJ, int NQ>
__device__ __forceinline__ void dw(float (&acc)[NJ][NQ], const float* __restrict__ gb, const float* __restrict__ xb) {
#pragma unroll(kUnrollDw)
  for (int s = 0; s < kSB; s += 4) {
    float4 g[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) g[j] = ld4(gb + j * 4 * kLD + s);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const float4 x = ld4(xb + q * 8 * kLD + s);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        float v = acc[j][q];
        v = fmaf(g[j].x, x.x, v);
        v = fmaf(g[j].y, x.y, v);
        v = fmaf(g[j].z, x.z, v);
        v = fmaf(g[j].w, x.w, v);
        acc[j][q] = v;
      }
    }
  }
}

// team bias-gradient sum: the two sample halves (lane / 16) combined, then
// added to the warp's 16 rows in smem (fixed order: deterministic)
__device__ __forceinline__ void bias_acc(float* __restrict__ dst, float v, int lane) {
  v += __shfl_xor_sync(0xffffffffu, v, 16);
  if (lane < 16) dst[lane] += v;
}

// sum over the 32 samples of row `row` split in two halves of 16 (lane / 16)
__device__ __forceinline__ float rowsum16(const float* __restrict__ p) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; k += 4) {
    const float4 v = ld4(p + k);
    s += (v.x + v.y) + (v.z + v.w);
  }
  return s;
}

struct Grads {
  float w0[4][4];     // layer 0: rows o0+r+4j, cols c+8q
  float w0x[2];       // layer 0 cols 32..35: row o0 + lane%16, cols 32 + 2*(lane/16) + {0,1}
  float wh[2][4][4];  // layers 1, 2
  float wl[2];        // output layer: row r, cols o0 + c + 8q
};

__device__ __forceinline__ void team_bar(int team) {
  asm volatile("bar.sync %0, 64;" ::"r"(team + 1) : "memory");
}

template <int SFIX>
__device__ __forceinline__ void train_item(const KParams& p, int item, float* smem) {
  int si = 0;
  if (p.n_stacks > 1 && item >= p.s[1].item_base) si = 1;
  const KStack& st = p.s[si];
  item -= st.item_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int team = warp / T, wt = warp % T, o0 = wt * OW;
  const int k = st.items ? st.items[2 * item] : item / st.P;
  const int split = st.items ? st.items[2 * item + 1] : item % st.P;
  const int S = SFIX > 0 ? SFIX : st.S, G = kSB / S;
  // this model's live rays (config 3: padding rows beyond are skipped) and
  // its chunking, a function of its own ray count only
  const int Rk = st.model_rays ? min(st.model_rays[k], st.R) : st.R;
  const int nblk = (Rk + G - 1) / G;
  const int Pk = max(1, (nblk + st.chunk - 1) / st.chunk);
  if (split >= Pk) return;  // dead chunk of a short model (grid without a work-item table)
  using LY = Lay<SFIX>;
  constexpr int kTeamFloats = LY::kTeam;
  float* base = smem + kWFloats + team * kTeamFloats;
  float* tS = base + LY::oTs;
  const int bps = (nblk + Pk - 1) / Pk;
  const int blk0 = split * bps, blk1 = min(nblk, blk0 + bps);

  // enc input with a compile-time S: the next block's rows, t, targets and
  // flag bytes are copied into the team's staging area by warp 1 with
  // cp.async while the current block computes (issued in the render window,
  // where warp 1 would otherwise idle), so no block waits on a global load.
  const bool pf = SFIX > 0 && st.pts == nullptr;
  float* stg = base + LY::oStage;
  const int D = st.D;
  auto prefetch = [&](int blkn) {  // warp 1 (wt == 1) only
    const int rb = blkn * G;
    const int nrn = min(G, Rk - rb), nsn = nrn * S;
    const int64_t r0 = int64_t(k) * st.R + rb, g0 = r0 * S;
    const float* src = st.enc + g0 * D;
    for (int i = lane; i < nsn * D; i += 32) cp_async4(stg + i, src + i);
    if (lane < nsn) cp_async4(stg + LY::kStEnc + lane, st.t + g0 + lane);
    if (lane < nrn) {
      float* d = stg + LY::kStTg + 4 * lane;
      cp_async4(d, st.tdepth + r0 + lane);
      cp_async4(d + 1, st.tcol + (r0 + lane) * 3);
      cp_async4(d + 2, st.tcol + (r0 + lane) * 3 + 1);
      cp_async4(d + 3, st.tcol + (r0 + lane) * 3 + 2);
    }
    // flag bytes: the aligned 4-byte words covering bytes [r0, r0 + nrn)
    // (inside the allocation: torch rounds device allocations to 512 B)
    if (lane < 3 * LY::kFw) {
      const int a = lane / LY::kFw, j = lane % LY::kFw;
      const uint8_t* arr = a == 0 ? st.tmask : (a == 1 ? st.valid : st.ok);
      const uintptr_t w0 = reinterpret_cast<uintptr_t>(arr + r0) & ~uintptr_t(3);
      const uintptr_t wl = reinterpret_cast<uintptr_t>(arr + r0 + nrn - 1) & ~uintptr_t(3);
      if (w0 + 4 * uintptr_t(j) <= wl)
        cp_async4(stg + LY::kStFl + a * LY::kFw + j, reinterpret_cast<const void*>(w0 + 4 * uintptr_t(j)));
    }
    cp_async_commit();
  };
  if (pf && wt == 1 && blk0 + team < blk1) prefetch(blk0 + team);

  // ---- stage the model's weights (rows of stride WS) and biases
  float* sW = smem;
  {
    const float* gp = st.params + int64_t(k) * st.block;
    const int fi0 = st.fi0;  // arena row length of W0 (<= 36)
    for (int i = tid; i < H * (D0 / 4); i += NTHR) {
      const int row = i / (D0 / 4), c4 = (i % (D0 / 4)) * 4;
      st4(sW + oW0 + row * WS + c4, c4 < fi0 ? ld4(gp + st.w_off[0] + row * fi0 + c4) : make_float4(0, 0, 0, 0));
    }
    for (int i = tid; i < 2 * H * (H / 4); i += NTHR) {
      const int l = 1 + i / (H * (H / 4)), r = i % (H * (H / 4));
      const int row = r / (H / 4), c4 = (r % (H / 4)) * 4;
      st4(sW + (l == 1 ? oW1 : oW2) + row * WS + c4, ld4(gp + st.w_off[l] + row * H + c4));
    }
    if (tid < 4 * (H / 4)) {
      const int row = tid / (H / 4), c4 = (tid % (H / 4)) * 4;
      st4(sW + oW3 + row * WS + c4, ld4(gp + st.w_off[3] + row * H + c4));
    }
    if (tid < H) {
      sW[oB0 + tid] = gp[st.b_off[0] + tid];
      sW[oB1 + tid] = gp[st.b_off[1] + tid];
      sW[oB2 + tid] = gp[st.b_off[2] + tid];
    }
    if (tid < 4) sW[oB3 + tid] = gp[st.b_off[3] + tid];
  }
  __syncthreads();

  Grads acc;
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc.w0[j][q] = 0.f;
  acc.w0x[0] = acc.w0x[1] = 0.f;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc.wh[h][j][q] = 0.f;
  acc.wl[0] = acc.wl[1] = 0.f;
  // bias gradients are summed per team in smem (rows [l*32 + o], output bias at 96..99)
  float* sDb = base + LY::oDb;
  float* sTg = base + LY::oTg;
  for (int i = wt * 32 + lane; i < 3 * H + 4; i += 64) sDb[i] = 0.f;

  // per-lane operand bases (every access below adds a compile-time offset)
  const int a = lane & 7, b = lane >> 3;       // micro-GEMM lane split: sample quad / output phase
  const int r = lane >> 3, c = lane & 7;       // weight-gradient lane split: row phase / column
  const float* wf0 = sW + oW0 + (o0 + b) * WS;
  const float* wf1 = sW + oW1 + (o0 + b) * WS;
  const float* wf2 = sW + oW2 + (o0 + b) * WS;
  // positional-encoding band coefficients 2^b / scale (f64 -> f32, as KF does)
  __shared__ float sCoef[8];
  if (tid < 8) sCoef[tid] = (st.pts && tid < st.n_freq) ? float(double(1u << tid) / double(st.pe_scale[k])) : 0.f;
  __syncthreads();

  for (int blk = blk0 + team; blk < blk1; blk += NT) {
    const int r_begin = blk * G;
    const int nr = min(G, Rk - r_begin);
    const int ns = nr * S;
    const int64_t gs0 = (int64_t(k) * st.R + r_begin) * S;

    // ---- layer-0 input: positional encoding (models.py:286-308 layout) or
    // the caller's encoded rows; warp wt fills samples [16wt, 16wt+16) x 2 halves of features
    {
      const int s = lane;  // each warp of the team encodes all 32 samples' half of the features
      float* E = base + rE * kLD;
      if (pf) {
        // this block's staged rows (issued one block ago): transpose [ns][D]
        // -> E[f][s]; the row stride D (odd for the reference's 33) makes the
        // column reads conflict free
        if (wt == 1) cp_async_wait_all();
        team_bar(team);
        const float* sr = stg + s * D;
#pragma unroll
        for (int f = wt * (D0 / 2); f < (wt + 1) * (D0 / 2); ++f) E[f * kLD + s] = (s < ns && f < D) ? sr[f] : 0.f;
        if (wt == 0) tS[s] = s < ns ? stg[LY::kStEnc + s] : 0.f;
        if (wt == 1 && s < nr) {
          float* t8 = sTg + s * kTgt;
          const float* tg = stg + LY::kStTg + 4 * s;
          t8[0] = tg[0];
          t8[1] = tg[1];
          t8[2] = tg[2];
          t8[3] = tg[3];
          const int rg = int(reinterpret_cast<uintptr_t>(st.tmask + int64_t(k) * st.R + r_begin) & 3) + s;
          const uint8_t* fl = reinterpret_cast<const uint8_t*>(stg + LY::kStFl);
          // each array's words were copied from its own aligned base
          const int rv = int(reinterpret_cast<uintptr_t>(st.valid + int64_t(k) * st.R + r_begin) & 3) + s;
          const int ro = int(reinterpret_cast<uintptr_t>(st.ok + int64_t(k) * st.R + r_begin) & 3) + s;
          t8[4] = fl[rg] != 0 ? 1.f : 0.f;
          t8[5] = fl[4 * LY::kFw + rv] != 0 ? 1.f : 0.f;
          t8[6] = fl[8 * LY::kFw + ro] != 0 ? 1.f : 0.f;
        }
      } else if (st.pts) {
        float pc[3] = {0.f, 0.f, 0.f};
        if (s < ns) {
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) pc[cc] = st.pts[(gs0 + s) * 3 + cc];
        }
        // warp 0: raw coords + bands [0, nb/2); warp 1: the other bands + zero rows
        int f = 0;
        if (st.include_input) {
          if (wt == 0) {
#pragma unroll
            for (int cc = 0; cc < 3; ++cc) E[cc * kLD + s] = pc[cc];
          }
          f = 3;
        }
        const int half = (st.n_freq + 1) / 2;
        const int bb0 = wt == 0 ? 0 : half, bb1 = wt == 0 ? half : st.n_freq;
        for (int bnd = bb0; bnd < bb1; ++bnd) {
          const float coef = sCoef[bnd];
          const int fb = f + 6 * bnd;
#pragma unroll
          for (int cc = 0; cc < 3; ++cc) {
            float sn, cs;
            sincospif(coef * pc[cc], &sn, &cs);
            E[(fb + cc) * kLD + s] = s < ns ? sn : 0.f;
            E[(fb + 3 + cc) * kLD + s] = s < ns ? cs : 0.f;
          }
        }
        if (wt == 1)
          for (int ff = st.D; ff < D0; ++ff) E[ff * kLD + s] = 0.f;
      } else {
        // the block's ns x D encoded values are contiguous: coalesced loads
        // by both warps, transposed into the feature-major tile
        const int D = st.D, tt = wt * 32 + lane;
        const float invD = 1.0f / float(D);
        const float* src = st.enc + gs0 * D;
        for (int idx = tt; idx < ns * D; idx += 64) {
          const int ss = __float2int_rz((float(idx) + 0.5f) * invD), ff = idx - ss * D;
          E[ff * kLD + ss] = __ldg(src + idx);
        }
        for (int idx = tt; idx < (D0 - D) * kSB; idx += 64) E[(D + idx / kSB) * kLD + (idx % kSB)] = 0.f;
        const int np_ = kSB - ns;
        if (np_ > 0)
          for (int idx = tt; idx < np_ * D; idx += 64) {
            const int ff = idx / np_;
            E[ff * kLD + ns + (idx - ff * np_)] = 0.f;
          }
      }
      if (!pf && wt == 0) tS[s] = s < ns ? st.t[gs0 + s] : 0.f;
      if (!pf && wt == 1 && s < nr) {  // this block's ray targets, read early (the render needs them mid-block)
        const int64_t rg = int64_t(k) * st.R + r_begin + s;
        float* t8 = sTg + s * kTgt;
        t8[0] = st.tdepth[rg];
        t8[1] = st.tcol[rg * 3 + 0];
        t8[2] = st.tcol[rg * 3 + 1];
        t8[3] = st.tcol[rg * 3 + 2];
        t8[4] = st.tmask[rg] != 0 ? 1.f : 0.f;
        t8[5] = st.valid[rg] != 0 ? 1.f : 0.f;
        t8[6] = st.ok[rg] != 0 ? 1.f : 0.f;
      }
    }
    team_bar(team);

    // ---------------- forward ----------------
    fwd16<D0>(wf0, sW + oB0 + o0 + b, base + rE * kLD + 4 * a, base + (rA1 + o0 + b) * kLD + 4 * a);
    team_bar(team);
    fwd16<H>(wf1, sW + oB1 + o0 + b, base + rA1 * kLD + 4 * a, base + (rA2 + o0 + b) * kLD + 4 * a);
    team_bar(team);
    fwd16<H>(wf2, sW + oB2 + o0 + b, base + rA2 * kLD + 4 * a, base + (rA3 + o0 + b) * kLD + 4 * a);
    team_bar(team);
    float* O = base + rO * kLD;
    if (wt == 0) {
      // output layer (4 logits -> sigmoid): lane = (sample quad a, output b)
      const float* xb = base + rA3 * kLD + 4 * a;
      const float* wb = sW + oW3 + b * WS;
      float z[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < H; kk += 4) {
        const float4 x0 = ld4(xb + (kk + 0) * kLD), x1 = ld4(xb + (kk + 1) * kLD);
        const float4 x2 = ld4(xb + (kk + 2) * kLD), x3 = ld4(xb + (kk + 3) * kLD);
        const float4 w = ld4(wb + kk);
        z[0] = fmaf(w.x, x0.x, z[0]); z[1] = fmaf(w.x, x0.y, z[1]); z[2] = fmaf(w.x, x0.z, z[2]); z[3] = fmaf(w.x, x0.w, z[3]);
        z[0] = fmaf(w.y, x1.x, z[0]); z[1] = fmaf(w.y, x1.y, z[1]); z[2] = fmaf(w.y, x1.z, z[2]); z[3] = fmaf(w.y, x1.w, z[3]);
        z[0] = fmaf(w.z, x2.x, z[0]); z[1] = fmaf(w.z, x2.y, z[1]); z[2] = fmaf(w.z, x2.z, z[2]); z[3] = fmaf(w.z, x2.w, z[3]);
        z[0] = fmaf(w.w, x3.x, z[0]); z[1] = fmaf(w.w, x3.y, z[1]); z[2] = fmaf(w.w, x3.z, z[2]); z[3] = fmaf(w.w, x3.w, z[3]);
      }
      const float bb = sW[oB3 + b];
      float4 rr;
      rr.x = 4 * a + 0 < ns ? sigmoid_f(z[0] + bb) : 0.f;
      rr.y = 4 * a + 1 < ns ? sigmoid_f(z[1] + bb) : 0.f;
      rr.z = 4 * a + 2 < ns ? sigmoid_f(z[2] + bb) : 0.f;
      rr.w = 4 * a + 3 < ns ? sigmoid_f(z[3] + bb) : 0.f;
      st4(O + b * kLD + 4 * a, rr);
      __syncwarp();
      // render + L1 losses + loss grads + render backward, one lane per ray
      if (lane < nr) {
        const int rg_ = r_begin + lane;
        const int sb = lane * S;
        const int64_t rg = int64_t(k) * st.R + rg_;
        RayTargets tg;
        const float* t8 = sTg + lane * kTgt;
        tg.depth = t8[0];
        tg.colour[0] = t8[1];
        tg.colour[1] = t8[2];
        tg.colour[2] = t8[3];
        tg.mask = t8[4] != 0.f;
        tg.valid = t8[5] != 0.f;
        tg.ok = t8[6] != 0.f;
        RayLossGrad lg;
        if constexpr (SFIX > 0) {
          lg = render_ray_smem<SFIX, kLD>(O, tS, sb, tg, st.wc, st.wo);
        } else {
          float* Tsc = tS + kSB;
          auto occ = [&](int i) { return O[sb + i]; };
          auto col = [&](int i, int cc) { return O[(1 + cc) * kLD + sb + i]; };
          auto tt = [&](int i) { return tS[sb + i]; };
          render_ray_forward(S, occ, col, tt, [&](int i, float v) { Tsc[sb + i] = v; });
          const RayFwd f = render_ray_sums(S, occ, col, tt, [&](int i) { return Tsc[sb + i]; });
          lg = ray_loss_grad(f, tg, st.wc, st.wo);
          render_ray_backward(S, occ, col, tt, [&](int i) { return Tsc[sb + i]; }, lg.dO, lg.dD, lg.dC,
                              [&](int i, float d_occ, const float* d_col) {
                                const float o = O[sb + i];
                                O[sb + i] = __fmul_rn(__fmul_rn(d_occ, o), __fsub_rn(1.0f, o));
#pragma unroll
                                for (int cc = 0; cc < 3; ++cc) {
                                  const float cv = O[(1 + cc) * kLD + sb + i];
                                  O[(1 + cc) * kLD + sb + i] = __fmul_rn(__fmul_rn(d_col[cc], cv), __fsub_rn(1.0f, cv));
                                }
                              });
        }
        st.ray_terms[rg * 3 + 0] = lg.l_depth;
        st.ray_terms[rg * 3 + 1] = lg.l_colour;
        st.ray_terms[rg * 3 + 2] = lg.l_occ;
      }
      __syncwarp();
      // pad samples (beyond the block's rays) carry zero output gradients
      if (lane >= ns) {
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) O[cc * kLD + lane] = 0.f;
      }
    } else if (pf && blk + NT < blk1) {
      prefetch(blk + NT);  // the staging area was consumed at this block's start
    }
    team_bar(team);

    // ---------------- backward ----------------
    // output layer: dW3[r][o0 + c + 8q] (4 x 16 per warp), db3, dx into A3
    {
      const float* g = O + r * kLD;
      const float* x = base + (rA3 + o0 + c) * kLD;
#pragma unroll
      for (int s = 0; s < kSB; s += 4) {
        const float4 gv = ld4(g + s);
        const float4 x0 = ld4(x + s), x1 = ld4(x + 8 * kLD + s);
        acc.wl[0] = fmaf(gv.w, x0.w, fmaf(gv.z, x0.z, fmaf(gv.y, x0.y, fmaf(gv.x, x0.x, acc.wl[0]))));
        acc.wl[1] = fmaf(gv.w, x1.w, fmaf(gv.z, x1.z, fmaf(gv.y, x1.y, fmaf(gv.x, x1.x, acc.wl[1]))));
      }
      if (wt == 0 && lane < 4) {
        float s4 = 0.f;
#pragma unroll
        for (int q = 0; q < kSB; q += 4) {
          const float4 v = ld4(O + lane * kLD + q);
          s4 += (v.x + v.y) + (v.z + v.w);
        }
        sDb[3 * H + lane] += s4;
      }
      __syncwarp();
      dx16<4>(sW + oW3 + o0 + 4 * b, O + 4 * a, base + (rA3 + o0 + 4 * b) * kLD + 4 * a);
    }
    team_bar(team);
    // layer 2: dW2 = G3 x A2^T, db2, dx into A2
    dw<4, 4>(acc.wh[1], base + (rA3 + o0 + r) * kLD, base + (rA2 + c) * kLD);
    bias_acc(sDb + 2 * H + o0, rowsum16(base + (rA3 + o0 + (lane & 15)) * kLD + (lane >> 4) * 16), lane);
    team_bar(team);
    dx16<H>(sW + oW2 + o0 + 4 * b, base + rA3 * kLD + 4 * a, base + (rA2 + o0 + 4 * b) * kLD + 4 * a);
    team_bar(team);
    // layer 1
    dw<4, 4>(acc.wh[0], base + (rA2 + o0 + r) * kLD, base + (rA1 + c) * kLD);
    bias_acc(sDb + H + o0, rowsum16(base + (rA2 + o0 + (lane & 15)) * kLD + (lane >> 4) * 16), lane);
    team_bar(team);
    dx16<H>(sW + oW1 + o0 + 4 * b, base + rA2 * kLD + 4 * a, base + (rA1 + o0 + 4 * b) * kLD + 4 * a);
    team_bar(team);
    // layer 0 (no dx into the input, models.py:394): columns 0..31, then 32..35
    dw<4, 4>(acc.w0, base + (rA1 + o0 + r) * kLD, base + (rE + c) * kLD);
    {
      const float* g = base + (rA1 + o0 + (lane & 15)) * kLD;
      const float* x = base + (rE + 32 + 2 * (lane >> 4)) * kLD;
#pragma unroll
      for (int s = 0; s < kSB; s += 4) {
        const float4 gv = ld4(g + s);
        const float4 x0 = ld4(x + s), x1 = ld4(x + kLD + s);
        acc.w0x[0] = fmaf(gv.w, x0.w, fmaf(gv.z, x0.z, fmaf(gv.y, x0.y, fmaf(gv.x, x0.x, acc.w0x[0]))));
        acc.w0x[1] = fmaf(gv.w, x1.w, fmaf(gv.z, x1.z, fmaf(gv.y, x1.y, fmaf(gv.x, x1.x, acc.w0x[1]))));
      }
    }
    bias_acc(sDb + o0, rowsum16(base + (rA1 + o0 + (lane & 15)) * kLD + (lane >> 4) * 16), lane);
    team_bar(team);
  }

  // ---------------- gradient write-out ----------------
  // each team writes its block (arena layout) into its own activation region,
  // then all threads add the regions in team order
  __syncthreads();
  {
    float* dst = smem + kWFloats + team * kTeamFloats;
    float db[4];  // this lane's bias-gradient sums, read before the region is overwritten
#pragma unroll
    for (int l = 0; l < 3; ++l) db[l] = sDb[l * H + o0 + (lane & 15)];
    db[3] = sDb[3 * H + (lane & 3)];
    __syncwarp();
    team_bar(team);
    const int fi0 = st.fi0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int o = o0 + r + 4 * j;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = c + 8 * q;
        if (i < fi0) dst[st.w_off[0] + o * fi0 + i] = acc.w0[j][q];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[st.w_off[h + 1] + o * H + c + 8 * q] = acc.wh[h][j][q];
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) dst[st.w_off[3] + r * H + o0 + c + 8 * q] = acc.wl[q];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = 32 + 2 * (lane >> 4) + e;
      if (i < fi0) dst[st.w_off[0] + (o0 + (lane & 15)) * fi0 + i] = acc.w0x[e];
    }
    if (lane < 16) {
#pragma unroll
      for (int l = 0; l < 3; ++l) dst[st.b_off[l] + o0 + lane] = db[l];
    }
    if (wt == 0 && lane < 4) dst[st.b_off[3] + lane] = db[3];
  }
  __syncthreads();
  const int k_block = st.block;
  float* gdst = (Pk == 1) ? st.grads + int64_t(k) * k_block : st.partials + (int64_t(k) * st.P + split) * k_block;
  {
    const float* r0 = smem + kWFloats;
    for (int i = tid; i < k_block / 4; i += NTHR) {
      float4 v = ld4(r0 + 4 * i);
#pragma unroll
      for (int t = 1; t < NT; ++t) {
        const float4 u = ld4(r0 + t * kTeamFloats + 4 * i);
        v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
      }
      st4(gdst + 4 * i, v);
    }
  }

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
  finalize_model(st, k, all_finite, true, smem + kWFloats, NT * kTeamFloats);
}

// One CTA per work item, or (p.queue set) a persistent grid whose CTAs pull
// items from an atomic counter: which CTA trains an item never changes its
// bits (the item's blocks, team order and partial slot are fixed by the item).
template <int SFIX>
__global__ void __launch_bounds__(NTHR, 2) kf32_train_kernel(const __grid_constant__ KParams p) {
  extern __shared__ __align__(16) float smem[];
  const unsigned long long t_start = p.trace ? vm_gtime() : 0;
  if (!p.queue) {
    train_item<SFIX>(p, blockIdx.x, smem);
    if (p.trace && threadIdx.x == 0) vm_trace_rec(p.trace, 1, t_start);
    return;
  }
  __shared__ int s_item;
  for (;;) {
    const unsigned long long t0 = p.trace ? vm_gtime() : 0;
    if (threadIdx.x == 0) s_item = atomicAdd(p.queue, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= p.n_items) break;
    train_item<SFIX>(p, item, smem);
    __syncthreads();  // smem (weights, team regions, s_item) free for the next item
    if (p.trace && threadIdx.x == 0) vm_trace_rec(p.trace, 1, t0);
  }
}

}  // namespace kf32

// True when every stack of the launch fits the specialised kernel.
bool kf32_supported(const KParams& p) {
  for (int i = 0; i < p.n_stacks; ++i) {
    const KStack& s = p.s[i];
    if (s.H != kf32::H || s.L != kf32::L || s.D > kf32::D0 || s.fi0 > kf32::D0 || s.tc) return false;
  }
  return true;
}

size_t kf32_smem_bytes() { return kf32::Lay<10>::kSmem > kf32::Lay<0>::kSmem ? kf32::Lay<10>::kSmem : kf32::Lay<0>::kSmem; }

int launch_kf32(const KParams& p, int grid, cudaStream_t s) {
  bool all10 = true;
  for (int i = 0; i < p.n_stacks; ++i) all10 &= p.s[i].S == 10;
  const void* fn = all10 ? reinterpret_cast<const void*>(kf32::kf32_train_kernel<10>)
                         : reinterpret_cast<const void*>(kf32::kf32_train_kernel<0>);
  const size_t smem = all10 ? kf32::Lay<10>::kSmem : kf32::Lay<0>::kSmem;
  VM_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  KParams q = p;
  if (q.queue) {  // persistent: two CTAs per SM pull the items
    static int sms = 0;
    if (!sms) VM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    q.n_items = grid;
    grid = std::min(grid, 2 * sms);  // the counter was zeroed by vm_train_step's init kernel
  }
  void* args[] = {&q};
  VM_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kf32::NTHR), args, smem, s));
  return VM_OK;
}

}  // namespace vm
