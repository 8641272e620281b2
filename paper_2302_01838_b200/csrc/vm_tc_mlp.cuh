// KT: tensor-core (tcgen05, 3xTF32) fused train step for wide per-object MLP
// fields (hidden 128, 4 layers: the reference's background model,
// trainer.py:70-71, models.py:19-55).  Same math as the FFMA kernel KF
// (models.py:311-398 forward/backward, render.py:230-333 render/losses) for
// one 128-row tile of samples (floor(128/S) whole rays) per CTA.
//
// Precision: every GEMM runs as 3xTF32 -- x = hi + lo with hi = rna_tf32(x),
// lo = rna_tf32(x - hi); A.B ~= lo_A.hi_B + hi_A.lo_B + hi_A.hi_B accumulated
// in fp32 in TMEM -- which keeps ~fp32 accuracy (probe: 3e-7 relative to
// sum|ab| for K=32), inside the north star's 1e-4 contract.  The 4-wide
// output layer, render, losses and their gradients run on CUDA cores in fp32
// with the reference's operation order.
//
// On-chip data flow (no activation ever touches HBM):
//  * TMEM (512 columns x 128 lanes, lane = sample row): R0 = MMA accumulator
//    (forward pre-activations, input-gradients, weight-gradient tiles),
//    R1..R3 = activations X1..X3 (fp32), overwritten in place by the
//    back-propagated gradients G2..G0 once they are no longer needed.
//  * Shared memory: a 3-slot ring of 64 KB operand slots (A | B, each a
//    hi/lo pair).  Forward / input-gradient GEMMs stage A = activations or
//    gradients [128 samples][32 features] (core-matrix interleaved, K-major,
//    conflict-free float4 stores by the owning thread) and B = a pre-split,
//    pre-laid-out weight chunk copied with cp.async from an L2-resident image
//    (tc_prep_kernel builds it once per step).  Weight-gradient GEMMs
//    dW = G^T X (K = samples) stage both operands transposed, 32 samples (one
//    warp's TMEM lanes) per chunk, as 128B-swizzled K-major tiles written
//    with conflict-free scalar stores.
//  * Thread 0 issues the MMAs (tcgen05.mma.cta_group::1.kind::tf32) and
//    commits each slot to an mbarrier; staging of chunk c+1 overlaps the MMAs
//    of chunk c.
//  * Weight gradients leave through TMEM -> registers -> the CTA's partial
//    gradient block; bias gradients are warp butterfly reductions; the
//    per-model sum over tiles is reduce_partials_kernel (fixed order).
#pragma once

#include "vm_tc.cuh"

#ifdef VM_TC_DEBUG
__device__ int vm_tc_dbg[256];
#define VM_TC_DBG(i, v) \
  do { if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) reinterpret_cast<volatile int*>(vm_tc_dbg)[i] = (v); } while (0)
#else
#define VM_TC_DBG(i, v) do { } while (0)
#endif

namespace vm {
namespace tck {

constexpr int kTM = 128;       // tile rows = TMEM lanes
constexpr int kThr = 128;      // 4 warps, warp w <-> TMEM lane quadrant w
constexpr int kNS = 3;         // ring slots
constexpr int kSlot = 65536;   // bytes per slot: A (32 KB) | B (32 KB)
constexpr int kHalfSlot = 32768;
constexpr int kK0 = 40;        // layer-0 fan-in padded for the MMA (33 -> 40)
constexpr int kN0 = 48;        // layer-0 fan-in rows of X0^T for dW0 (N % 16)

// Pre-split weight image (floats) per model: chunks of [H rows][kw cols]
// (hi tile then lo tile, interleaved layout), forward W_l (rows = fo, K = fi)
// for l = 0..L-2 and input-gradient W_l^T (rows = fi, K = fo) for l = 1..L-2.
template <int H, int L>
struct Img {
  static constexpr int kC32 = 2 * H * 32;
  static constexpr int kC8 = 2 * H * 8;
  static constexpr int n_chunks = 2 + 2 * (L - 2) * (H / 32);
  __host__ __device__ static constexpr int fwd_off(int l) {
    return l == 0 ? 0 : kC32 + kC8 + (l - 1) * (H / 32) * kC32;
  }
  __host__ __device__ static constexpr int dx_off(int l) { return fwd_off(L - 1) + (l - 1) * (H / 32) * kC32; }
  static constexpr int total = dx_off(L - 1);
};

template <int H, int L>
__global__ void __launch_bounds__(256) tc_prep_kernel(const __grid_constant__ KStack st, float* __restrict__ img) {
  using I = Img<H, L>;
  const int k = blockIdx.y;
  int c = blockIdx.x;
  const float* P = st.params + int64_t(k) * st.block;
  float* out = img + int64_t(k) * I::total;
  // decode chunk id -> (use, layer, chunk, kw, base)
  int l, cc, kw, base;
  bool dx;
  if (c < 2) {
    dx = false; l = 0; cc = c; kw = (c == 0) ? 32 : 8; base = c == 0 ? 0 : I::kC32;
  } else {
    c -= 2;
    const int per = H / 32;
    const int nf = (L - 2) * per;
    dx = c >= nf;
    if (dx) c -= nf;
    l = 1 + c / per;
    cc = c % per;
    kw = 32;
    base = (dx ? I::dx_off(l) : I::fwd_off(l)) + cc * I::kC32;
  }
  const int fi_pad = (l == 0) ? st.fi0 : H;
  const int fi_real = (l == 0) ? st.D : H;
  const float* W = P + st.w_off[l];
  for (int e = threadIdx.x; e < H * kw; e += blockDim.x) {
    const int n = e / kw, kk = e % kw;
    const int kidx = cc * 32 + kk;
    float v;
    if (!dx) v = (kidx < fi_real) ? W[n * fi_pad + kidx] : 0.f;  // rows fo, K = fi
    else v = W[kidx * fi_pad + n];                               // rows fi, K = fo
    float hi, lo;
    tc::split3(v, hi, lo);
    const uint32_t o = tc::ilv_off(n, kk, kw) / 4;
    out[base + o] = hi;
    out[base + H * kw + o] = lo;
  }
}

// byte offset of (row, col) in a 128B-swizzled K-major tile with 32 columns
__device__ __forceinline__ uint32_t sw128_off(int row, int col) {
  return uint32_t(row * 128 + ((((col >> 2) ^ row) & 7) << 4) + (col & 3) * 4);
}

// SWIZZLE_128B K-major descriptor (8-row groups 1024 B apart)
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  return tc::sdesc(saddr, 16, 1024) | (uint64_t(2) << 61);
}

// Layer-0 input row of one sample: the positional encoding of models.py:286-308
// (f32 sincospif, same as KF's load_block) or the caller's encoded row.
__device__ __forceinline__ void input_row(const KStack& st, int k, int64_t g, bool valid, float (&x)[kK0]) {
#pragma unroll
  for (int f = 0; f < kK0; ++f) x[f] = 0.f;
  if (!valid) return;
  if (st.pts) {
    const float scale = st.pe_scale[k];
    float p[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) p[c] = st.pts[g * 3 + c];
    int f = 0;
    if (st.include_input) {
#pragma unroll
      for (int c = 0; c < 3; ++c) x[c] = p[c];
      f = 3;
    }
#pragma unroll
    for (int b = 0; b < 6; ++b) {
      if (b < st.n_freq) {
        const float coef = float(double(1u << b) / double(scale));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float sn, cs;
          sincospif(coef * p[c], &sn, &cs);
          const int fs = f + 6 * b + c;
          if (fs + 3 < kK0) {
            x[fs] = sn;
            x[fs + 3] = cs;
          }
        }
      }
    }
  } else {
    const float* src = st.enc + g * st.D;
#pragma unroll
    for (int f = 0; f < kK0; ++f)
      if (f < st.D) x[f] = src[f];
  }
}

template <int H, int L>
struct Smem {
  static constexpr int kDbW = (L - 1) * H + 4;               // per-warp bias-grad partials
  static constexpr int ring = kNS * kSlot;
  static constexpr int bias = ring;                          // (L-1)*H floats
  static constexpr int w3 = bias + (L - 1) * H * 4;          // 4*H
  static constexpr int b3 = w3 + 4 * H * 4;                  // 4 (+pad)
  static constexpr int out = b3 + 16;                        // 4*kTM
  static constexpr int tt = out + 4 * kTM * 4;               // kTM
  static constexpr int tr = tt + kTM * 4;                    // kTM
  static constexpr int db = tr + kTM * 4;                    // 4 warps x kDbW
  static constexpr int bars = (db + 4 * kDbW * 4 + 7) / 8 * 8;  // 3*kNS + 1 u64
  static constexpr int tmem = bars + (3 * kNS + 1) * 8;
  static constexpr int total = tmem + 16;
};

// One MMA chunk of the per-tile schedule (identical for every role).
struct Chunk {
  int sw;      // 0: interleaved K-major pair (A rows = samples), 1: 128B-swizzled transposed pair
  int kw;      // K columns staged (interleaved)
  int nks;     // k-steps of 8
  int n;       // MMA N
  int m_rows;  // rows of the swizzled A tile
  int first, last;
  int w_off;   // weight-image offset (floats) of the B half, -1: B staged by the compute warps
  int w_floats;
};

template <int H, int L, class F>
__device__ __forceinline__ void for_each_chunk(F&& f) {
  using I = Img<H, L>;
  int j = 0;
  f(j++, Chunk{0, 32, 4, H, 0, 1, 0, I::fwd_off(0), I::kC32});
  f(j++, Chunk{0, 8, 1, H, 0, 0, 1, I::fwd_off(0) + I::kC32, I::kC8});
  for (int l = 1; l <= L - 2; ++l)
    for (int c = 0; c < H / 32; ++c)
      f(j++, Chunk{0, 32, 4, H, 0, c == 0, c == H / 32 - 1, I::fwd_off(l) + c * I::kC32, I::kC32});
  for (int c = 0; c < 4; ++c) f(j++, Chunk{1, 32, 4, 16, H, c == 0, c == 3, -1, 0});
  for (int l = L - 2; l >= 0; --l) {
    for (int c = 0; c < 4; ++c) f(j++, Chunk{1, 32, 4, l == 0 ? kN0 : H, H, c == 0, c == 3, -1, 0});
    if (l > 0)
      for (int c = 0; c < H / 32; ++c)
        f(j++, Chunk{0, 32, 4, H, 0, c == 0, c == H / 32 - 1, I::dx_off(l) + c * I::kC32, I::kC32});
  }
}

constexpr int kComputeThr = 128;           // warps 0-3: staging, epilogues, render
constexpr int kTCThreads = kComputeThr + 32;  // warp 4: MMA issuer

__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

template <int H, int L>
__global__ void __launch_bounds__(kTCThreads, 1)
    tc_train_kernel(const __grid_constant__ KParams p, int si, const float* __restrict__ img_all) {
  static_assert(H * L <= 512, "TMEM columns");
  static_assert(H == 128, "M = H for the weight-gradient MMAs");
  using I = Img<H, L>;
  using SM = Smem<H, L>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const KStack& st = p.s[si];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = blockIdx.x / st.P, tile = blockIdx.x % st.P;
  const int S = st.S, G = kTM / S;
  const int r0 = tile * G, nr = min(G, st.R - r0), ns = nr * S;
  const int row = tid;  // compute warps: sample row within the tile == TMEM lane
  const int64_t gs0 = int64_t(k) * st.R * S + int64_t(r0) * S;
  const float* __restrict__ img = img_all + int64_t(k) * I::total;
  const float* __restrict__ Pk = st.params + int64_t(k) * st.block;

  float* sBias = reinterpret_cast<float*>(smem + SM::bias);
  float* sW3 = reinterpret_cast<float*>(smem + SM::w3);
  float* sB3 = reinterpret_cast<float*>(smem + SM::b3);
  float* sOut = reinterpret_cast<float*>(smem + SM::out);
  float* sT = reinterpret_cast<float*>(smem + SM::tt);
  float* sTr = reinterpret_cast<float*>(smem + SM::tr);
  float* sDb = reinterpret_cast<float*>(smem + SM::db);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::bars);
  uint64_t* empty = full + kNS;
  uint64_t* wfull = empty + kNS;
  uint64_t* accf = wfull + kNS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::tmem);

  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(&full[s], kComputeThr);
      tc::mbar_init(&empty[s], 1);
      tc::mbar_init(&wfull[s], 1);
    }
    tc::mbar_init(accf, 1);
    tc::mbar_fence_init();
  }
  for (int l = 0; l < L - 1; ++l)
    for (int i = tid; i < H; i += kTCThreads) sBias[l * H + i] = Pk[st.b_off[l] + i];
  for (int i = tid; i < 4 * H; i += kTCThreads) sW3[i] = Pk[st.w_off[L - 1] + i];
  if (tid < 4) sB3[tid] = Pk[st.b_off[L - 1] + tid];
  for (int i = tid; i < 4 * SM::kDbW; i += kTCThreads) sDb[i] = 0.f;
  if (tid < kTM) sT[row] = row < ns ? st.t[gs0 + row] : 0.f;
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = *tmem_slot;

  if (warp == 4) {
    // ------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      uint32_t wpar = 0;
      for_each_chunk<H, L>([&](int j, const Chunk& ci) {
        const int s = j % kNS;
        VM_TC_DBG(33, j);
        tc::mbar_wait(&full[s], (j / kNS) & 1);
        VM_TC_DBG(34, j);
        if (ci.w_off >= 0) {
          tc::mbar_wait(&wfull[s], (wpar >> s) & 1);
          wpar ^= 1u << s;
        }
        tc::fence_after_sync();
        const uint32_t sa = tc::smem_u32(smem + s * kSlot);
        const uint32_t idesc = tc::idesc_tf32(128, ci.n, false, false);
        if (!ci.sw) {
          const int kw = ci.kw;
          const uint32_t a_lo = sa + kTM * kw * 4, b_hi = sa + kHalfSlot, b_lo = b_hi + ci.n * kw * 4;
          for (int ks = 0; ks < ci.nks; ++ks) {
            const uint32_t o = ks * 256;
            const uint64_t ah = tc::sdesc(sa + o, 128, kw * 32), al = tc::sdesc(a_lo + o, 128, kw * 32);
            const uint64_t bh = tc::sdesc(b_hi + o, 128, kw * 32), bl = tc::sdesc(b_lo + o, 128, kw * 32);
            tc::mma_tf32(tm, al, bh, idesc, (ci.first && ks == 0) ? 0u : 1u);
            tc::mma_tf32(tm, ah, bl, idesc, 1u);
            tc::mma_tf32(tm, ah, bh, idesc, 1u);
          }
        } else {
          const uint32_t a_lo = sa + ci.m_rows * 128, b_hi = sa + kHalfSlot, b_lo = b_hi + ci.n * 128;
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t o = ks * 32;
            const uint64_t ah = sdesc_sw128(sa + o), al = sdesc_sw128(a_lo + o);
            const uint64_t bh = sdesc_sw128(b_hi + o), bl = sdesc_sw128(b_lo + o);
            tc::mma_tf32(tm, al, bh, idesc, (ci.first && ks == 0) ? 0u : 1u);
            tc::mma_tf32(tm, ah, bl, idesc, 1u);
            tc::mma_tf32(tm, ah, bh, idesc, 1u);
          }
        }
        tc::mma_commit(&empty[s]);
        if (ci.last) tc::mma_commit(accf);
        VM_TC_DBG(32, j + 1);
#ifdef VM_TC_DEBUG
        if (blockIdx.x < 64) reinterpret_cast<volatile int*>(vm_tc_dbg)[192 + blockIdx.x] = j + 1;
#endif
      });
    }
    __syncwarp();
  } else {
    // ------------------------------------------- compute warps 0-3 (128 rows)
    const uint32_t tq = tm + (uint32_t(32 * warp) << 16);  // this warp's lane quadrant
    auto R = [&](int j) { return tq + uint32_t(j * H); };  // TMEM region j (column base)
    float* myDb = sDb + warp * SM::kDbW;
    uint32_t it = 0, accn = 0;
    auto acquire = [&]() -> uint8_t* {
      const uint32_t s = it % kNS;
      VM_TC_DBG(warp * 8 + 2, int(it));
      if (it >= uint32_t(kNS)) tc::mbar_wait(&empty[s], ((it / kNS) - 1) & 1);
      VM_TC_DBG(warp * 8 + 3, int(it));
      return smem + s * kSlot;
    };
    // weight chunk: after acquiring the slot (so its previous use is complete)
    // one thread starts the TMA bulk copy of the pre-split weight chunk into
    // the slot's B half; the MMA thread waits for its bytes on wfull.
    auto acquire_w = [&](int w_off, int floats) -> uint8_t* {
      uint8_t* slot = acquire();
      if (tid == 0) {
        uint64_t* wb = &wfull[(it % kNS)];
        tc::mbar_arrive_tx(wb, uint32_t(floats * 4));
        tc::bulk_g2s(slot + kHalfSlot, img + w_off, uint32_t(floats * 4), wb);
      }
      return slot;
    };
    auto release = [&]() {  // this thread's part of the chunk is staged
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::mbar_arrive(&full[it % kNS]);
      ++it;
      VM_TC_DBG(warp * 8 + 0, int(it));
#ifdef VM_TC_DEBUG
      if (warp == 0 && lane == 0 && blockIdx.x < 64) reinterpret_cast<volatile int*>(vm_tc_dbg)[128 + blockIdx.x] = int(it);
#endif
    };
    auto wait_acc = [&]() {
      VM_TC_DBG(warp * 8 + 4, int(accn));
      tc::mbar_wait(accf, accn & 1);
      ++accn;
      VM_TC_DBG(warp * 8 + 1, int(accn));
      tc::fence_after_sync();
    };
    // A operand row (this thread's sample) -> interleaved K-major hi/lo
    auto stage_row = [&](uint8_t* slot, int kw, const float* v) {
      float* hi = reinterpret_cast<float*>(slot);
      float* lo = reinterpret_cast<float*>(slot + kTM * kw * 4);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (4 * q < kw) {
          float4 h, l;
          tc::split3(v[4 * q + 0], h.x, l.x);
          tc::split3(v[4 * q + 1], h.y, l.y);
          tc::split3(v[4 * q + 2], h.z, l.z);
          tc::split3(v[4 * q + 3], h.w, l.w);
          const uint32_t o = tc::ilv_off(row, 4 * q, kw) / 4;
          st4(hi + o, h);
          st4(lo + o, l);
        }
      }
    };
    // element (row i, sample lane) of a transposed 128B-swizzled hi/lo tile
    auto put_t = [&](uint8_t* t, int rows, int i, float v) {
      float h, l;
      tc::split3(v, h, l);
      const uint32_t o = sw128_off(i, lane);
      *reinterpret_cast<float*>(t + o) = h;
      *reinterpret_cast<float*>(t + rows * 128 + o) = l;
    };
    auto ld32 = [&](uint32_t ta, float (&v)[32]) {
      float a[16], b[16];
      tc::tmem_ld16(ta, a);
      tc::tmem_ld16(ta + 16, b);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j] = a[j];
        v[16 + j] = b[j];
      }
    };
    // warp butterfly: lane j ends with the sum over the warp's 32 rows of v[j]
    auto warp_colsum = [&](float (&v)[32]) -> float {
#pragma unroll
      for (int w = 16; w >= 1; w >>= 1) {
        const bool up = (lane & w) != 0;
#pragma unroll
        for (int j = 0; j < w; ++j) {
          const float mine = up ? v[j + w] : v[j];
          const float other = up ? v[j] : v[j + w];
          v[j] = mine + __shfl_xor_sync(0xffffffffu, other, w);
        }
      }
      return v[0];
    };

    // ----------------------------------------------------------- forward
    {
      float x0[kK0];
      input_row(st, k, gs0 + row, row < ns, x0);
      stage_row(acquire_w(I::fwd_off(0), I::kC32), 32, x0);
      release();
      stage_row(acquire_w(I::fwd_off(0) + I::kC32, I::kC8), 8, x0 + 32);
      release();
    }
    for (int l = 0; l < L - 1; ++l) {
      wait_acc();
      // X_{l+1} = relu(Z_l + b_l) -> R_{l+1}
      for (int cc = 0; cc < H; cc += 16) {
        float v[16];
        tc::tmem_ld16(R(0) + cc, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = relu_np(v[j] + sBias[l * H + cc + j]);
        tc::tmem_st16(R(l + 1) + cc, v);
      }
      tc::tmem_st_wait();
      if (l == L - 2) break;
      for (int c = 0; c < H / 32; ++c) {
        float v[32];
        ld32(R(l + 1) + 32 * c, v);
        stage_row(acquire_w(I::fwd_off(l + 1) + c * I::kC32, I::kC32), 32, v);
        release();
      }
    }
    // output layer (4 logits) on CUDA cores, sigmoid heads (models.py:341-342)
    {
      float z[4] = {0.f, 0.f, 0.f, 0.f};
      for (int cc = 0; cc < H; cc += 16) {
        float v[16];
        tc::tmem_ld16(R(L - 1) + cc, v);
#pragma unroll
        for (int j = 0; j < 16; ++j)
#pragma unroll
          for (int o = 0; o < 4; ++o) z[o] = fmaf(sW3[o * H + cc + j], v[j], z[o]);
      }
#pragma unroll
      for (int o = 0; o < 4; ++o) sOut[o * kTM + row] = sigmoid_f(z[o] + sB3[o]);
    }
    compute_sync();
    // render + L1 losses + loss grads + render backward, one thread per ray
    if (tid < nr) {
      const int r = r0 + tid, sb = tid * S;
      const int64_t rg = int64_t(k) * st.R + r;
      auto occ = [&](int i) { return sOut[sb + i]; };
      auto col = [&](int i, int c) { return sOut[(1 + c) * kTM + sb + i]; };
      auto tt = [&](int i) { return sT[sb + i]; };
      render_ray_forward(S, occ, col, tt, [&](int i, float v) { sTr[sb + i] = v; });
      const RayFwd f = render_ray_sums(S, occ, col, tt, [&](int i) { return sTr[sb + i]; });
      RayTargets tg;
      tg.depth = st.tdepth[rg];
      tg.colour[0] = st.tcol[rg * 3 + 0];
      tg.colour[1] = st.tcol[rg * 3 + 1];
      tg.colour[2] = st.tcol[rg * 3 + 2];
      tg.mask = st.tmask[rg] != 0;
      tg.valid = st.valid[rg] != 0;
      tg.ok = st.ok[rg] != 0;
      const RayLossGrad lg = ray_loss_grad(f, tg, st.wc, st.wo);
      st.ray_terms[rg * 3 + 0] = lg.l_depth;
      st.ray_terms[rg * 3 + 1] = lg.l_colour;
      st.ray_terms[rg * 3 + 2] = lg.l_occ;
      render_ray_backward(S, occ, col, tt, [&](int i) { return sTr[sb + i]; }, lg.dO, lg.dD, lg.dC,
                          [&](int i, float d_occ, const float* d_col) {
                            const float o = sOut[sb + i];
                            sOut[sb + i] = __fmul_rn(__fmul_rn(d_occ, o), __fsub_rn(1.0f, o));
#pragma unroll
                            for (int c = 0; c < 3; ++c) {
                              const float cv = sOut[(1 + c) * kTM + sb + i];
                              sOut[(1 + c) * kTM + sb + i] =
                                  __fmul_rn(__fmul_rn(d_col[c], cv), __fsub_rn(1.0f, cv));
                            }
                          });
    }
    compute_sync();
    float g3[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) g3[o] = row < ns ? sOut[o * kTM + row] : 0.f;

    float* gdst = (st.P == 1) ? st.grads + int64_t(k) * st.block
                              : st.partials + (int64_t(k) * st.P + tile) * st.block;

    // ---------------------------------------------------------- backward
    // output layer: dW3^T = X3^T G3 (MMA, M = H, N = 16), db3, and
    // G2 = (G3 W3) * (X3 > 0) written over X3 in TMEM.
    for (int c = 0; c < 4; ++c) {
      uint8_t* s = acquire();
      if (warp == c) {
        for (int cc = 0; cc < H; cc += 16) {
          float v[16], g[16];
          tc::tmem_ld16(R(L - 1) + cc, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int i = cc + j;
            put_t(s, H, i, v[j]);
            float a = 0.f;
#pragma unroll
            for (int o = 0; o < 4; ++o) a = fmaf(g3[o], sW3[o * H + i], a);
            g[j] = v[j] > 0.f ? a : 0.f;
          }
          tc::tmem_st16(R(L - 1) + cc, g);
        }
        tc::tmem_st_wait();
#pragma unroll
        for (int o = 0; o < 16; ++o) put_t(s + kHalfSlot, 16, o, o < 4 ? g3[o] : 0.f);
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          float a = g3[o];
#pragma unroll
          for (int w = 16; w >= 1; w >>= 1) a += __shfl_xor_sync(0xffffffffu, a, w);
          if (lane == 0) myDb[(L - 1) * H + o] += a;
        }
      }
      release();
    }
    wait_acc();
    {
      float v[16];
      tc::tmem_ld16(R(0), v);
      const int i = row;  // lane = fan-in index
#pragma unroll
      for (int o = 0; o < 4; ++o) gdst[st.w_off[L - 1] + o * H + i] = v[o];
    }

    for (int l = L - 2; l >= 0; --l) {
      // dW_l = G_l^T X_l, K = samples: chunk c = warp c's 32 rows
      const int nfi = (l == 0) ? kN0 : H;
      for (int c = 0; c < 4; ++c) {
        uint8_t* s = acquire();
        if (warp == c) {
          for (int cc = 0; cc < H; cc += 32) {
            float g[32];
            ld32(R(l + 1) + cc, g);
#pragma unroll
            for (int j = 0; j < 32; ++j) put_t(s, H, cc + j, g[j]);
            myDb[l * H + cc + lane] += warp_colsum(g);
          }
          if (l == 0) {
            float x0[kK0];
            input_row(st, k, gs0 + row, row < ns, x0);
#pragma unroll
            for (int i = 0; i < kN0; ++i) put_t(s + kHalfSlot, kN0, i, i < kK0 ? x0[i] : 0.f);
          } else {
            for (int cc = 0; cc < H; cc += 16) {
              float v[16];
              tc::tmem_ld16(R(l) + cc, v);
#pragma unroll
              for (int j = 0; j < 16; ++j) put_t(s + kHalfSlot, H, cc + j, v[j]);
            }
          }
        }
        release();
      }
      wait_acc();
      {  // drain dW_l (lane = fan-out row)
        const int o = row;
        const int fi_pad = (l == 0) ? st.fi0 : H;
        float* dst = gdst + st.w_off[l] + o * fi_pad;
        for (int cc = 0; cc < nfi; cc += 16) {
          float v[16];
          tc::tmem_ld16(R(0) + cc, v);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (cc + 4 * q < fi_pad)
              st4(dst + cc + 4 * q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        }
      }
      if (l == 0) break;
      // G_{l-1} = (G_l W_l) * (X_l > 0): A = G_l rows, B = W_l^T chunks (TMA)
      for (int c = 0; c < H / 32; ++c) {
        float v[32];
        ld32(R(l + 1) + 32 * c, v);
        stage_row(acquire_w(I::dx_off(l) + c * I::kC32, I::kC32), 32, v);
        release();
      }
      wait_acc();
      for (int cc = 0; cc < H; cc += 16) {
        float d[16], a[16];
        tc::tmem_ld16(R(0) + cc, d);
        tc::tmem_ld16(R(l) + cc, a);
#pragma unroll
        for (int j = 0; j < 16; ++j) d[j] = a[j] > 0.f ? d[j] : 0.f;
        tc::tmem_st16(R(l) + cc, d);
      }
      tc::tmem_st_wait();
    }
    compute_sync();
    // bias gradients: per-warp partials summed in warp order (deterministic)
    for (int i = tid; i < (L - 1) * H + 4; i += kComputeThr) {
      const float v = ((sDb[i] + sDb[SM::kDbW + i]) + sDb[2 * SM::kDbW + i]) + sDb[3 * SM::kDbW + i];
      if (i < (L - 1) * H) gdst[st.b_off[i / H] + (i % H)] = v;
      else gdst[st.b_off[L - 1] + (i - (L - 1) * H)] = v;
    }
  }

  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tm, 512);
#ifdef VM_TC_DEBUG
  if (tid == 0) atomicAdd(&vm_tc_dbg[64], 1);
#endif
  if (st.P > 1) return;
  // single-tile model: finish like KF's P == 1 path
  __threadfence_block();
  __syncthreads();
  const float* gk = st.grads + int64_t(k) * st.block;
  bool finite = true;
  for (int i = tid; i < st.block / 4; i += kTCThreads) {
    const float4 v = ld4(gk + 4 * i);
    finite &= isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
  }
  const bool all_finite = __syncthreads_and(finite);
  finalize_model(st, k, all_finite, true, reinterpret_cast<float*>(smem), kNS * kSlot / 4);
}

}  // namespace tck
}  // namespace vm
