// KT: tensor-core (tcgen05, 3xTF32) fused train step for wide per-object MLP
// fields (hidden 128, 4 layers: the reference's background model,
// trainer.py:70-71, models.py:19-55).  Same math as the FFMA kernel KF
// (models.py:311-398 forward/backward, render.py:230-333 render/losses) for
// one 128-row tile of samples (floor(128/S) whole rays) per CTA.
//
// Precision: every GEMM runs as 3xTF32 -- x = hi + lo with hi = tf32(x)
// (round to nearest) and lo = x - hi; A.B ~= lo_A.hi_B + hi_A.lo_B + hi_A.hi_B
// accumulated in fp32 in TMEM (probe: 3e-7 relative to sum|ab| for K=32;
// one-step gradients ~2e-6 relative to an f64 run), inside the north star's
// 1e-4 contract.  The 4-wide output layer, render, losses and their gradients
// run on CUDA cores in fp32 with the reference's operation order.
//
// On-chip data flow (no activation ever touches HBM):
//  * TMEM (512 columns x 128 lanes, lane = sample row): R0 = accumulator of
//    the forward pre-activations, the input-gradients (dx) and the output
//    layer's dW3; R1..R3 = activations X1..X3 (fp32).  In the backward each
//    thread keeps its row of G_l in registers, so dW_l accumulates into
//    R(l+1) (the region X_{l+1} occupied) while dx_l accumulates into R0 on a
//    second accumulator barrier: both GEMMs of a layer are issued back to
//    back and dW_l drains while dx_l runs.
//  * Shared memory: a 3-slot ring of 64 KB operand slots (A | B, each a
//    hi/lo pair).  Forward / input-gradient GEMMs stage A = activations or
//    gradients [128 samples][32 features] (core-matrix interleaved, K-major,
//    conflict-free float4 stores by the owning thread) and B = a pre-split,
//    pre-laid-out weight chunk brought in by a TMA bulk copy from an
//    L2-resident image (tc_prep_kernel builds it once per step).
//    Weight-gradient GEMMs (K = samples, one quadrant's 32 rows per chunk)
//    use MN-major SWIZZLE_128B_BASE32B tiles written as float4s by the
//    sample's thread (dW^T = X^T G for every layer; layer 0's fan-in rows
//    >= 64 are not staged since only rows < fi0 are drained).
//  * Warps 0-7 (two per TMEM lane quadrant, 64 columns each) stage, run the
//    epilogues and the render chain; warp 8 lane 0 issues the MMAs
//    (tcgen05.mma.cta_group::1.kind::tf32) from an smem schedule table and
//    commits each slot / GEMM to mbarriers, so staging of later chunks
//    overlaps the MMAs of earlier ones.
//  * Weight gradients leave through TMEM -> registers -> the CTA's partial
//    gradient block; bias gradients are warp butterfly reductions; the
//    per-model sum over tiles is reduce_partials_kernel (fixed order).
#pragma once

#include "vm_tc.cuh"

#ifdef VM_TC_DEBUG
__device__ int vm_tc_dbg[512];
#define VM_TC_DBG(i, v) \
  do { if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) reinterpret_cast<volatile int*>(vm_tc_dbg)[i] = (v); } while (0)
#else
#define VM_TC_DBG(i, v) do { } while (0)
#endif
#ifdef VM_TC_DEBUG
#define VM_TC_T(ev) \
  do { if (blockIdx.x == 0 && threadIdx.x == 0) { reinterpret_cast<volatile int*>(vm_tc_dbg)[96 + (ev)] = int(clock64() - vm_t0); } } while (0)
#else
#define VM_TC_T(ev) do { } while (0)
#endif

namespace vm {
namespace tck {

constexpr int kTM = 128;       // tile rows = TMEM lanes
constexpr int kNS = 3;         // ring slots
constexpr int kSlot = 65536;   // bytes per slot: A (32 KB) | B (32 KB)
constexpr int kHalfSlot = 32768;
constexpr int kK0 = 40;        // layer-0 fan-in padded for the MMA (33 -> 40)

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
  int c = blockIdx.x >> 2;  // 4 CTAs per chunk
  const int part = blockIdx.x & 3;
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
  const int per = H * kw / 4;
  for (int e = part * per + threadIdx.x; e < (part + 1) * per; e += blockDim.x) {
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
// 3xTF32 operand split used for staging: hi = x rounded to the nearest tf32
// (ties away, like cvt.rna, without its inf/nan guard: a non-finite value
// stays non-finite and is caught by the gradient check), lo = x - hi (exact,
// |lo| <= 2^-11 |x|); the tensor core keeps lo's top 19 bits, so the split
// error is <= 2^-22 |x|.  Two integer ALU ops + one FADD per element: the
// ALU pipe (2 cycles per warp instruction per SMSP) bounds the staging.
// Precision knobs (A/B builds): rounding lo to tf32 before the tensor core
// reads it, and a 4th product lo.lo, change the weight-gradient error by < 1%
// (measured, scripts/diag_kt_grad.py: ~3e-6 of max|g| either way) -- the
// error is dominated by the tensor core's fp32 accumulation (truncating adds,
// ~48 per 128-sample chain), not by the operand split -- so both stay off.
#ifndef VM_KT_ROUND_LO
#define VM_KT_ROUND_LO 0
#endif
#ifndef VM_KT_PRODUCTS
#define VM_KT_PRODUCTS 3
#endif
__device__ __forceinline__ void split_fast(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
  lo = __fsub_rn(x, hi);
#if VM_KT_ROUND_LO
  // lo rounded to tf32 here (the tensor core would truncate it): x = hi + lo
  // to ~2^-24 relative, so with the lo.lo product every tf32 product is exact
  lo = __uint_as_float((__float_as_uint(lo) + 0x1000u) & 0xFFFFE000u);
#endif
}

__device__ __forceinline__ uint32_t sw128_off(int row, int col) {
  return uint32_t(row * 128 + ((((col >> 2) ^ row) & 7) << 4) + (col & 3) * 4);
}

// MN-major tf32 operand tile of 32 samples (K) x 128 features (MN) in the
// SWIZZLE_128B_BASE32B layout (the only MN-major layout tf32 accepts): each
// sample's 32-feature group is one 128-B row, 32-B granules XOR-permuted by
// sample % 4; 4-sample atoms 512 B apart (SBO), 32-feature groups 4 KB apart
// (LBO).  A thread owning a sample writes its features as float4s.
constexpr int kMnLo = 16384;  // lo tile offset within a 32-KB operand half
__device__ __forceinline__ uint32_t mn_off(int s, int f) {
  return uint32_t((f >> 5) * 4096 + (s >> 2) * 512 + (s & 3) * 128 + ((((f & 31) >> 3) ^ (s & 3)) << 5) +
                  (f & 7) * 4);
}
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t saddr) {
  return tc::sdesc(saddr, 4096, 512) | (uint64_t(1) << 61);
}

// SWIZZLE_128B K-major descriptor (8-row groups 1024 B apart)
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  return tc::sdesc(saddr, 16, 1024) | (uint64_t(2) << 61);
}

// Layer-0 input row of one sample: the positional encoding of models.py:286-308
// (f32 sincospif, same as KF's load_block; per-band coefficients 2^b/scale
// precomputed in f64 -> f32 per model in smem) or the caller's encoded row.
// Every index is a compile-time constant so the row stays in registers.
__device__ __forceinline__ void input_row(const KStack& st, const float* __restrict__ coef, int64_t g, bool valid,
                                          float (&x)[kK0]) {
#pragma unroll
  for (int f = 0; f < kK0; ++f) x[f] = 0.f;
  if (!valid) return;
  if (st.pts) {
    float p[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) p[c] = st.pts[g * 3 + c];
    float e[6][6];  // [band][sin x3, cos x3]
#pragma unroll
    for (int b = 0; b < 6; ++b)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        float sn = 0.f, cs = 0.f;
        if (b < st.n_freq) sincospif(coef[b] * p[c], &sn, &cs);
        e[b][c] = sn;
        e[b][3 + c] = cs;
      }
    if (st.include_input) {
#pragma unroll
      for (int c = 0; c < 3; ++c) x[c] = p[c];
#pragma unroll
      for (int b = 0; b < 6; ++b)
#pragma unroll
        for (int j = 0; j < 6; ++j)
          if (3 + 6 * b + j < kK0) x[3 + 6 * b + j] = e[b][j];
    } else {
#pragma unroll
      for (int b = 0; b < 6; ++b)
#pragma unroll
        for (int j = 0; j < 6; ++j)
          if (6 * b + j < kK0) x[6 * b + j] = e[b][j];
    }
  } else {
    const float* src = st.enc + g * st.D;
#pragma unroll
    for (int f = 0; f < kK0; ++f) x[f] = (f < st.D) ? src[f] : 0.f;
  }
}

constexpr int kCW = 8;                        // compute warps: 2 per TMEM lane quadrant
constexpr int kComputeThr = kCW * 32;         // staging, epilogues, render
constexpr int kTCThreads = kComputeThr + 32;  // + warp 8: MMA issuer

template <int H, int L>
struct Smem {
  static constexpr int kDbW = (L - 1) * H + 4;               // per-warp bias-grad partials
  static constexpr int ring = kNS * kSlot;
  static constexpr int bias = ring;                          // (L-1)*H floats
  static constexpr int w3t = bias + (L - 1) * H * 4;         // [H][4] output weights, transposed
  static constexpr int b3 = w3t + 4 * H * 4;                 // 4 (+pad)
  static constexpr int zp = b3 + 16;                         // [2 halves][4][kTM] partial logits
  static constexpr int out = zp + 2 * 4 * kTM * 4;           // 4*kTM
  static constexpr int tt = out + 4 * kTM * 4;               // kTM
  static constexpr int tr = tt + kTM * 4;                    // kTM
  static constexpr int coef = tr + kTM * 4;                  // 8 PE coefficients
  static constexpr int tgt = coef + 8 * 4;                   // [kTM rays][8] targets (depth, rgb, flags)
  static constexpr int db = tgt + kTM * 8 * 4;               // kCW warps x kDbW
  static constexpr int bars = (db + kCW * kDbW * 4 + 7) / 8 * 8;  // 3*kNS + 2 u64
  static constexpr int tmem = bars + (3 * kNS + 2) * 8;
  static constexpr int chunks = tmem + 16;                     // schedule table (MMA warp)
  static constexpr int total = chunks + 64 * 36;
};

// One MMA chunk of the per-tile schedule (identical for every role).
struct Chunk {
  int sw;      // 0: interleaved K-major pair (A rows = samples), 1: 128B-swizzled K-major transposed
               // pair, 2: MN-major pair (SWIZZLE_128B_BASE32B, K = samples)
  int kw;      // K columns staged (interleaved)
  int nks;     // k-steps of 8
  int n;       // MMA N
  int m_rows;  // rows of the swizzled A tile
  int first, last;
  int w_off;   // weight-image offset (floats) of the B half, -1: B staged by the compute warps
  int w_floats;
  int dst = 0;  // TMEM accumulator column (KT backward: dW_l into the region G_l was read from)
  int acc = 0;  // accumulator barrier the last chunk commits to (1: KT's dx GEMMs)
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
  // output layer dW3 (N = 16) on the dx barrier: drained while dW_{L-2} runs
  for (int c = 0; c < 4; ++c) f(j++, Chunk{2, 32, 4, 16, H, c == 0, c == 3, -1, 0, 0, 1});
  // backward, per hidden layer l: dW_l (into TMEM region l+1, which held G_l)
  // then dx_l (into region 0, on its own accumulator barrier), so the two
  // GEMMs run back to back while the compute warps drain dW_l
  for (int l = L - 2; l >= 0; --l) {
    for (int c = 0; c < 4; ++c) f(j++, Chunk{2, 32, 4, H, H, c == 0, c == 3, -1, 0, (l + 1) * H, 0});
    if (l > 0)
      for (int c = 0; c < H / 32; ++c)
        f(j++, Chunk{0, 32, 4, H, 0, c == 0, c == H / 32 - 1, I::dx_off(l) + c * I::kC32, I::kC32, 0, 1});
  }
}

__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <int H, int L>
__global__ void __launch_bounds__(kTCThreads, 1)
    tc_train_kernel(const __grid_constant__ KParams p, int si, const float* __restrict__ img_all) {
  static_assert(H * L <= 512, "TMEM columns");
  static_assert(H == 128, "M = H for the weight-gradient MMAs; 2 x 64-column halves");
  constexpr int HC = H / 2;  // columns owned by one compute warp
  using I = Img<H, L>;
  using SM = Smem<H, L>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const KStack& st = p.s[si];
  const unsigned long long t_start = p.trace ? vm_gtime() : 0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = blockIdx.x / st.P, tile = blockIdx.x % st.P;
  const int S = st.S, G = kTM / S;
  const int r0 = tile * G, nr = min(G, st.R - r0), ns = nr * S;
  const int64_t gs0 = int64_t(k) * st.R * S + int64_t(r0) * S;
  const float* __restrict__ img = img_all + int64_t(k) * I::total;
  const float* __restrict__ Pk = st.params + int64_t(k) * st.block;

  float* sBias = reinterpret_cast<float*>(smem + SM::bias);
  float* sW3t = reinterpret_cast<float*>(smem + SM::w3t);
  float* sB3 = reinterpret_cast<float*>(smem + SM::b3);
  float* sZ = reinterpret_cast<float*>(smem + SM::zp);
  float* sOut = reinterpret_cast<float*>(smem + SM::out);
  float* sT = reinterpret_cast<float*>(smem + SM::tt);
  float* sTr = reinterpret_cast<float*>(smem + SM::tr);
  float* sDb = reinterpret_cast<float*>(smem + SM::db);
  float* sCoef = reinterpret_cast<float*>(smem + SM::coef);
  float* sTgt = reinterpret_cast<float*>(smem + SM::tgt);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::bars);
  uint64_t* empty = full + kNS;
  uint64_t* wfull = empty + kNS;
  uint64_t* accf = wfull + kNS;  // [2]: layer/dW accumulators, dx accumulators
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::tmem);

  if (warp == 0) tc::tmem_alloc(tmem_slot, 512);
  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(&full[s], kComputeThr);
      tc::mbar_init(&empty[s], 1);
      tc::mbar_init(&wfull[s], 1);
    }
    tc::mbar_init(&accf[0], 1);
    tc::mbar_init(&accf[1], 1);
    tc::mbar_fence_init();
  }
  for (int l = 0; l < L - 1; ++l)
    for (int i = tid; i < H; i += kTCThreads) sBias[l * H + i] = Pk[st.b_off[l] + i];
  for (int i = tid; i < 4 * H; i += kTCThreads) sW3t[(i % H) * 4 + i / H] = Pk[st.w_off[L - 1] + i];
  if (tid < 4) sB3[tid] = Pk[st.b_off[L - 1] + tid];
  for (int i = tid; i < kCW * SM::kDbW; i += kTCThreads) sDb[i] = 0.f;
  if (tid < kTM) sT[tid] = tid < ns ? st.t[gs0 + tid] : 0.f;
  if (tid < 8) sCoef[tid] = (st.pts && tid < st.n_freq) ? float(double(1u << tid) / double(st.pe_scale[k])) : 0.f;
  if (tid < nr) {  // this tile's ray targets, read once (render needs them mid-chain)
    const int64_t rg = int64_t(k) * st.R + r0 + tid;
    float* t8 = sTgt + tid * 8;
    t8[0] = st.tdepth[rg];
    t8[1] = st.tcol[rg * 3 + 0];
    t8[2] = st.tcol[rg * 3 + 1];
    t8[3] = st.tcol[rg * 3 + 2];
    t8[4] = st.tmask[rg] != 0 ? 1.f : 0.f;
    t8[5] = st.valid[rg] != 0 ? 1.f : 0.f;
    t8[6] = st.ok[rg] != 0 ? 1.f : 0.f;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = *tmem_slot;
#ifdef VM_TC_DEBUG
  const long long vm_t0 = clock64();
  int vm_ev = 0;
#endif

  if (warp == kCW) {
    // ------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      // the static schedule goes to smem once, so the issue loop below is a
      // single copy of code (instruction-cache friendly)
      Chunk* tab = reinterpret_cast<Chunk*>(smem + SM::chunks);
      int nch = 0;
      for_each_chunk<H, L>([&](int j, const Chunk& ci) { tab[j] = ci; nch = j + 1; });
      uint32_t wpar = 0;
#pragma unroll 1
      for (int j = 0; j < nch; ++j) {
        const Chunk ci = tab[j];
        const int s = j % kNS;
        tc::mbar_wait(&full[s], (j / kNS) & 1);
#ifdef VM_TC_DEBUG
        if (blockIdx.x == 0) reinterpret_cast<volatile int*>(vm_tc_dbg)[320 + j] = int(clock64() - vm_t0);
#endif
        if (ci.w_off >= 0) {
          tc::mbar_wait(&wfull[s], (wpar >> s) & 1);
          wpar ^= 1u << s;
        }
#ifdef VM_TC_DEBUG
        if (blockIdx.x == 0) reinterpret_cast<volatile int*>(vm_tc_dbg)[256 + j] = int(clock64() - vm_t0);
#endif
        tc::fence_after_sync();
        const uint32_t sa = tc::smem_u32(smem + s * kSlot);
        const uint32_t idesc = tc::idesc_tf32(128, ci.n, false, false);
        const uint32_t tmd = tm + uint32_t(ci.dst);
        if (!ci.sw) {
          const int kw = ci.kw;
          const uint32_t a_lo = sa + kTM * kw * 4, b_hi = sa + kHalfSlot, b_lo = b_hi + ci.n * kw * 4;
          for (int ks = 0; ks < ci.nks; ++ks) {
            const uint32_t o = ks * 256;
            const uint64_t ah = tc::sdesc(sa + o, 128, kw * 32), al = tc::sdesc(a_lo + o, 128, kw * 32);
            const uint64_t bh = tc::sdesc(b_hi + o, 128, kw * 32), bl = tc::sdesc(b_lo + o, 128, kw * 32);
            tc::mma_tf32(tmd, al, bh, idesc, (ci.first && ks == 0) ? 0u : 1u);
            tc::mma_tf32(tmd, ah, bl, idesc, 1u);
            tc::mma_tf32(tmd, ah, bh, idesc, 1u);
            if (VM_KT_PRODUCTS > 3) tc::mma_tf32(tmd, al, bl, idesc, 1u);
          }
        } else if (ci.sw == 2) {
          const uint32_t idesc_mn = tc::idesc_tf32(128, ci.n, true, true);
          const uint32_t a_lo = sa + kMnLo, b_hi = sa + kHalfSlot, b_lo = b_hi + kMnLo;
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t o = ks * 1024;
            const uint64_t ah = sdesc_mn(sa + o), al = sdesc_mn(a_lo + o);
            const uint64_t bh = sdesc_mn(b_hi + o), bl = sdesc_mn(b_lo + o);
            tc::mma_tf32(tmd, al, bh, idesc_mn, (ci.first && ks == 0) ? 0u : 1u);
            tc::mma_tf32(tmd, ah, bl, idesc_mn, 1u);
            tc::mma_tf32(tmd, ah, bh, idesc_mn, 1u);
            if (VM_KT_PRODUCTS > 3) tc::mma_tf32(tmd, al, bl, idesc_mn, 1u);
          }
        } else {
          const uint32_t a_lo = sa + ci.m_rows * 128, b_hi = sa + kHalfSlot, b_lo = b_hi + ci.n * 128;
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t o = ks * 32;
            const uint64_t ah = sdesc_sw128(sa + o), al = sdesc_sw128(a_lo + o);
            const uint64_t bh = sdesc_sw128(b_hi + o), bl = sdesc_sw128(b_lo + o);
            tc::mma_tf32(tmd, al, bh, idesc, (ci.first && ks == 0) ? 0u : 1u);
            tc::mma_tf32(tmd, ah, bl, idesc, 1u);
            tc::mma_tf32(tmd, ah, bh, idesc, 1u);
            if (VM_KT_PRODUCTS > 3) tc::mma_tf32(tmd, al, bl, idesc, 1u);
          }
        }
        tc::mma_commit(&empty[s]);
        if (ci.last) tc::mma_commit(&accf[ci.acc]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------- compute warps: (quadrant q, half h)
    const int q = warp & 3, h = warp >> 2;
    const int row = 32 * q + lane;                          // sample row == TMEM lane
    const int c0 = h * HC;                                  // first owned column
    const uint32_t tq = tm + (uint32_t(32 * q) << 16);      // this warp's lane quadrant
    auto R = [&](int j) { return tq + uint32_t(j * H); };   // TMEM region j (column base)
    float* myDb = sDb + warp * SM::kDbW;
    uint32_t it = 0, accn[2] = {0, 0};
    auto acquire = [&]() -> uint8_t* {
      const uint32_t s = it % kNS;
      if (it >= uint32_t(kNS)) tc::mbar_wait(&empty[s], ((it / kNS) - 1) & 1);
#ifdef VM_TC_DEBUG
      if (blockIdx.x == 0 && threadIdx.x == 0) reinterpret_cast<volatile int*>(vm_tc_dbg)[384 + it] = int(clock64() - vm_t0);
#endif
      return smem + s * kSlot;
    };
    // weight chunk: after acquiring the slot (its previous use is complete, so
    // no mbarrier phase can be skipped) the first thread of the half that
    // stages the chunk's A operand starts the TMA bulk copy of the pre-split
    // weight chunk into the slot's B half, so each half's copies are issued
    // at its own pace; the MMA thread waits for the bytes on wfull.
    auto acquire_w = [&](int w_off, int floats, int issuer_half) -> uint8_t* {
      uint8_t* slot = acquire();
      if (tid == issuer_half * 128) {
        uint64_t* wb = &wfull[it % kNS];
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
    };
    auto wait_acc = [&](int a = 0) {  // a = 1: the dx accumulator
      VM_TC_T(vm_ev);
#ifdef VM_TC_DEBUG
      ++vm_ev;
#endif
      tc::mbar_wait(&accf[a], accn[a] & 1);
      ++accn[a];
      tc::fence_after_sync();
      VM_TC_T(vm_ev);
#ifdef VM_TC_DEBUG
      ++vm_ev;
#endif
    };
    // `n4` float4 groups of this thread's row at chunk columns [col, col+4*n4)
    auto stage_row = [&](uint8_t* slot, int kw, int col, const auto& v, int n4) {
      float* hi = reinterpret_cast<float*>(slot);
      float* lo = reinterpret_cast<float*>(slot + kTM * kw * 4);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        if (g < n4) {
          float4 a, b;
          split_fast(v[4 * g + 0], a.x, b.x);
          split_fast(v[4 * g + 1], a.y, b.y);
          split_fast(v[4 * g + 2], a.z, b.z);
          split_fast(v[4 * g + 3], a.w, b.w);
          const uint32_t o = tc::ilv_off(row, col + 4 * g, kw) / 4;
          st4(hi + o, a);
          st4(lo + o, b);
        }
      }
    };
    // element (tile row i, sample lane) of a transposed 128B-swizzled hi/lo tile
    // 32 features [f0, f0+32) of this lane's sample into an MN-major hi/lo tile
    auto put_mn = [&](uint8_t* t, int f0, const float (&v)[32], int nq = 8) {  // nq float4 quads (compile-time)
#pragma unroll
      for (int m = 0; m < nq; ++m) {
        float4 a, b;
        split_fast(v[4 * m + 0], a.x, b.x);
        split_fast(v[4 * m + 1], a.y, b.y);
        split_fast(v[4 * m + 2], a.z, b.z);
        split_fast(v[4 * m + 3], a.w, b.w);
        const uint32_t o = mn_off(lane, f0 + 4 * m);
        *reinterpret_cast<float4*>(t + o) = a;
        *reinterpret_cast<float4*>(t + kMnLo + o) = b;
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
    auto ld32 = [&](uint32_t ta, float (&v)[32]) {
      uint32_t r[16];
      VM_TMEM_LD16(ta, r);
      uint32_t r2[16];
      VM_TMEM_LD16(ta + 16, r2);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j] = __uint_as_float(r[j]);
        v[16 + j] = __uint_as_float(r2[j]);
      }
    };
    // two 32-column groups with one wait (TMEM load latency paid once)
    auto ld64 = [&](uint32_t ta, uint32_t tb, float (&va)[32], float (&vb)[32]) {
      uint32_t r0[16], r1[16], r2[16], r3[16];
      VM_TMEM_LD16(ta, r0);
      VM_TMEM_LD16(ta + 16, r1);
      VM_TMEM_LD16(tb, r2);
      VM_TMEM_LD16(tb + 16, r3);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        va[j] = __uint_as_float(r0[j]);
        va[16 + j] = __uint_as_float(r1[j]);
        vb[j] = __uint_as_float(r2[j]);
        vb[16 + j] = __uint_as_float(r3[j]);
      }
    };
    auto st32 = [&](uint32_t ta, const float (&v)[32]) {
      uint32_t r[16], r2[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        r[j] = __float_as_uint(v[j]);
        r2[j] = __float_as_uint(v[16 + j]);
      }
      VM_TMEM_ST16(ta, r);
      VM_TMEM_ST16(ta + 16, r2);
    };

    // ----------------------------------------------------------- forward
    {
      float x0[kK0];
      input_row(st, sCoef, gs0 + row, row < ns, x0);
      float xa[32], xb[8];
#pragma unroll
      for (int i = 0; i < 32; ++i) xa[i] = x0[i];
#pragma unroll
      for (int i = 0; i < 8; ++i) xb[i] = x0[32 + i];
      // chunk 0 (fan-in columns 0-31) by half 0, chunk 1 (32-39) by half 1
      uint8_t* s0 = acquire_w(I::fwd_off(0), I::kC32, 0);
      if (h == 0) stage_row(s0, 32, 0, xa, 8);
      release();
      uint8_t* s1 = acquire_w(I::fwd_off(0) + I::kC32, I::kC8, 1);
      if (h == 1) stage_row(s1, 8, 0, xb, 2);
      release();
    }
#pragma unroll 1
    for (int l = 0; l < L - 1; ++l) {
      wait_acc();
      // X_{l+1} = relu(Z_l + b_l) over the owned 64 columns -> R_{l+1} and
      // registers; the next layer's chunks (32 columns each) are staged by
      // the half that owns them, the other half only releases the slot.
      float x[2][32];
      ld64(R(0) + c0, R(0) + c0 + 32, x[0], x[1]);
#pragma unroll
      for (int g = 0; g < 2; ++g) {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[g][j] = relu_np(x[g][j] + sBias[l * H + c0 + 32 * g + j]);
        st32(R(l + 1) + c0 + 32 * g, x[g]);
      }
      tc::tmem_st_wait();
      if (l == L - 2) {
        // output layer (4 logits), partial over the owned columns
        float z[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float4 w = ld4(sW3t + 4 * (c0 + 32 * g + j));
            z[0] = fmaf(w.x, x[g][j], z[0]);
            z[1] = fmaf(w.y, x[g][j], z[1]);
            z[2] = fmaf(w.z, x[g][j], z[2]);
            z[3] = fmaf(w.w, x[g][j], z[3]);
          }
#pragma unroll
        for (int o = 0; o < 4; ++o) sZ[(h * 4 + o) * kTM + row] = z[o];
        break;
      }
#pragma unroll 1
      for (int c = 0; c < H / 32; ++c) {
        uint8_t* sl = acquire_w(I::fwd_off(l + 1) + c * I::kC32, I::kC32, c >> 1);
        if ((c >> 1) == h) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = (c & 1) ? x[1][j] : x[0][j];
          stage_row(sl, 32, 0, v, 8);
        }
        release();
      }
    }
    VM_TC_T(26);
    compute_sync();
    VM_TC_T(27);
    if (h == 0) {
#pragma unroll
      for (int o = 0; o < 4; ++o)
        sOut[o * kTM + row] = sigmoid_f((sZ[o * kTM + row] + sZ[(4 + o) * kTM + row]) + sB3[o]);
    }
    compute_sync();
    VM_TC_T(28);
    // render + L1 losses + loss grads + render backward, one thread per ray,
    // rays spread over the 8 warps (4 sub-partitions)
    {
      const int rr = lane * kCW + warp;
      if (rr < nr) {
        const int r = r0 + rr, sb = rr * S;
        const int64_t rg = int64_t(k) * st.R + r;
        const float* t8 = sTgt + rr * 8;
        RayTargets tg;
        tg.depth = t8[0];
        tg.colour[0] = t8[1];
        tg.colour[1] = t8[2];
        tg.colour[2] = t8[3];
        tg.mask = t8[4] != 0.f;
        tg.valid = t8[5] != 0.f;
        tg.ok = t8[6] != 0.f;
        RayLossGrad lg;
        if (S == 10) {
          constexpr int NS = 10;
          float o[NS], cl[3][NS], tv[NS];
#pragma unroll
          for (int i = 0; i < NS; ++i) {
            o[i] = sOut[sb + i];
            tv[i] = sT[sb + i];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) cl[ch][i] = sOut[(1 + ch) * kTM + sb + i];
          }
          lg = render_ray_fixed<NS>(o, cl, tv, tg, st.wc, st.wo);
#pragma unroll
          for (int i = 0; i < NS; ++i) {
            sOut[sb + i] = o[i];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) sOut[(1 + ch) * kTM + sb + i] = cl[ch][i];
          }
        } else {
          auto occ = [&](int i) { return sOut[sb + i]; };
          auto col = [&](int i, int c) { return sOut[(1 + c) * kTM + sb + i]; };
          auto tt = [&](int i) { return sT[sb + i]; };
          render_ray_forward(S, occ, col, tt, [&](int i, float v) { sTr[sb + i] = v; });
          const RayFwd f = render_ray_sums(S, occ, col, tt, [&](int i) { return sTr[sb + i]; });
          lg = ray_loss_grad(f, tg, st.wc, st.wo);
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
        st.ray_terms[rg * 3 + 0] = lg.l_depth;
        st.ray_terms[rg * 3 + 1] = lg.l_colour;
        st.ray_terms[rg * 3 + 2] = lg.l_occ;
      }
    }
    VM_TC_T(29);
    compute_sync();
    VM_TC_T(30);
    float g3[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) g3[o] = row < ns ? sOut[o * kTM + row] : 0.f;

    float* gdst = (st.P == 1) ? st.grads + int64_t(k) * st.block
                              : st.partials + (int64_t(k) * st.P + tile) * st.block;

    // ---------------------------------------------------------- backward
    // output layer: dW3^T = X3^T G3 (MMA, M = H, N = 16), db3, and
    // G2 = (G3 W3) * (X3 > 0) kept in registers (owned columns).  G_l rows
    // stay in registers from here on: each dx epilogue produces the next
    // (dW_{l-1} accumulates over TMEM region l, so nothing is stored back).
    float gv[2][32];
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint8_t* sl = acquire();
      if (q == c) {
        float xv[2][32];
        ld64(R(L - 1) + c0, R(L - 1) + c0 + 32, xv[0], xv[1]);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float (&v)[32] = xv[g];
          put_mn(sl, c0 + 32 * g, v);  // A = X3 (M = fan-in)
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float4 w = ld4(sW3t + 4 * (c0 + 32 * g + j));
            const float a = fmaf(g3[3], w.w, fmaf(g3[2], w.z, fmaf(g3[1], w.y, g3[0] * w.x)));
            gv[g][j] = v[j] > 0.f ? a : 0.f;
          }
        }
        if (h == 0) {
          float gb[32];
#pragma unroll
          for (int o = 0; o < 32; ++o) gb[o] = o < 4 ? g3[o < 4 ? o : 0] : 0.f;
          put_mn(sl + kHalfSlot, 0, gb, 4);  // B = G3: the MMA reads N = 16 columns (4 live)
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            float a = g3[o];
#pragma unroll
            for (int w = 16; w >= 1; w >>= 1) a += __shfl_xor_sync(0xffffffffu, a, w);
            if (lane == 0) myDb[(L - 1) * H + o] += a;
          }
        }
      }
      release();
    }

#pragma unroll 1
    for (int l = L - 2; l >= 0; --l) {
      // dW_l = G_l^T X_l, K = samples: chunk c = quadrant c's 32 rows, each
      // half stages its 64 features of both operands.  Every layer computes
      // dW_l^T = X_l^T G_l from MN-major tiles (A = X_l, B = G_l, each thread
      // writes its own sample's features as float4s), so TMEM lane = fan-in
      // and the drain writes whole 128-B rows of the gradient (layer 0: the
      // rows i < fi0 only).
      // Every thread holds its G_l row (owned columns) in registers before
      // its first release: dW_l accumulates into TMEM region l+1, and the row
      // feeds the dx_l operand and the bias gradient.
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint8_t* sl = acquire();
        if (q == c) {
          uint8_t* gt = sl + kHalfSlot;  // B = G_l (N = fan-out)
          uint8_t* xt = sl;              // A = X_l (M = fan-in; layer 0: rows >= 64 not staged)
          put_mn(gt, c0, gv[0]);
          put_mn(gt, c0 + 32, gv[1]);
          if (l == 0) {
            // last weight-gradient GEMM of the tile: let the partial-reduce
            // grid (launched programmatically behind this one) be scheduled
            // now; it waits on griddepcontrol.wait for this grid's completion
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
            // layer-0 input recomputed (positional encoding) by the half
            // owning features 0..63.  A rows (fan-in) 64..127 are left as
            // they are: row i of dW0^T depends only on A row i, and the drain
            // stores rows i < fi0 (<= 40) only
            if (h == 0) {
              float xa[32], xb[32];
              float x0[kK0];
              input_row(st, sCoef, gs0 + row, row < ns, x0);
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                xa[i] = x0[i];
                xb[i] = (32 + i < kK0) ? x0[32 + i < kK0 ? 32 + i : 0] : 0.f;
              }
              put_mn(xt, c0, xa);
              put_mn(xt, c0 + 32, xb);
            }
          } else {
            float xv[2][32];
            ld64(R(l) + c0, R(l) + c0 + 32, xv[0], xv[1]);
            put_mn(xt, c0, xv[0]);
            put_mn(xt, c0 + 32, xv[1]);
          }
        }
        release();
      }
      if (l == L - 2) {  // dW3^T (region 0, dx barrier): drained before dx_l reuses region 0
        wait_acc(1);
        if (h == 0) {
          float v[16];
          tc::tmem_ld16(R(0), v);
          const int i = row;  // lane = fan-in index
#pragma unroll
          for (int o = 0; o < 4; ++o) gdst[st.w_off[L - 1] + o * H + i] = v[o];
        }
      }
      // G_{l-1} = (G_l W_l) * (X_l > 0): A = G_l rows (chunk c by the half
      // owning those columns), B = W_l^T chunks (TMA); issued right behind
      // dW_l, into region 0 on the dx barrier
      if (l > 0) {
#pragma unroll 1
        for (int c = 0; c < H / 32; ++c) {
          uint8_t* sl = acquire_w(I::dx_off(l) + c * I::kC32, I::kC32, c >> 1);
          if ((c >> 1) == h) {
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = (c & 1) ? gv[1][j] : gv[0][j];
            stage_row(sl, 32, 0, v, 8);
          }
          release();
        }
      }
      // bias gradient db_l: column sums of G_l over the warp's 32 rows (while
      // the tensor core runs dW_l / dx_l)
#pragma unroll
      for (int g = 0; g < 2; ++g) myDb[l * H + c0 + 32 * g + lane] += warp_colsum(gv[g]);
      wait_acc();
      {  // drain dW_l^T from region l+1: lane = fan-in i, columns = this half's fan-out rows
        const int i = row;
        const int fi_pad = (l == 0) ? st.fi0 : H;  // layer 0: fan-in rows >= 36 do not exist
        float* dst = gdst + st.w_off[l] + i;
#pragma unroll
        for (int cc = 0; cc < HC; cc += 16) {
          float v[16];
          tc::tmem_ld16(R(l + 1) + c0 + cc, v);  // warp-wide (.sync.aligned): no divergence before it
          if (i < fi_pad) {
#pragma unroll
            for (int j = 0; j < 16; ++j) dst[(c0 + cc + j) * fi_pad] = v[j];
          }
        }
      }
      if (l == 0) break;
      wait_acc(1);
      // G_{l-1} = dx * (X_l > 0), kept in registers for the next layer
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        float a[32];
        ld64(R(0) + c0 + 32 * g, R(l) + c0 + 32 * g, gv[g], a);
#pragma unroll
        for (int j = 0; j < 32; ++j) gv[g][j] = a[j] > 0.f ? gv[g][j] : 0.f;
      }
    }
    compute_sync();
    VM_TC_T(vm_ev);
    // bias gradients: per-warp partials summed in warp order (deterministic)
    for (int i = tid; i < (L - 1) * H + 4; i += kComputeThr) {
      float v = sDb[i];
#pragma unroll
      for (int w = 1; w < kCW; ++w) v += sDb[w * SM::kDbW + i];
      if (i < (L - 1) * H) gdst[st.b_off[i / H] + (i % H)] = v;
      else gdst[st.b_off[L - 1] + (i - (L - 1) * H)] = v;
    }
  }

  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tm, 512);
  if (p.trace && tid == 0) vm_trace_rec(p.trace, 2, t_start);
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

// ---------------------------------------------------------------------------
// KT forward only (inference: occupancy grids, view rays; meshing.py:64-97,
// :453-579): the same 3xTF32 tcgen05 layer GEMMs as KT's forward, as a
// persistent kernel looping over groups of NT 128-sample tiles (blockIdx.y =
// model).  No activation is kept for a backward pass, so each tile in flight
// needs one TMEM accumulator (128 columns).  With NT = 2 the chunk stream
// interleaves the two tiles layer by layer (L0 t0, L0 t1, L1 t0, L1 t1, ...),
// so the tensor core runs one tile's GEMM while the compute warps drain and
// stage the other's; every role walks the same order, group after group, with
// the ring and accumulator phases running on.
template <int H, int L, int NT>
struct FwdSmem {
  static constexpr int ring = kNS * kSlot;
  static constexpr int bias = ring;                      // (L-1)*H floats
  static constexpr int w3t = bias + (L - 1) * H * 4;     // [H][4]
  static constexpr int b3 = w3t + 4 * H * 4;             // 4 (+pad)
  static constexpr int zp = b3 + 16;                     // [NT][2 halves][4][kTM]
  static constexpr int bars = (zp + NT * 2 * 4 * kTM * 4 + 7) / 8 * 8;
  static constexpr int tmem = bars + (3 * kNS + NT) * 8;
  static constexpr int total = tmem + 16;
};

// chunk c of layer li of the forward schedule (layer 0: 2 chunks, K = 32 + 8)
template <int H, int L>
__device__ __forceinline__ Chunk fwd_chunk(int li, int c) {
  using I = Img<H, L>;
  if (li == 0) return c == 0 ? Chunk{0, 32, 4, H, 0, 1, 0, I::fwd_off(0), I::kC32}
                             : Chunk{0, 8, 1, H, 0, 0, 1, I::fwd_off(0) + I::kC32, I::kC8};
  return Chunk{0, 32, 4, H, 0, c == 0, c == H / 32 - 1, I::fwd_off(li) + c * I::kC32, I::kC32};
}

template <int H, int L, int NT>
__global__ void __launch_bounds__(kTCThreads, 1)
    tc_forward_kernel(const __grid_constant__ KStack st, const float* __restrict__ img_all, int64_t n,
                      float* __restrict__ occ, float* __restrict__ col) {
  static_assert(H == 128, "two 64-column halves per TMEM lane quadrant");
  static_assert(NT == 1 || NT == 2, "tiles in flight");
  constexpr int HC = H / 2;
  using I = Img<H, L>;
  using SM = FwdSmem<H, L, NT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = blockIdx.y;
  const int64_t n_groups = (n + int64_t(kTM) * NT - 1) / (int64_t(kTM) * NT);
  const float* __restrict__ img = img_all + int64_t(k) * I::total;
  const float* __restrict__ Pk = st.params + int64_t(k) * st.block;

  float* sBias = reinterpret_cast<float*>(smem + SM::bias);
  float* sW3t = reinterpret_cast<float*>(smem + SM::w3t);
  float* sB3 = reinterpret_cast<float*>(smem + SM::b3);
  float* sZ = reinterpret_cast<float*>(smem + SM::zp);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::bars);
  uint64_t* empty = full + kNS;
  uint64_t* wfull = empty + kNS;
  uint64_t* accf = wfull + kNS;  // [NT]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SM::tmem);

  if (warp == 0) tc::tmem_alloc(tmem_slot, 128 * NT);
  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(&full[s], kComputeThr);
      tc::mbar_init(&empty[s], 1);
      tc::mbar_init(&wfull[s], 1);
    }
    for (int t = 0; t < NT; ++t) tc::mbar_init(&accf[t], 1);
    tc::mbar_fence_init();
  }
  for (int l = 0; l < L - 1; ++l)
    for (int i = tid; i < H; i += kTCThreads) sBias[l * H + i] = Pk[st.b_off[l] + i];
  for (int i = tid; i < 4 * H; i += kTCThreads) sW3t[(i % H) * 4 + i / H] = Pk[st.w_off[L - 1] + i];
  if (tid < 4) sB3[tid] = Pk[st.b_off[L - 1] + tid];
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = *tmem_slot;

  if (warp == kCW) {
    // ------------------------------------------------ MMA issuer (one thread)
    if (lane == 0) {
      uint32_t wpar = 0, j = 0;
      for (int64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
#pragma unroll 1
        for (int li = 0; li < L - 1; ++li)
#pragma unroll 1
          for (int t = 0; t < NT; ++t) {
            const uint32_t d = tm + uint32_t(t * 128);
            const int nc = li == 0 ? 2 : H / 32;
#pragma unroll 1
            for (int c = 0; c < nc; ++c) {
              const Chunk ci = fwd_chunk<H, L>(li, c);
              const uint32_t s = j % kNS;
              tc::mbar_wait(&full[s], (j / kNS) & 1);
              tc::mbar_wait(&wfull[s], (wpar >> s) & 1);
              wpar ^= 1u << s;
              tc::fence_after_sync();
              const uint32_t sa = tc::smem_u32(smem + s * kSlot);
              const uint32_t idesc = tc::idesc_tf32(128, ci.n, false, false);
              const int kw = ci.kw;
              const uint32_t a_lo = sa + kTM * kw * 4, b_hi = sa + kHalfSlot, b_lo = b_hi + ci.n * kw * 4;
              for (int ks = 0; ks < ci.nks; ++ks) {
                const uint32_t o = ks * 256;
                const uint64_t ah = tc::sdesc(sa + o, 128, kw * 32), al = tc::sdesc(a_lo + o, 128, kw * 32);
                const uint64_t bh = tc::sdesc(b_hi + o, 128, kw * 32), bl = tc::sdesc(b_lo + o, 128, kw * 32);
                tc::mma_tf32(d, al, bh, idesc, (ci.first && ks == 0) ? 0u : 1u);
                tc::mma_tf32(d, ah, bl, idesc, 1u);
                tc::mma_tf32(d, ah, bh, idesc, 1u);
              }
              tc::mma_commit(&empty[s]);
              if (ci.last) tc::mma_commit(&accf[t]);
              ++j;
            }
          }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------- compute warps: (quadrant q, half h)
    const int q = warp & 3, h = warp >> 2;
    const int row = 32 * q + lane;
    const int c0 = h * HC;
    const uint32_t tq = tm + (uint32_t(32 * q) << 16);
    uint32_t it = 0, accn[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) accn[t] = 0;
    auto acquire_w = [&](int w_off, int floats, int issuer_half) -> uint8_t* {
      const uint32_t s = it % kNS;
      if (it >= uint32_t(kNS)) tc::mbar_wait(&empty[s], ((it / kNS) - 1) & 1);
      uint8_t* slot = smem + s * kSlot;
      if (tid == issuer_half * 128) {
        tc::mbar_arrive_tx(&wfull[s], uint32_t(floats * 4));
        tc::bulk_g2s(slot + kHalfSlot, img + w_off, uint32_t(floats * 4), &wfull[s]);
      }
      return slot;
    };
    auto release = [&]() {
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::mbar_arrive(&full[it % kNS]);
      ++it;
    };
    auto stage_row = [&](uint8_t* slot, int kw, const auto& v, int n4) {
      float* hi = reinterpret_cast<float*>(slot);
      float* lo = reinterpret_cast<float*>(slot + kTM * kw * 4);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        if (g < n4) {
          float4 a, b;
          split_fast(v[4 * g + 0], a.x, b.x);
          split_fast(v[4 * g + 1], a.y, b.y);
          split_fast(v[4 * g + 2], a.z, b.z);
          split_fast(v[4 * g + 3], a.w, b.w);
          const uint32_t o = tc::ilv_off(row, 4 * g, kw) / 4;
          st4(hi + o, a);
          st4(lo + o, b);
        }
      }
    };
    auto ld64 = [&](uint32_t ta, uint32_t tb, float (&va)[32], float (&vb)[32]) {
      uint32_t r0[16], r1[16], r2[16], r3[16];
      VM_TMEM_LD16(ta, r0);
      VM_TMEM_LD16(ta + 16, r1);
      VM_TMEM_LD16(tb, r2);
      VM_TMEM_LD16(tb + 16, r3);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        va[jj] = __uint_as_float(r0[jj]);
        va[16 + jj] = __uint_as_float(r1[jj]);
        vb[jj] = __uint_as_float(r2[jj]);
        vb[16 + jj] = __uint_as_float(r3[jj]);
      }
    };
    for (int64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
      // layer-0 operands of every tile of the group
#pragma unroll 1
      for (int t = 0; t < NT; ++t) {
        const int64_t g = (grp * NT + t) * kTM + row;
        float x0[kK0];
        input_row(st, nullptr, int64_t(k) * n + g, g < n, x0);
        float xa[32], xb[8];
#pragma unroll
        for (int i = 0; i < 32; ++i) xa[i] = x0[i];
#pragma unroll
        for (int i = 0; i < 8; ++i) xb[i] = x0[32 + i];
        uint8_t* s0 = acquire_w(I::fwd_off(0), I::kC32, 0);
        if (h == 0) stage_row(s0, 32, xa, 8);
        release();
        uint8_t* s1 = acquire_w(I::fwd_off(0) + I::kC32, I::kC8, 1);
        if (h == 1) stage_row(s1, 8, xb, 2);
        release();
      }
#pragma unroll 1
      for (int l = 0; l < L - 1; ++l) {
#pragma unroll 1
        for (int t = 0; t < NT; ++t) {
          tc::mbar_wait(&accf[t], accn[t] & 1);
          ++accn[t];
          tc::fence_after_sync();
          float x[2][32];
          ld64(tq + uint32_t(t * 128) + c0, tq + uint32_t(t * 128) + c0 + 32, x[0], x[1]);
#pragma unroll
          for (int gg = 0; gg < 2; ++gg)
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) x[gg][jj] = relu_np(x[gg][jj] + sBias[l * H + c0 + 32 * gg + jj]);
          if (l == L - 2) {  // output layer (4 logits), partial over the owned columns
            float z[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int gg = 0; gg < 2; ++gg)
#pragma unroll
              for (int jj = 0; jj < 32; ++jj) {
                const float4 w = ld4(sW3t + 4 * (c0 + 32 * gg + jj));
                z[0] = fmaf(w.x, x[gg][jj], z[0]);
                z[1] = fmaf(w.y, x[gg][jj], z[1]);
                z[2] = fmaf(w.z, x[gg][jj], z[2]);
                z[3] = fmaf(w.w, x[gg][jj], z[3]);
              }
#pragma unroll
            for (int o = 0; o < 4; ++o) sZ[((t * 2 + h) * 4 + o) * kTM + row] = z[o];
            continue;
          }
#pragma unroll 1
          for (int c = 0; c < H / 32; ++c) {
            uint8_t* sl = acquire_w(I::fwd_off(l + 1) + c * I::kC32, I::kC32, c >> 1);
            if ((c >> 1) == h) {
              float v[32];
#pragma unroll
              for (int jj = 0; jj < 32; ++jj) v[jj] = (c & 1) ? x[1][jj] : x[0][jj];
              stage_row(sl, 32, v, 8);
            }
            release();
          }
        }
      }
      compute_sync();
      if (h == 0) {
#pragma unroll 1
        for (int t = 0; t < NT; ++t) {
          const int64_t g = (grp * NT + t) * kTM + row;
          if (g < n) {
            const int64_t gk = int64_t(k) * n + g;
            const float* z0 = sZ + (t * 2 + 0) * 4 * kTM;
            const float* z1 = sZ + (t * 2 + 1) * 4 * kTM;
            occ[gk] = sigmoid_f((z0[row] + z1[row]) + sB3[0]);
#pragma unroll
            for (int o = 1; o < 4; ++o)
              col[gk * 3 + o - 1] = sigmoid_f((z0[o * kTM + row] + z1[o * kTM + row]) + sB3[o]);
          }
        }
      }
      compute_sync();  // sZ is rewritten by the next group
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free(tm, 128 * NT);
}

}  // namespace tck
}  // namespace vm
