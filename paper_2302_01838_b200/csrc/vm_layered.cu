// Layered train step / evaluation for the architectures the fused kernels
// (KF32, KT, the generic FFMA kernel) do not cover: hidden widths above 128
// (the paper's Fig. 6 sweeps up to 1024), encodings wider
// than 40, layer counts or stack pairs without a fused instantiation, more
// than 32 samples per ray.  The reference accepts all of these
// (models.py:19-55 puts no bound on the widths).
//
// The same math as the fused path, one layer at a time over the stacked
// arena (one model = one batch entry of every launch):
//   forward   z_l = x_l W_l^T + b_l, ReLU          models.py:311-355
//   per ray   sigmoid heads, render, L1 losses, loss grads, render backward,
//             sigmoid'                             render.py:230-333 (bit-exact chain given z)
//   backward  [dW_l^T ; db_l] = [x_l | 1]^T dz_l    models.py:358-398
//             dz_{l-1} = (dz_l W_l) * (x_l > 0)
//   Adam      models.py:401-467 (vm_adam.cuh op order, the fused path's skip rules)
// The GEMMs are one batched SIMT FP32 kernel (128-row tiles, 8x8 or 4x4
// register blocks per thread, double-buffered smem, explicit FFMA).  The
// weight-gradient GEMM reduces over samples split into a fixed number of
// chunks that depends only on the model's own sample count and layer shape,
// summed in chunk order: vectorised == sequential stays bit-exact.
#include "vm_mlp.cuh"

#include <algorithm>

namespace vm {
namespace lyr {

constexpr int kBK = 8;     // k-depth of a smem stage
constexpr int kGT = 256;   // threads per GEMM CTA
constexpr int kMaxS = 64;  // samples per ray of the per-ray kernel
constexpr int kSent = 0x7f7f7f7f;

enum Epi : int { kEpiBias = 0, kEpiBiasRelu = 1, kEpiMask = 2, kEpiStore = 3, kEpiHeads = 4 };

// C[M x N] = sum_{k < Kd} A(m, k) B(k, n) per batch entry (blockIdx.z).
struct Gemm {
  int M, N, Kd;
  const float* A;     // AK: A(m,k) = A[m*lda + k]; else A[k*lda + m]
  int64_t lda, sA;
  int a_valid;        // rows m >= a_valid read as 0 ...
  int a_ones;         // ... except row a_ones, which reads as 1 (the bias row of dW); -1: none
  const float* B;     // BKc: B(k,n) = B[n*ldb + k]; else B[k*ldb + n]
  int64_t ldb, sB;
  float* C;
  int64_t ldc, sC, sCsplit;
  const float* bias;  // kEpiBias/kEpiBiasRelu/kEpiHeads: + bias[n]
  int64_t sBias;
  const float* mask;  // kEpiMask: C *= (mask[m*ldm + n] > 0)
  int64_t ldm, sM;
  float* occ;         // kEpiHeads: occ[m] = sigmoid(z0), col[m*3 + c] = sigmoid(z_{1+c})
  float* col;
  int64_t sO;
  int splits, kchunk; // blockIdx.z = batch * splits + split; split s reduces k in [s*kchunk, (s+1)*kchunk)
  int db_row;         // kEpiStore, >= 0: the m0 == 0 CTAs also store the column sums of B (sum_k B(k, n),
                      // the bias gradient) as element db_row of C^T's row n, accumulated in the same k order
                      // (kEpiStore writes C transposed: C^T[n*ldc + m], ldc % 4 == 0)
};

template <int BM, int BN, int TM, int TN, bool AK, bool BKc, int EPI>
__global__ void __launch_bounds__(kGT, 2) gemm_kernel(const __grid_constant__ Gemm g) {
  static_assert((BM / TM) * (BN / TN) == kGT, "one register block per thread");
  constexpr int EA = BM * kBK / kGT, EB = BN * kBK / kGT;
  __shared__ __align__(16) float As[2][kBK][BM];
  __shared__ __align__(16) float Bs[2][kBK][BN];
  const int batch = blockIdx.z / g.splits, split = blockIdx.z % g.splits;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const float* __restrict__ A = g.A + batch * g.sA;
  const float* __restrict__ B = g.B + batch * g.sB;
  const int k_begin = split * g.kchunk;
  const int k_end = min(g.Kd, k_begin + g.kchunk);
  const int tid = threadIdx.x;
  float ra[EA], rb[EB];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < EA; ++e) {
      const int L = tid * EA + e;
      const int m = AK ? L / kBK : L % BM, k = AK ? L % kBK : L / BM;
      const int gm = m0 + m, gk = k0 + k;
      float v = 0.f;
      if (gk < k_end) {
        if (gm == g.a_ones) v = 1.f;
        else if (gm < g.a_valid) v = AK ? __ldg(A + int64_t(gm) * g.lda + gk) : __ldg(A + int64_t(gk) * g.lda + gm);
      }
      ra[e] = v;
    }
#pragma unroll
    for (int e = 0; e < EB; ++e) {
      const int L = tid * EB + e;
      const int n = BKc ? L / kBK : L % BN, k = BKc ? L % kBK : L / BN;
      const int gn = n0 + n, gk = k0 + k;
      rb[e] = (gk < k_end && gn < g.N) ? (BKc ? __ldg(B + int64_t(gn) * g.ldb + gk) : __ldg(B + int64_t(gk) * g.ldb + gn))
                                       : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < EA; ++e) {
      const int L = tid * EA + e;
      As[buf][AK ? L % kBK : L / BM][AK ? L / kBK : L % BM] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < EB; ++e) {
      const int L = tid * EB + e;
      Bs[buf][BKc ? L % kBK : L / BN][BKc ? L / kBK : L % BN] = rb[e];
    }
  };
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  // an 8-wide register block is two 4-wide halves BM/2 (BN/2) apart, so a
  // warp's LDS.128 fragment reads cover contiguous 16-B chunks (a contiguous
  // 8-float block per thread would put every fourth thread on the same banks)
  auto row = [&](int i) { return TM == 8 ? (i & 4 ? BM / 2 : 0) + ty * 4 + (i & 3) : ty * TM + i; };
  auto colx = [&](int j) { return TN == 8 ? (j & 4 ? BN / 2 : 0) + tx * 4 + (j & 3) : tx * TN + j; };
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
  // bias gradient: column sums of B, by the threads of register-block row 0
  // of the first M tile (each column has exactly one such thread)
  const bool dbt = EPI == kEpiStore && g.db_row >= 0 && blockIdx.y == 0 && ty == 0;
  float dbacc[TN];
#pragma unroll
  for (int j = 0; j < TN; ++j) dbacc[j] = 0.f;
  int buf = 0;
  if (k_begin < k_end) {
    load(k_begin);
    store(0);
  }
  __syncthreads();
  for (int k0 = k_begin; k0 < k_end; k0 += kBK) {
    const bool more = k0 + kBK < k_end;
    if (more) load(k0 + kBK);
    // fragments of step kk+1 are read from smem while step kk's FFMAs issue
    float a[2][TM], b[2][TN];
    auto frag = [&](int kk, int f) {
#pragma unroll
      for (int i = 0; i < TM; i += 4) {
        const float4 v = *reinterpret_cast<const float4*>(&As[buf][kk][row(i)]);
        a[f][i] = v.x, a[f][i + 1] = v.y, a[f][i + 2] = v.z, a[f][i + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < TN; j += 4) {
        const float4 v = *reinterpret_cast<const float4*>(&Bs[buf][kk][colx(j)]);
        b[f][j] = v.x, b[f][j + 1] = v.y, b[f][j + 2] = v.z, b[f][j + 3] = v.w;
      }
    };
    frag(0, 0);
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      if (kk + 1 < kBK) frag(kk + 1, (kk + 1) & 1);
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = __fmaf_rn(a[kk & 1][i], b[kk & 1][j], acc[i][j]);
      if constexpr (EPI == kEpiStore) {
        if (dbt) {
#pragma unroll
          for (int j = 0; j < TN; ++j) dbacc[j] = __fadd_rn(dbacc[j], b[kk & 1][j]);
        }
      }
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  // epilogue
  if constexpr (EPI == kEpiStore) {
    // weight-gradient partials as C^T (output-major, the arena's dW row
    // order): four consecutive m of one n per float4
    float* C = g.C + batch * g.sC + split * g.sCsplit;
#pragma unroll
    for (int i = 0; i < TM; i += 4) {
      const int m = m0 + row(i);
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int n = n0 + colx(j);
        if (n >= g.N) continue;
        if (m + 3 < g.M) {
          st4(C + int64_t(n) * g.ldc + m, make_float4(acc[i][j], acc[i + 1][j], acc[i + 2][j], acc[i + 3][j]));
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (m + u < g.M) C[int64_t(n) * g.ldc + m + u] = acc[i + u][j];
        }
      }
    }
  }
  if (dbt) {
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + colx(j);
      if (n < g.N) g.C[batch * g.sC + split * g.sCsplit + int64_t(n) * g.ldc + g.db_row] = dbacc[j];
    }
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    if constexpr (EPI == kEpiStore) break;
    const int m = m0 + row(i);
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + colx(j);
      if (n >= g.N) continue;
      float v = acc[i][j];
      if constexpr (EPI == kEpiBias || EPI == kEpiBiasRelu || EPI == kEpiHeads) {
        v = __fadd_rn(v, g.bias[batch * g.sBias + n]);  // z += b (models.py:336)
        if constexpr (EPI == kEpiBiasRelu) v = np_maximum(v, 0.f);
      }
      if constexpr (EPI == kEpiMask) v = __fmul_rn(v, g.mask[batch * g.sM + int64_t(m) * g.ldm + n] > 0.f ? 1.f : 0.f);
      if constexpr (EPI == kEpiHeads) {
        const float sg = sigmoid_f(v);
        const int64_t row = batch * g.sO + m;
        if (n == 0) g.occ[row] = sg;
        else g.col[row * 3 + (n - 1)] = sg;
      } else {
        g.C[batch * g.sC + split * g.sCsplit + int64_t(m) * g.ldc + n] = v;
      }
    }
  }
}

template <int EPI, bool AK, bool BKc>
int launch_gemm(const Gemm& g, int batches, cudaStream_t s) {
  if (batches == 0 || g.M == 0 || g.N == 0) return VM_OK;
  VM_REQUIRE(int64_t(batches) * g.splits <= 65535, "layered: too many models x sample chunks for one launch");
  if (g.N <= 32) {
    const dim3 grid((g.N + 31) / 32, (g.M + 127) / 128, batches * g.splits);
    VM_REQUIRE(grid.y <= 65535, "layered: too many rows for one launch");
    gemm_kernel<128, 32, 4, 4, AK, BKc, EPI><<<grid, kGT, 0, s>>>(g);
  } else {
    const dim3 grid((g.N + 127) / 128, (g.M + 127) / 128, batches * g.splits);
    VM_REQUIRE(grid.y <= 65535, "layered: too many rows for one launch");
    gemm_kernel<128, 128, 8, 8, AK, BKc, EPI><<<grid, kGT, 0, s>>>(g);
  }
  VM_CUDA(cudaGetLastError());
  return VM_OK;
}

// ---------------------------------------------------------------- per ray
struct RayArgs {
  int K, R, S;
  const float* z;      // [K][R*S][4] output-layer pre-activations
  const float* t;      // [K][R][S]
  const float* tdepth; // [K][R]
  const float* tcol;   // [K][R][3]
  const uint8_t* tmask;
  const uint8_t* valid;
  const uint8_t* ok;
  float wc, wo;
  float* dz;     // [K][R*S][4] sigmoid-input gradients
  float* terms;  // [K][R][3] per-ray loss terms
};

// sigmoid heads (models.py:353-354), render_rays (render.py:230-246),
// compute_losses' per-ray terms + loss_output_grads (render.py:284-333),
// render_backward (render.py:249-281), and the sigmoid derivative of
// models.py:372-373: the fused kernels' per-ray chain, op for op.
__global__ void __launch_bounds__(128) ray_kernel(const __grid_constant__ RayArgs a) {
  const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (idx >= int64_t(a.K) * a.R) return;
  const int S = a.S;
  const float* z = a.z + idx * S * 4;
  float o[kMaxS], c[kMaxS][3], tt[kMaxS], tr[kMaxS];
  for (int i = 0; i < S; ++i) {
    o[i] = sigmoid_f(z[i * 4]);
    for (int ch = 0; ch < 3; ++ch) c[i][ch] = sigmoid_f(z[i * 4 + 1 + ch]);
    tt[i] = a.t[idx * S + i];
  }
  auto occ = [&](int i) { return o[i]; };
  auto col = [&](int i, int ch) { return c[i][ch]; };
  auto tv = [&](int i) { return tt[i]; };
  auto trv = [&](int i) { return tr[i]; };
  render_ray_forward(S, occ, col, tv, [&](int i, float v) { tr[i] = v; });
  const RayFwd f = render_ray_sums(S, occ, col, tv, trv);
  RayTargets tg;
  tg.depth = a.tdepth[idx];
  for (int ch = 0; ch < 3; ++ch) tg.colour[ch] = a.tcol[idx * 3 + ch];
  tg.mask = a.tmask[idx] != 0;
  tg.valid = a.valid[idx] != 0;
  tg.ok = a.ok[idx] != 0;
  const RayLossGrad lgr = ray_loss_grad(f, tg, a.wc, a.wo);
  a.terms[idx * 3 + 0] = lgr.l_depth;
  a.terms[idx * 3 + 1] = lgr.l_colour;
  a.terms[idx * 3 + 2] = lgr.l_occ;
  float* dz = a.dz + idx * S * 4;
  render_ray_backward(S, occ, col, tv, trv, lgr.dO, lgr.dD, lgr.dC, [&](int i, float d_occ, const float* d_col) {
    dz[i * 4] = __fmul_rn(__fmul_rn(d_occ, o[i]), __fsub_rn(1.0f, o[i]));
    for (int ch = 0; ch < 3; ++ch)
      dz[i * 4 + 1 + ch] = __fmul_rn(__fmul_rn(d_col[ch], c[i][ch]), __fsub_rn(1.0f, c[i][ch]));
  });
}

// Standalone backward (vm_backward): sigmoid-input gradients from given output
// gradients, dz = g * s * (1 - s) (models.py:372-373).
__global__ void heads_grad_kernel(int64_t n, const float* __restrict__ z, const float* __restrict__ gocc,
                                  const float* __restrict__ gcol, float* __restrict__ dz) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const float so = sigmoid_f(z[i * 4]);
  dz[i * 4] = __fmul_rn(__fmul_rn(gocc[i], so), __fsub_rn(1.0f, so));
  for (int ch = 0; ch < 3; ++ch) {
    const float sc = sigmoid_f(z[i * 4 + 1 + ch]);
    dz[i * 4 + 1 + ch] = __fmul_rn(__fmul_rn(gcol[i * 3 + ch], sc), __fsub_rn(1.0f, sc));
  }
}

// ---------------------------------------------------------------- per model
struct MetaArgs {
  int R;
  const uint8_t* ok;
  const uint8_t* frozen;
  const int32_t* model_rays;
  const float* terms;
  const int64_t* step;
  const float* corr1;
  const float* corr2;
  int corr_len;
  double beta1, beta2;
  float* losses;    // [K][3]
  int32_t* status;  // this stack's 4 words
  uint8_t* upd;
  float2* corr;
};

// Update mask ray_ok.any(-1) & ~frozen (trainer.py:504, models.py:418-420),
// this step's bias corrections, the loss triple as numpy's pairwise sum over
// rays (render.py:305-307) and the non-finite-loss flag (trainer.py:404-407).
__global__ void __launch_bounds__(128) meta_kernel(const __grid_constant__ MetaArgs a) {
  const int k = blockIdx.x, tid = threadIdx.x;
  bool any_ok = false;
  for (int r = tid; r < a.R; r += blockDim.x) any_ok |= a.ok[int64_t(k) * a.R + r] != 0;
  const bool upd = __syncthreads_or(any_ok);
  if (tid == 0) {
    a.upd[k] = upd && !a.frozen[k] ? 1 : 0;
    a.corr[k] = bias_corrections(a.corr1, a.corr2, a.corr_len, a.beta1, a.beta2, a.step[k]);
  }
  if (tid < 3) {
    const float* terms = a.terms + int64_t(k) * a.R * 3;
    // rows past a model's live ray count are the reference's zero padding
    const int live = a.model_rays ? min(a.model_rays[k], a.R) : a.R;
    const float sum = pairwise_sum([&](int64_t r) { return r < live ? terms[r * 3 + tid] : 0.f; }, a.R);
    a.losses[int64_t(k) * 3 + tid] = sum;
    if (!isfinite(sum)) atomicMin(&a.status[1], k);
  }
}

struct ReduceArgs {
  int M, N, splits;       // partial blocks [splits][N][ldp] per model (C^T; M = fi_pad + 1: element fi_pad = db)
  int ldp;
  int fi_pad;
  const float* part;
  float* grads;           // [K][block]
  int64_t block, w_off, b_off;
  const uint8_t* upd;     // non-finite check for updating models (null: none)
  int32_t* status;
};

// Sums the sample chunks of one layer's weight gradient in chunk order and
// scatters [dW^T ; db] into the arena layout (dW row o, column i at
// w_off + o*fi_pad + i; db at b_off + o); a non-finite value of a model Adam
// would update raises status[0] (models.py:423-428).
__global__ void __launch_bounds__(256) reduce_kernel(const __grid_constant__ ReduceArgs a) {
  const int k = blockIdx.y;
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t MN = int64_t(a.M) * a.N;
  const int64_t blk = int64_t(a.ldp) * a.N;  // one sample chunk's partial block
  bool bad = false;
  if (e < MN) {
    // e enumerates output o = e / M (row of dW) and input i = e % M, in the
    // order of both the partials (C^T rows of ldp floats) and the arena
    const int o = int(e / a.M), i = int(e % a.M);
    const float* p = a.part + int64_t(k) * a.splits * blk + int64_t(o) * a.ldp + i;
    float v = p[0];
    for (int s = 1; s < a.splits; ++s) v = __fadd_rn(v, p[s * blk]);
    float* gk = a.grads + int64_t(k) * a.block;
    if (i == a.fi_pad) gk[a.b_off + o] = v;
    else gk[a.w_off + int64_t(o) * a.fi_pad + i] = v;
    bad = !isfinite(v);
  }
  if (a.upd && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0 && a.upd[k]) atomicMin(&a.status[0], k);
}

struct AdamArgs {
  float* P;
  float* M;
  float* V;
  const float* G;
  int64_t* step;
  int64_t block;
  int chunks;
  const uint8_t* upd;
  const float2* corr;
  int32_t* status;        // this stack's words
  const int32_t* prior;   // words of the stacks trained before this one (4 each)
  int n_prior;
  AdamConsts c;
};

// models.py:444-461 on every updating model, unless this stack saw a
// non-finite gradient or an earlier stack a non-finite gradient or loss
// (the reference raises before reaching this stack, trainer.py:364-390).
__global__ void __launch_bounds__(256) adam_kernel(const __grid_constant__ AdamArgs a) {
  const int k = blockIdx.y, ch = blockIdx.x;
  bool skip = a.status[0] != kSent;
  for (int j = 0; j < a.n_prior; ++j) skip |= a.prior[4 * j] != kSent || a.prior[4 * j + 1] != kSent;
  if (k == 0 && ch == 0 && threadIdx.x == 0) a.status[2] = skip ? 0 : 1;
  if (skip || !a.upd[k]) return;
  const float2 c = a.corr[k];
  const int64_t base = int64_t(k) * a.block;
  for (int64_t i = (int64_t(ch) * blockDim.x + threadIdx.x) * 4; i < a.block; i += int64_t(a.chunks) * blockDim.x * 4)
    adam_vec4(a.P + base, a.M + base, a.V + base, a.G + base, i, c.x, c.y, a.c);
  if (ch == 0 && threadIdx.x == 0) a.step[k] += 1;
}

__global__ void status_init_kernel(int32_t* status, int n) {
  if (threadIdx.x < n) status[threadIdx.x] = kSent;
}

// ---------------------------------------------------------------- host plan
inline size_t al(size_t x) { return (x + 255) / 256 * 256; }

// Sample chunks of a weight-gradient GEMM: enough CTAs per model to fill the
// GPU at small widths, >= 512 samples each; a function of the model's own
// shape only (vectorised == sequential bits).
inline int dw_splits(int64_t n_samples, int M, int N) {
  const int tiles = ((M + 127) / 128) * ((N + (N <= 32 ? 31 : 127)) / (N <= 32 ? 32 : 128));
  const int64_t by_n = std::max<int64_t>(1, (n_samples + 511) / 512);
  const int64_t by_t = std::max(1, 32 / tiles);
  return int(std::min(by_n, by_t));
}
inline int dw_chunk(int64_t n_samples, int splits) {
  const int64_t c = (n_samples + splits - 1) / splits;
  return int((c + kBK - 1) / kBK * kBK);
}

struct Plan {
  VmLayout L;
  int K, hp;
  int64_t N;  // samples per model
  size_t off_act, off_z, off_dz0, off_dz1, off_part, off_grads, off_terms, off_upd, off_corr, bytes;
  size_t part_floats;  // per model, max over layers
};

int plan(const VmStack& st, int64_t n_samples, int R, bool train, bool keep_acts, Plan& p) {
  int rc = compute_layout(st.arch, p.L);
  if (rc) {
    set_error("layered: unsupported architecture");
    return rc;
  }
  p.K = st.count;
  p.hp = p.L.hidden_pad;
  p.N = n_samples;
  const size_t K = size_t(p.K), N = size_t(n_samples), hp = size_t(p.hp);
  const int nl = p.L.n_layers;
  size_t off = 0;
  // activations of layers 0..L-2 (all kept for the backward; two ping-pong
  // buffers for a forward-only evaluation)
  const size_t n_act = keep_acts ? size_t(nl - 1) : std::min<size_t>(2, nl - 1);
  p.off_act = off;   off = al(off + n_act * K * N * hp * 4);
  p.off_z = off;     off = al(off + (train ? K * N * 4 * 4 : 0));
  const size_t dzw = std::max<size_t>(hp, 4);
  p.off_dz0 = off;   off = al(off + (keep_acts ? K * N * dzw * 4 : 0));
  p.off_dz1 = off;   off = al(off + (keep_acts ? K * N * dzw * 4 : 0));
  p.part_floats = 0;
  if (keep_acts)
    for (int l = 0; l < nl; ++l) {
      const int M = p.L.fi_pad[l] + 1, Nn = p.L.fo_pad[l];
      p.part_floats = std::max(p.part_floats, size_t(dw_splits(n_samples, M, Nn)) * (M + 3) * Nn);
    }
  p.off_part = off;  off = al(off + K * p.part_floats * 4);
  p.off_grads = off; off = al(off + (train ? K * size_t(p.L.block) * 4 : 0));
  p.off_terms = off; off = al(off + (train ? K * size_t(R) * 3 * 4 : 0));
  p.off_upd = off;   off = al(off + (train ? K : 0));
  p.off_corr = off;  off = al(off + (train ? K * 8 : 0));
  p.bytes = off;
  return VM_OK;
}

// Forward of every layer: act_l (l < L-1) and either the raw output z
// (training) or the sigmoid heads into occ/col (evaluation).
int forward(const VmStack& st, const Plan& p, const float* enc, int D, char* ws, bool keep_acts, float* z,
            float* occ, float* col, cudaStream_t s) {
  const int nl = p.L.n_layers, K = p.K;
  const int64_t N = p.N, hp = p.hp;
  float* act = reinterpret_cast<float*>(ws + p.off_act);
  const float* x = enc;
  int64_t ldx = D;
  int valid_k = D;
  for (int l = 0; l < nl; ++l) {
    Gemm g{};
    g.M = int(N);
    g.N = p.L.fo_pad[l];
    g.Kd = valid_k;
    g.A = x, g.lda = ldx, g.sA = N * ldx;
    g.a_valid = int(N), g.a_ones = -1;
    g.B = st.params + p.L.w_off[l], g.ldb = p.L.fi_pad[l], g.sB = p.L.block;
    g.bias = st.params + p.L.b_off[l], g.sBias = p.L.block;
    g.splits = 1, g.kchunk = valid_k;
    const bool last = l == nl - 1;
    int rc;
    if (!last) {
      float* out = act + (keep_acts ? size_t(l) : size_t(l % 2)) * K * N * hp;
      g.C = out, g.ldc = hp, g.sC = N * hp;
      rc = launch_gemm<kEpiBiasRelu, true, true>(g, K, s);
      x = out;
      ldx = hp;
      valid_k = int(hp);
    } else if (z) {
      g.C = z, g.ldc = 4, g.sC = N * 4;
      rc = launch_gemm<kEpiBias, true, true>(g, K, s);
    } else {
      g.occ = occ, g.col = col, g.sO = N;
      rc = launch_gemm<kEpiHeads, true, true>(g, K, s);
    }
    if (rc) return rc;
  }
  return VM_OK;
}

// Backward of every layer from the output dz (in dz0): weight gradients into
// `grads` (arena layout), non-finite check against `upd`.
int backward(const VmStack& st, const Plan& p, const float* enc, int D, char* ws, float* grads, const uint8_t* upd,
             int32_t* status, cudaStream_t s) {
  const int nl = p.L.n_layers, K = p.K;
  const int64_t N = p.N, hp = p.hp;
  const float* act = reinterpret_cast<const float*>(ws + p.off_act);
  float* dzb[2] = {reinterpret_cast<float*>(ws + p.off_dz0), reinterpret_cast<float*>(ws + p.off_dz1)};
  float* part = reinterpret_cast<float*>(ws + p.off_part);
  int cur = 0;
  for (int l = nl - 1; l >= 0; --l) {
    const int fo_pad = p.L.fo_pad[l], fi_pad = p.L.fi_pad[l];
    const float* x = l == 0 ? enc : act + size_t(l - 1) * K * N * hp;
    const int64_t ldx = l == 0 ? D : hp;
    // [dW^T ; db] = [x | 1]^T dz, split over samples (the ones row, db, as
    // the column sums of dz inside the same launch: no extra M tile)
    Gemm g{};
    g.M = fi_pad;
    g.N = fo_pad;
    g.Kd = int(N);
    g.A = x, g.lda = ldx, g.sA = N * ldx;
    g.a_valid = l == 0 ? D : int(hp);
    g.a_ones = -1;
    g.db_row = fi_pad;
    g.B = dzb[cur], g.ldb = fo_pad, g.sB = N * fo_pad;
    g.splits = dw_splits(N, fi_pad + 1, g.N);
    g.kchunk = dw_chunk(N, g.splits);
    g.C = part, g.ldc = fi_pad + 4, g.sCsplit = int64_t(fi_pad + 4) * g.N, g.sC = g.splits * g.sCsplit;
    int rc = launch_gemm<kEpiStore, false, false>(g, K, s);
    if (rc) return rc;
    ReduceArgs r{};
    r.M = fi_pad + 1, r.N = g.N, r.ldp = fi_pad + 4, r.splits = g.splits, r.fi_pad = fi_pad;
    r.part = part, r.grads = grads, r.block = p.L.block, r.w_off = p.L.w_off[l], r.b_off = p.L.b_off[l];
    r.upd = upd, r.status = status;
    const int64_t MN = int64_t(r.M) * g.N;
    reduce_kernel<<<dim3(unsigned((MN + 255) / 256), K), 256, 0, s>>>(r);
    VM_CUDA(cudaGetLastError());
    if (l == 0) break;
    // dz_{l-1} = (dz_l W_l) * (x_l > 0)
    Gemm d{};
    d.M = int(N);
    d.N = fi_pad;
    d.Kd = fo_pad;
    d.A = dzb[cur], d.lda = fo_pad, d.sA = N * fo_pad;
    d.a_valid = int(N), d.a_ones = -1;
    d.B = st.params + p.L.w_off[l], d.ldb = fi_pad, d.sB = p.L.block;
    d.C = dzb[cur ^ 1], d.ldc = fi_pad, d.sC = N * fi_pad;
    d.mask = x, d.ldm = hp, d.sM = N * hp;
    d.splits = 1, d.kchunk = fo_pad;
    rc = launch_gemm<kEpiMask, true, false>(d, K, s);
    if (rc) return rc;
    cur ^= 1;
  }
  return VM_OK;
}

int check_batch(const VmStack& st, const VmBatch& b) {
  VM_REQUIRE(b.n_models == st.count, "vm_train_step: batch leading axis != params.count");
  VM_REQUIRE(b.input_dim == st.arch.input_dim, "vm_train_step: encoding dim mismatch");
  VM_REQUIRE(b.n_points >= 1 && b.n_points <= kMaxS, "vm_train_step: points per ray must be in [1, 64]");
  VM_REQUIRE(b.n_rays >= 1 || st.count == 0, "vm_train_step: no rays");
  VM_REQUIRE(b.encoded != nullptr || st.count == 0,
             "vm_train_step: this architecture takes the layered path, which needs the encoded input");
  return VM_OK;
}

}  // namespace lyr

// VM_LAYERED=1 routes every train step through the layered path (A/B and the
// cross-check of the fused kernels against it).
bool layered_forced() {
  static const bool on = [] {
    const char* e = std::getenv("VM_LAYERED");
    return e && e[0] == '1';
  }();
  return on;
}

size_t layered_train_bytes(const VmStack* stacks, const VmBatch* batches, int n, int first) {
  size_t m = 0;
  for (int i = first; i < n; ++i) {
    lyr::Plan p;
    if (lyr::check_batch(stacks[i], batches[i])) return 0;
    if (lyr::plan(stacks[i], int64_t(batches[i].n_rays) * batches[i].n_points, batches[i].n_rays, true, true, p))
      return 0;
    m = std::max(m, p.bytes);  // stacks run one after another: one region serves all
  }
  return m;
}

int train_layered(const VmStack* stacks, const VmBatch* batches, int n, int first, VmLossWeights w, float* losses,
                  int32_t* status, void* workspace, size_t workspace_bytes, cudaStream_t s) {
  VM_REQUIRE(n >= 1 && n <= VM_MAX_STACKS && first >= 0 && first < n, "vm_train_step: 1 or 2 stacks supported");
  for (int i = first; i < n; ++i) {
    const int rc = lyr::check_batch(stacks[i], batches[i]);
    if (rc) return rc;
  }
  VM_REQUIRE(workspace_bytes >= layered_train_bytes(stacks, batches, n, first), "vm_train_step: workspace too small");
  lyr::status_init_kernel<<<1, 32, 0, s>>>(status + 4 * first, 4 * (n - first));
  VM_CUDA(cudaGetLastError());
  char* ws = static_cast<char*>(workspace);
  int loss_off = 0;
  for (int i = 0; i < first; ++i) loss_off += stacks[i].count;
  for (int i = first; i < n; ++i) {
    const VmStack& st = stacks[i];
    const VmBatch& b = batches[i];
    const int K = st.count;
    if (K == 0) continue;
    lyr::Plan p;
    int rc = lyr::plan(st, int64_t(b.n_rays) * b.n_points, b.n_rays, true, true, p);
    if (rc) return rc;
    float* z = reinterpret_cast<float*>(ws + p.off_z);
    float* dz = reinterpret_cast<float*>(ws + p.off_dz0);
    float* grads = reinterpret_cast<float*>(ws + p.off_grads);
    float* terms = reinterpret_cast<float*>(ws + p.off_terms);
    uint8_t* upd = reinterpret_cast<uint8_t*>(ws + p.off_upd);
    float2* corr = reinterpret_cast<float2*>(ws + p.off_corr);
    int32_t* stw = status + 4 * i;
    rc = lyr::forward(st, p, b.encoded, st.arch.input_dim, ws, true, z, nullptr, nullptr, s);
    if (rc) return rc;
    lyr::RayArgs ra{K, b.n_rays, b.n_points, z, b.t, b.target_depth, b.target_colour, b.target_mask,
                    b.valid_depth, b.ray_ok, w.colour, w.occupancy, dz, terms};
    const int64_t rays = int64_t(K) * b.n_rays;
    lyr::ray_kernel<<<unsigned((rays + 127) / 128), 128, 0, s>>>(ra);
    VM_CUDA(cudaGetLastError());
    lyr::MetaArgs ma{b.n_rays, b.ray_ok, st.frozen, b.model_rays, terms, st.step, st.corr1, st.corr2, st.corr_len,
                     st.beta1, st.beta2, losses + int64_t(loss_off) * 3, stw, upd, corr};
    lyr::meta_kernel<<<K, 128, 0, s>>>(ma);
    VM_CUDA(cudaGetLastError());
    rc = lyr::backward(st, p, b.encoded, st.arch.input_dim, ws, grads, upd, stw, s);
    if (rc) return rc;
    lyr::AdamArgs aa{};
    aa.P = st.params, aa.M = st.m, aa.V = st.v, aa.G = grads, aa.step = st.step;
    aa.block = p.L.block;
    aa.chunks = int(std::min<int64_t>(64, (p.L.block / 4 + 255) / 256));
    aa.upd = upd, aa.corr = corr, aa.status = stw, aa.prior = status, aa.n_prior = i;
    aa.c = adam_consts(st);
    lyr::adam_kernel<<<dim3(aa.chunks, K), 256, 0, s>>>(aa);
    VM_CUDA(cudaGetLastError());
    loss_off += K;
  }
  return VM_OK;
}

// vm_forward / vm_backward for the architectures the fused kernels lack: the
// layer buffers in a stream-ordered temporary (the standalone entry points'
// convention, like vm_losses).
int layered_fwd_bwd(const VmStack& st, const float* enc, int64_t n_samples, const float* gocc, const float* gcol,
                    float* occ, float* col, float* grads, bool backward, cudaStream_t s) {
  lyr::Plan p;
  int rc = lyr::plan(st, n_samples, 0, false, backward, p);
  if (rc) return rc;
  const int K = st.count;
  const int D = st.arch.input_dim;
  if (K == 0) return VM_OK;
  if (n_samples == 0) {
    if (backward) VM_CUDA(cudaMemsetAsync(grads, 0, size_t(K) * p.L.block * 4, s));
    return VM_OK;
  }
  const size_t zb = backward ? size_t(K) * n_samples * 16 : 0;
  char* ws = nullptr;
  VM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), p.bytes + zb, s));
  float* z = backward ? reinterpret_cast<float*>(ws + p.bytes) : nullptr;
  rc = lyr::forward(st, p, enc, D, ws, backward, z, occ, col, s);
  if (!rc && backward) {
    const int64_t n = int64_t(K) * n_samples;
    lyr::heads_grad_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(n, z, gocc, gcol,
                                                                      reinterpret_cast<float*>(ws + p.off_dz0));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_check(e, "heads_grad_kernel");
    if (!rc) rc = lyr::backward(st, p, enc, D, ws, grads, nullptr, nullptr, s);
  }
  const cudaError_t fe = cudaFreeAsync(ws, s);
  if (rc) return rc;
  VM_CUDA(fe);
  return VM_OK;
}

}  // namespace vm
