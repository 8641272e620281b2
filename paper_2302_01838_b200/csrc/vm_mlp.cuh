// Fused per-object MLP field kernel (KF): positional-encoded samples ->
// forward -> occupancy render + L1 loss -> render backward -> MLP backward ->
// per-object weight-gradient reduction, with every activation on chip.
//
// Reference math: models.py:311-398 (forward/backward), render.py:230-333
// (render, losses, grads), trainer.py:480-506 (the train_on_batch chain).
//
// Execution model (B200, sm_100a):
//  * One CTA (8 warps) per work item = (stack, model, ray range).  The model's
//    whole parameter block (13.7 KB at hidden 32, 153 KB at hidden 128) is
//    staged in shared memory once; hidden/output weight rows are XOR-swizzled
//    in 16-B chunks so both the forward (rows across lanes) and the dx pass
//    (columns across lanes) read them bank-conflict free.
//  * Samples are processed in 32-sample blocks = floor(32/S) whole rays, so
//    the render never crosses a block.  A "team" of T warps owns one block at
//    a time (T=1 at hidden 32: eight independent warps; T=8 at hidden 128:
//    the whole CTA) and splits every layer's output dimension between its
//    warps.  Activations are feature-major in smem (row stride 36 floats),
//    which makes every GEMM operand a conflict-free LDS.128.
//  * Register-blocked FP32 FFMA micro-GEMMs: forward 4 samples x OW/4 outputs
//    per lane (32 FMA per 3 LDS.128 at OW=32), dx likewise, and dW as a
//    K=samples GEMM accumulated straight into registers that persist across
//    all blocks of the work item.  Backward runs in place: dz of layer l
//    overwrites layer l's activation buffer once its dW is taken.
//  * End of item: teams are summed in fixed order (deterministic) and the
//    gradient block is written; when a model is split over several CTAs the
//    last one to finish (atomic ticket) sums the partials in order, the
//    per-ray losses with numpy's pairwise order, and raises the non-finite
//    flags Adam needs.
#pragma once

#include "vm_adam.cuh"
#include "vm_render.cuh"

namespace vm {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kSB = 32;    // samples per block
constexpr int kLD = 36;    // activation row stride in floats (== 4 mod 32)
constexpr int kDpMax = 40; // max padded input rows

template <int H> struct TeamCfg;
// hidden 32: teams of 2 warps (16 outputs each) so a warp's share of the
// register-resident weight gradient is ~58 floats and two 8-warp CTAs fit an
// SM (16 warps; 128 registers, ~92 KB smem each).
template <> struct TeamCfg<32> { static constexpr int T = 2, OW = 16; };
template <> struct TeamCfg<64> { static constexpr int T = 4, OW = 16; };
template <> struct TeamCfg<128> { static constexpr int T = 8, OW = 16; };

enum Mode : int { kTrain = 0, kForward = 1, kBackward = 2 };

struct KStack {
  int H, L, D, Dp, fi0;
  int block, w_floats, team_floats;
  int w_off[VM_MAX_LAYERS], b_off[VM_MAX_LAYERS];
  int K, R, S, G, P;          // models, rays, points/ray, rays/block, CTAs per model
  int tc;                     // 1: trained by the tensor-core kernel KT (vm_tc_mlp.cuh)
  int ls_sep;                 // 1: loss sums by loss_sums_kernel (split tensor-core stacks), not the reduce
  int64_t N;                  // samples per model (forward/backward modes)
  int model_base;             // global model index of model 0 (losses/status)
  int chunk;                  // ray blocks per work item (FFMA kernels)
  const int* model_rays;      // [K] live rays per model (config 3), or null: all R
  const int* items;           // [2*n_items] (model, chunk) work items, or null: item = k*P + chunk
  int n_items;
  int item_base;              // first CTA index of this stack
  const float* params;
  const uint8_t* frozen;
  const int64_t* step;
  const float* corr1;
  const float* corr2;
  int corr_len;
  double beta1, beta2;
  const float* enc;       // [K][R*S][D] encoded samples, or
  const float* pts;       // [K][R*S][3] box-normalised points (PE fused here)
  const float* pe_scale;  // [K] per-model PE scale (points path)
  int n_freq, include_input;
  const float* t;
  const float* tdepth;
  const float* tcol;
  const uint8_t* tmask;
  const uint8_t* valid;
  const uint8_t* ok;
  const float* gocc;
  const float* gcol;
  float* occ_out;
  float* col_out;
  float* grads;      // [K][block]
  float* partials;   // [K*P][block] (P > 1)
  float* ray_terms;  // [K][R][3]
  int* counters;     // [K]
  uint8_t* upd;      // [K]
  float2* corr;      // [K] bias corrections for this step
  float* losses;     // [K][3] (already offset by model_base)
  int32_t* status;   // [4]
  float wc, wo;
};

struct KParams {
  KStack s[2];
  int n_stacks;
  int* queue;      // persistent FFMA kernel: next work item (zeroed before the launch), or null
  int n_items;     // work items over all stacks (persistent kernel)
  unsigned long long* trace;  // VM_TRACE=1: per-CTA/item schedule records, or null
};



// vm_kf32.cu: the specialised hidden-32 / 4-layer train kernel
bool kf32_supported(const KParams& p);
size_t kf32_smem_bytes();
int launch_kf32(const KParams& p, int grid, cudaStream_t s);
// vm_kh32.cu: the same step on the warp-level tensor path (3xTF32 mma.sync)
bool kh32_supported(const KParams& p);
int launch_kh32(const KParams& p, int grid, cudaStream_t s);

__device__ __forceinline__ void team_sync(int team, int T) {
  if (T == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(T * 32) : "memory");
  }
}

__device__ __forceinline__ int swz(int row, int col) {  // col multiple of 4
  return (((col >> 2) ^ (row & 7)) << 2);
}

__device__ __forceinline__ float relu_np(float z) { return z != z ? z : fmaxf(z, 0.0f); }
__device__ __forceinline__ float sigmoid_f(float z) { return 1.0f / (1.0f + expf(-z)); }

// ---- forward: Y[o][s] = relu(sum_k W[o][k] X[k][s] + b[o]) for o in
// [o0, o0+OW): lane = (a: sample quad, b: output phase), outputs interleaved.
template <int OW, bool SWZ, int KC>
__device__ __forceinline__ void fwd_layer(const float* __restrict__ W, int ws, const float* __restrict__ bias,
                                          const float* __restrict__ X, int Krt, float* __restrict__ Y, int o0,
                                          int lane) {
  constexpr int NJ = OW / 4;
  const int a = lane & 7, b = lane >> 3;
  const int K = KC > 0 ? KC : Krt;
  float acc[NJ][4];
#pragma unroll
  for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll(KC > 0 ? 8 : 1)
  for (int k = 0; k < K; k += 4) {
    const float4 x0 = ld4(X + (k + 0) * kLD + 4 * a);
    const float4 x1 = ld4(X + (k + 1) * kLD + 4 * a);
    const float4 x2 = ld4(X + (k + 2) * kLD + 4 * a);
    const float4 x3 = ld4(X + (k + 3) * kLD + 4 * a);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int o = o0 + b + 4 * j;
      const float4 w = ld4(W + o * ws + (SWZ ? swz(o, k) : k));
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
  for (int j = 0; j < NJ; ++j) {
    const int o = o0 + b + 4 * j;
    const float bb = bias[o];
    float4 r;
    r.x = relu_np(acc[j][0] + bb);
    r.y = relu_np(acc[j][1] + bb);
    r.z = relu_np(acc[j][2] + bb);
    r.w = relu_np(acc[j][3] + bb);
    st4(Y + o * kLD + 4 * a, r);
  }
}

// ---- output layer (4 logits -> sigmoid): lane = (sample quad a, output b).
template <int H>
__device__ __forceinline__ void fwd_out(const float* __restrict__ W, const float* __restrict__ bias,
                                        const float* __restrict__ X, float* __restrict__ O, int lane) {
  const int a = lane & 7, b = lane >> 3;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int k = 0; k < H; k += 4) {
    const float4 x0 = ld4(X + (k + 0) * kLD + 4 * a);
    const float4 x1 = ld4(X + (k + 1) * kLD + 4 * a);
    const float4 x2 = ld4(X + (k + 2) * kLD + 4 * a);
    const float4 x3 = ld4(X + (k + 3) * kLD + 4 * a);
    const float4 w = ld4(W + b * H + swz(b, k));
    acc[0] = fmaf(w.x, x0.x, acc[0]); acc[1] = fmaf(w.x, x0.y, acc[1]);
    acc[2] = fmaf(w.x, x0.z, acc[2]); acc[3] = fmaf(w.x, x0.w, acc[3]);
    acc[0] = fmaf(w.y, x1.x, acc[0]); acc[1] = fmaf(w.y, x1.y, acc[1]);
    acc[2] = fmaf(w.y, x1.z, acc[2]); acc[3] = fmaf(w.y, x1.w, acc[3]);
    acc[0] = fmaf(w.z, x2.x, acc[0]); acc[1] = fmaf(w.z, x2.y, acc[1]);
    acc[2] = fmaf(w.z, x2.z, acc[2]); acc[3] = fmaf(w.z, x2.w, acc[3]);
    acc[0] = fmaf(w.w, x3.x, acc[0]); acc[1] = fmaf(w.w, x3.y, acc[1]);
    acc[2] = fmaf(w.w, x3.z, acc[2]); acc[3] = fmaf(w.w, x3.w, acc[3]);
  }
  const float bb = bias[b];
  float4 r;
  r.x = sigmoid_f(acc[0] + bb);
  r.y = sigmoid_f(acc[1] + bb);
  r.z = sigmoid_f(acc[2] + bb);
  r.w = sigmoid_f(acc[3] + bb);
  st4(O + b * kLD + 4 * a, r);
}

// ---- dx: A[i][s] <- (sum_o W[o][i] G[o][s]) * (A[i][s] > 0) for i in
// [i0, i0+OW) (in place), K = rows of G.  Lane b owns OW/4 contiguous inputs.
template <int OW, int K, int H>
__device__ __forceinline__ void dx_layer(const float* __restrict__ W, const float* __restrict__ G,
                                         float* __restrict__ A, int i0, int lane) {
  constexpr int NI = OW / 4;
  const int a = lane & 7, b = lane >> 3;
  const int ib = i0 + b * NI;
  float acc[NI][4];
#pragma unroll
  for (int c = 0; c < NI; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0.f;
#pragma unroll(K > 8 ? 4 : K)
  for (int o = 0; o < K; ++o) {
    const float4 g = ld4(G + o * kLD + 4 * a);
#pragma unroll
    for (int c4 = 0; c4 < NI / 4; ++c4) {
      const int i = ib + 4 * c4;
      const float4 w = ld4(W + o * H + swz(o, i));
      acc[4 * c4 + 0][0] = fmaf(w.x, g.x, acc[4 * c4 + 0][0]); acc[4 * c4 + 0][1] = fmaf(w.x, g.y, acc[4 * c4 + 0][1]);
      acc[4 * c4 + 0][2] = fmaf(w.x, g.z, acc[4 * c4 + 0][2]); acc[4 * c4 + 0][3] = fmaf(w.x, g.w, acc[4 * c4 + 0][3]);
      acc[4 * c4 + 1][0] = fmaf(w.y, g.x, acc[4 * c4 + 1][0]); acc[4 * c4 + 1][1] = fmaf(w.y, g.y, acc[4 * c4 + 1][1]);
      acc[4 * c4 + 1][2] = fmaf(w.y, g.z, acc[4 * c4 + 1][2]); acc[4 * c4 + 1][3] = fmaf(w.y, g.w, acc[4 * c4 + 1][3]);
      acc[4 * c4 + 2][0] = fmaf(w.z, g.x, acc[4 * c4 + 2][0]); acc[4 * c4 + 2][1] = fmaf(w.z, g.y, acc[4 * c4 + 2][1]);
      acc[4 * c4 + 2][2] = fmaf(w.z, g.z, acc[4 * c4 + 2][2]); acc[4 * c4 + 2][3] = fmaf(w.z, g.w, acc[4 * c4 + 2][3]);
      acc[4 * c4 + 3][0] = fmaf(w.w, g.x, acc[4 * c4 + 3][0]); acc[4 * c4 + 3][1] = fmaf(w.w, g.y, acc[4 * c4 + 3][1]);
      acc[4 * c4 + 3][2] = fmaf(w.w, g.z, acc[4 * c4 + 3][2]); acc[4 * c4 + 3][3] = fmaf(w.w, g.w, acc[4 * c4 + 3][3]);
    }
  }
#pragma unroll
  for (int c = 0; c < NI; ++c) {
    float* p = A + (ib + c) * kLD + 4 * a;
    const float4 av = ld4(p);
    float4 r;
    r.x = acc[c][0] * (av.x > 0.f ? 1.f : 0.f);
    r.y = acc[c][1] * (av.y > 0.f ? 1.f : 0.f);
    r.z = acc[c][2] * (av.z > 0.f ? 1.f : 0.f);
    r.w = acc[c][3] * (av.w > 0.f ? 1.f : 0.f);
    st4(p, r);
  }
}

// ---- dW[o][i] += sum_s G[o][s] X[i][s]: rows o = o0 + r + 4j (j < NJ),
// cols i = c0 + c + 8q (q < NQ, only q < nq live); lane = (r: 0..3, c: 0..7).
template <int NJ, int NQ>
__device__ __forceinline__ void dw_acc(float (&acc)[NJ][NQ], const float* __restrict__ G, int o0,
                                       const float* __restrict__ X, int c0, int nq, int lane) {
  const int r = lane >> 3, c = lane & 7;
#pragma unroll 2
  for (int s = 0; s < kSB; s += 4) {
    float4 g[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) g[j] = ld4(G + (o0 + r + 4 * j) * kLD + s);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (q < nq) {
        const float4 x = ld4(X + (c0 + c + 8 * q) * kLD + s);
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
}

// ---- db[o] += sum_s G[o][s] for the warp's OW rows.
template <int OW>
__device__ __forceinline__ float db_acc(const float* __restrict__ G, int o0, int lane) {
  constexpr int SPL = 32 / OW;
  constexpr int NS = kSB / SPL;
  const int row = o0 + (lane % OW), part = lane / OW;
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NS; k += 4) {
    const float4 v = ld4(G + row * kLD + part * NS + k);
    s += (v.x + v.y) + (v.z + v.w);
  }
  return s;
}

// Register-resident gradient accumulators of one warp.
template <int H, int L>
struct WarpGrads {
  static constexpr int T = TeamCfg<H>::T, OW = TeamCfg<H>::OW;
  static constexpr int NJ = OW / 4;
  static constexpr int NQH = H / 8;       // hidden fan-in column groups
  static constexpr int NQ0 = kDpMax / 8;  // layer-0 column groups
  static constexpr int NQL = H / 8 / T;   // output layer column groups per warp
  static constexpr int NH = L - 2;        // hidden->hidden layers
  float w0[NJ][NQ0];
  float wh[NH > 0 ? NH : 1][NJ][NQH];
  float wl[1][NQL];
  float bh[L - 1];   // bias of layers 0..L-2 (row o0 + lane%OW, partial over sample part)
  float bl;          // output-layer bias (lanes 0..3 of warp 0 in team)

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int q = 0; q < NQ0; ++q) w0[j][q] = 0.f;
#pragma unroll
    for (int h = 0; h < (NH > 0 ? NH : 1); ++h)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int q = 0; q < NQH; ++q) wh[h][j][q] = 0.f;
#pragma unroll
    for (int q = 0; q < NQL; ++q) wl[0][q] = 0.f;
#pragma unroll
    for (int l = 0; l < L - 1; ++l) bh[l] = 0.f;
    bl = 0.f;
  }
};

// Per-model epilogue of a training step: update mask = ray_ok.any(-1)
// (trainer.py:504) and active = !frozen; the model's loss triple as numpy's
// pairwise sum over rays of the per-ray terms (render.py:305-307); the
// non-finite flags Adam and the host need (models.py:423-428,
// trainer.py:404-407); this step's bias corrections.  Called by all threads
// of a CTA.  `meta` selects the writer of the per-model words.
static __device__ __noinline__ void model_loss_sums(const KStack& st, int k, float* scratch, int scratch_floats);

__device__ inline void finalize_model(const KStack& st, int k, bool all_finite, bool meta, float* scratch,
                               int scratch_floats, bool sums = true) {
  const int tid = threadIdx.x;
  // non-meta CTAs only need the update mask when their chunk is non-finite
  // (both conditions are CTA-uniform, so the barrier below is too)
  if (!meta && all_finite) return;
  bool any_ok = false;
  for (int r = tid; r < st.R; r += blockDim.x) any_ok |= st.ok[int64_t(k) * st.R + r] != 0;
  const bool upd = __syncthreads_or(any_ok);
  const bool active = upd && !st.frozen[k];
  if (tid == 0 && active && !all_finite) atomicMin(&st.status[0], k);
  if (!meta) return;
  if (tid == 0) {
    st.upd[k] = active ? 1 : 0;
    st.corr[k] = bias_corrections(st.corr1, st.corr2, st.corr_len, st.beta1, st.beta2, st.step[k]);
  }
  if (sums) model_loss_sums(st, k, scratch, scratch_floats);
}

// The model's three loss sums over its rays in numpy's pairwise order
// (render.py:301-308) and the non-finite-loss flag.  Called by all threads.
static __device__ __noinline__ void model_loss_sums(const KStack& st, int k, float* scratch, int scratch_floats) {
  const int tid = threadIdx.x;
  // stage the per-ray terms in smem (coalesced), then 3 threads sum them in
  // numpy's pairwise order without a global-load latency per add
  const float* terms = st.ray_terms + int64_t(k) * st.R * 3;
  // rows past the model's live ray count are zero padding (config 3): their
  // terms are 0 in the reference's sums (render.py:301-308); kernels that skip
  // them never write these slots
  const int live3 = 3 * (st.model_rays ? min(st.model_rays[k], st.R) : st.R);
  const bool staged = st.R * 3 <= scratch_floats;
  if (staged) {
    // 8 independent loads in flight per thread (one L2 round trip per 8 rows
    // of the CTA, not per row)
    const int n3 = st.R * 3, nt = blockDim.x;
    for (int i0 = 0; i0 < n3; i0 += 8 * nt) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * nt + tid;
        v[u] = i < live3 ? __ldcg(terms + i) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * nt + tid;
        if (i < n3) scratch[i] = v[u];
      }
    }
    __syncthreads();
  }
  // more than one pairwise leaf: the leaves (<= 128 rays each) are summed by
  // separate threads, then combined in the recursion's order (same bits)
  constexpr int kMaxLeaves = 64;
  __shared__ int64_t lf_start[kMaxLeaves];
  __shared__ int lf_len[kMaxLeaves];
  __shared__ float lf_sum[3][kMaxLeaves];
  __shared__ int lf_n;
  const bool parallel = staged && st.R > 128 && 3 * kMaxLeaves <= int(blockDim.x);
  if (parallel) {
    if (tid == 0) lf_n = pairwise_leaves(st.R, lf_start, lf_len, kMaxLeaves);
    __syncthreads();
  }
  if (parallel && lf_n <= kMaxLeaves) {
    if (tid < 3 * lf_n) {
      const int j = tid % 3, lf = tid / 3;
      lf_sum[j][lf] = pairwise_sum_leaf([&](int64_t r) { return scratch[r * 3 + j]; }, lf_start[lf], lf_len[lf]);
    }
    __syncthreads();
    if (tid < 3) {
      int next = 0;
      const float sum = pairwise_combine(st.R, lf_sum[tid], next);
      st.losses[int64_t(k) * 3 + tid] = sum;
      if (!isfinite(sum)) atomicMin(&st.status[1], k);
    }
  } else if (tid < 3) {
    const int j = tid;
    const float sum = staged ? pairwise_sum([&](int64_t r) { return scratch[r * 3 + j]; }, st.R)
                             : pairwise_sum([&](int64_t r) { return r * 3 < live3 ? __ldcg(terms + r * 3 + j) : 0.f; },
                                            st.R);
    st.losses[int64_t(k) * 3 + j] = sum;
    if (!isfinite(sum)) atomicMin(&st.status[1], k);
  }
}


}  // namespace vm
