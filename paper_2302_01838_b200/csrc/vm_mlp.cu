// Fused train / forward / backward kernels over stacked per-object MLPs and
// their C-ABI launchers (vm_train_step, vm_forward, vm_backward).
#include "vm_mlp.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace vm {

// Stage the model block into smem; hidden and output weight rows swizzled.
template <int H, int L>
__device__ __forceinline__ void load_weights(const KStack& st, const float* __restrict__ gp, float* __restrict__ sW) {
  const int tid = threadIdx.x;
  // layer 0 (plain) + biases: copy as 16-B chunks without swizzle.
  {
    const int n4 = (st.w_off[1]) / 4;  // W0 and b0 are contiguous at the block start
    for (int i = tid; i < n4; i += kThreads) st4(sW + 4 * i, ld4(gp + 4 * i));
  }
#pragma unroll
  for (int l = 1; l < L; ++l) {
    const int rows = (l == L - 1) ? 4 : H;
    const int cpr = H / 4;
    const float* src = gp + st.w_off[l];
    float* dst = sW + st.w_off[l];
    for (int i = tid; i < rows * cpr; i += kThreads) {
      const int row = i / cpr, ch = i % cpr;
      st4(dst + row * H + swz(row, 4 * ch), ld4(src + row * H + 4 * ch));
    }
    const float* bsrc = gp + st.b_off[l];
    float* bdst = sW + st.b_off[l];
    for (int i = tid; i < rows / 4; i += kThreads) st4(bdst + 4 * i, ld4(bsrc + 4 * i));
  }
}

// Load the block's samples into E (feature-major) and t.  Encoded input is
// transposed from [sample][D]; point input is encoded on the fly with
// models.py:286-308's layout [p, sin(pi 2^i p / s) x3, cos(...) x3 per band]
// (f32 sincospif: tolerance-level vs the reference's f64 encoding).
__device__ __forceinline__ void load_block(const KStack& st, int k, int64_t gs0, int ns, float* __restrict__ E,
                                           float* __restrict__ tS, int tt, int nthr, bool with_t) {
  const int D = st.D;
  if (st.pts) {
    const float scale = st.pe_scale[k];
    for (int s = tt; s < kSB; s += nthr) {
      float p[3] = {0.f, 0.f, 0.f};
      if (s < ns) {
#pragma unroll
        for (int c = 0; c < 3; ++c) p[c] = st.pts[(gs0 + s) * 3 + c];
      }
      int f = 0;
      if (st.include_input) {
#pragma unroll
        for (int c = 0; c < 3; ++c) E[c * kLD + s] = p[c];
        f = 3;
      }
      for (int b = 0; b < st.n_freq; ++b, f += 6) {
        const float coef = float(double(1u << b) / double(scale));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float sn, cs;
          sincospif(coef * p[c], &sn, &cs);
          E[(f + c) * kLD + s] = s < ns ? sn : 0.f;
          E[(f + 3 + c) * kLD + s] = s < ns ? cs : 0.f;
        }
      }
    }
  } else {
    const float* src = st.enc + gs0 * D;
    for (int idx = tt; idx < kSB * D; idx += nthr) {
      const int s = idx / D, f = idx - s * D;
      E[f * kLD + s] = s < ns ? src[idx] : 0.f;
    }
  }
  for (int idx = tt; idx < (st.Dp - D) * kSB; idx += nthr) E[(D + idx / kSB) * kLD + (idx % kSB)] = 0.f;
  if (with_t && tt < kSB) tS[tt] = tt < ns ? st.t[gs0 + tt] : 0.f;
}

}  // namespace vm

#include "vm_tc_mlp.cuh"

namespace vm {

constexpr int kRedThreads = 256;
constexpr int kRedDirect = 8;                                 // P <= 8: one thread sums a float4's partials
constexpr int kRedGroups = 16;                                // partial groups per output column (P > 8)
constexpr int kRedChunk = kRedThreads / kRedGroups * 4;       // floats per reduce CTA (64)

// Sum the P partial gradient blocks of every split model in a fixed order
// (deterministic): group q of the CTA adds partials [q*P/16, (q+1)*P/16)
// sequentially (loads issued in batches of 6 before the adds; few registers
// so 6 CTAs fit an SM), then the 16 group sums are added in
// group order through shared memory.  One CTA per (model, 64-float chunk);
// chunk 0 also finalises the model.
__host__ __device__ inline int red_chunk_floats(int P) { return P <= kRedDirect ? kRedThreads * 4 : kRedChunk; }

__global__ void __launch_bounds__(kRedThreads, 6) reduce_partials_kernel(const __grid_constant__ KParams p,
                                                                          int only_stack) {
  struct Rec {  // schedule record at every exit
    const KParams& p;
    unsigned long long t;
    __device__ ~Rec() {
      if (p.trace && threadIdx.x == 0) vm_trace_rec(p.trace, 3, t);
    }
  } rec{p, p.trace ? vm_gtime() : 0ull};
  // launched with programmatic stream serialization behind KT: the CTAs may
  // be resident before KT finishes and wait here for its partials
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // let the Adam grid queued behind this one be scheduled now (it waits on
  // griddepcontrol.wait for this grid's completion before reading)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) float red_smem[];
  __shared__ float4 gsum[kRedGroups][kRedChunk / 4];
  int b = blockIdx.x, si = 0;
  for (; si < p.n_stacks; ++si) {
    const KStack& s = p.s[si];
    if (s.P <= 1 || (only_stack >= 0 && si != only_stack)) continue;
    const int cf = red_chunk_floats(s.P);
    const int n = s.K * ((s.block + cf - 1) / cf);
    if (b < n) break;
    b -= n;
  }
  if (si >= p.n_stacks) return;
  const KStack& st = p.s[si];
  const int cf = red_chunk_floats(st.P);
  const int chunks = (st.block + cf - 1) / cf;
  const int k = b / chunks, ch = b % chunks;
  bool finite = true;
  if (st.P <= kRedDirect) {
    // few partials (split FFMA items): one thread per float4, partials in order
    const int i = ch * cf + 4 * threadIdx.x;
    if (i < st.block) {
      const float* pb = st.partials + int64_t(k) * st.P * st.block + i;
      float4 w[kRedDirect];
#pragma unroll
      for (int u = 0; u < kRedDirect; ++u)
        if (u < st.P) w[u] = __ldcg(reinterpret_cast<const float4*>(pb + int64_t(u) * st.block));
      float4 tot = w[0];
#pragma unroll
      for (int u = 1; u < kRedDirect; ++u)
        if (u < st.P) {
          tot.x += w[u].x; tot.y += w[u].y; tot.z += w[u].z; tot.w += w[u].w;
        }
      st4(st.grads + int64_t(k) * st.block + i, tot);
      finite = isfinite(tot.x) && isfinite(tot.y) && isfinite(tot.z) && isfinite(tot.w);
    }
    const bool all_finite = __syncthreads_and(finite);
    finalize_model(st, k, all_finite, ch == 0, red_smem, st.R * 3, !st.ls_sep);
    return;
  }
  const int col = threadIdx.x % (kRedChunk / 4), q = threadIdx.x / (kRedChunk / 4);
  const int i = ch * kRedChunk + 4 * col;
  const int per = (st.P + kRedGroups - 1) / kRedGroups;
  const int p0 = min(st.P, q * per), p1 = min(st.P, p0 + per);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < st.block && p0 < p1) {
    const float* pb = st.partials + int64_t(k) * st.P * st.block + i;
    const int64_t stride = st.block;
    v = __ldcg(reinterpret_cast<const float4*>(pb + p0 * stride));
    int pp = p0 + 1;
    for (; pp + 6 <= p1; pp += 6) {
      float4 w[6];
#pragma unroll
      for (int u = 0; u < 6; ++u) w[u] = __ldcg(reinterpret_cast<const float4*>(pb + (pp + u) * stride));
#pragma unroll
      for (int u = 0; u < 6; ++u) {
        v.x += w[u].x; v.y += w[u].y; v.z += w[u].z; v.w += w[u].w;
      }
    }
    for (; pp < p1; ++pp) {
      const float4 w = __ldcg(reinterpret_cast<const float4*>(pb + pp * stride));
      v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
    }
  }
  gsum[q][col] = v;
  __syncthreads();
  if (q == 0 && i < st.block) {
    float4 tot = gsum[0][col];
#pragma unroll
    for (int g = 1; g < kRedGroups; ++g) {
      const float4 u = gsum[g][col];
      tot.x += u.x; tot.y += u.y; tot.z += u.z; tot.w += u.w;
    }
    st4(st.grads + int64_t(k) * st.block + i, tot);
    finite = isfinite(tot.x) && isfinite(tot.y) && isfinite(tot.z) && isfinite(tot.w);
  }
  const bool all_finite = __syncthreads_and(finite);
  finalize_model(st, k, all_finite, ch == 0, red_smem, st.R * 3, !st.ls_sep);
}

// Pairwise-summation leaves of an R-row column (host-computed once per call).
struct LeafTable {
  int n;
  int start[64], len[64];
  int n_ops;
  unsigned char ops[128];  // postfix of pairwise_combine: 0 = push the next leaf sum, 1 = add the top two
};

// postfix program of pairwise_combine(n) (vm_common.cuh): leaves (n <= 128)
// push, inner nodes add their left and right results in that order
void combine_program(int64_t n, LeafTable& lt) {
  if (n <= 128) {
    lt.ops[lt.n_ops++] = 0;
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  combine_program(n2, lt);
  combine_program(n - n2, lt);
  lt.ops[lt.n_ops++] = 1;
}

// Loss sums of a tensor-core stack's models: one CTA per (model, loss term):
// the column is staged in smem, each leaf of numpy's pairwise recursion is
// summed by its own thread, and thread 0 combines the leaves in the
// recursion's order (same bits as pairwise_sum over the column).  Runs on a
// second branch concurrently with the partial reduce and Adam.
__global__ void __launch_bounds__(128) loss_sums_kernel(const __grid_constant__ KParams p, int si,
                                                        const __grid_constant__ LeafTable lt) {
  extern __shared__ __align__(16) float ls_col[];
  __shared__ float lf_sum[64];
  const unsigned long long t0 = p.trace ? vm_gtime() : 0;
  const KStack& st = p.s[si];
  const int k = blockIdx.x, j = blockIdx.y, tid = threadIdx.x, R = st.R;
  const float* terms = st.ray_terms + int64_t(k) * R * 3;
  const int live = st.model_rays ? min(st.model_rays[k], R) : R;  // padding rows sum as 0 (config 3)
  for (int r0 = 0; r0 < R; r0 += 8 * 128) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = r0 + u * 128 + tid;
      v[u] = r < live ? __ldcg(terms + int64_t(r) * 3 + j) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = r0 + u * 128 + tid;
      if (r < R) ls_col[r] = v[u];
    }
  }
  __syncthreads();
  if (tid < lt.n) lf_sum[tid] = pairwise_sum_leaf([&](int64_t r) { return ls_col[r]; }, lt.start[tid], lt.len[tid]);
  __syncthreads();
  if (tid == 0) {
    // the combine as a flat postfix program (no recursion): same additions,
    // same order as pairwise_combine
    float stk[8];
    int sp = 0, next = 0;
    for (int o = 0; o < lt.n_ops; ++o) {
      if (lt.ops[o] == 0) {
        stk[sp++] = lf_sum[next++];
      } else {
        const float b = stk[--sp];
        stk[sp - 1] = __fadd_rn(stk[sp - 1], b);
      }
    }
    const float sum = stk[0];
    st.losses[int64_t(k) * 3 + j] = sum;
    if (!isfinite(sum)) atomicMin(&st.status[1], k);
    if (p.trace) vm_trace_rec(p.trace, 7, t0);
  }
}

template <int H, int L, int MODE>
__device__ void run_item(const KStack& st, int item, float* smem) {
  using Cfg = TeamCfg<H>;
  constexpr int T = Cfg::T, OW = Cfg::OW, NTEAMS = kWarps / T;
  using WG = WarpGrads<H, L>;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int team = warp / T, wt = warp % T;
  const int o0 = wt * OW;

  const int k = item / st.P, split = item % st.P;
  const int kg = st.model_base + k;
  float* sW = smem;
  float* base = smem + st.w_floats + team * st.team_floats;
  float* E = base;
  float* Abuf = E + st.Dp * kLD;               // (L-1) hidden buffers of H rows
  float* O = Abuf + (L - 1) * H * kLD;         // 4 rows
  float* Tsc = O + 4 * kLD;                    // 32
  float* tS = Tsc + kSB;                       // 32

  load_weights<H, L>(st, st.params + int64_t(k) * st.block, sW);
  __syncthreads();

  // block range of this item
  int64_t gs_model;  // first sample of the model
  int nblk_model, S = st.S, G = st.G;
  if (MODE == kTrain) {
    gs_model = int64_t(k) * st.R * S;
    nblk_model = (st.R + G - 1) / G;
  } else {
    gs_model = int64_t(k) * st.N;
    nblk_model = int((st.N + kSB - 1) / kSB);
  }
  const int bps = (nblk_model + st.P - 1) / st.P;
  const int blk0 = split * bps, blk1 = min(nblk_model, blk0 + bps);

  WG acc;
  acc.zero();

  for (int blk = blk0 + team; blk < blk1; blk += NTEAMS) {
    int ns, nr = 0, r_begin = 0;
    int64_t gs0;
    if (MODE == kTrain) {
      r_begin = blk * G;
      nr = min(G, st.R - r_begin);
      ns = nr * S;
      gs0 = gs_model + int64_t(r_begin) * S;
    } else {
      gs0 = gs_model + int64_t(blk) * kSB;
      { const int64_t rem = st.N - int64_t(blk) * kSB; ns = int(rem < kSB ? rem : kSB); }
    }
    load_block(st, k, gs0, ns, E, tS, wt * 32 + lane, T * 32, MODE == kTrain);
    team_sync(team, T);

    // ---------------- forward ----------------
    float* X = E;
    for (int l = 0; l < L - 1; ++l) {
      float* Y = Abuf + l * H * kLD;
      if (l == 0)
        fwd_layer<OW, false, 0>(sW + st.w_off[0], st.fi0, sW + st.b_off[0], X, st.fi0, Y, o0, lane);
      else
        fwd_layer<OW, true, H>(sW + st.w_off[l], H, sW + st.b_off[l], X, H, Y, o0, lane);
      team_sync(team, T);
      X = Y;
    }
    if (wt == 0) fwd_out<H>(sW + st.w_off[L - 1], sW + st.b_off[L - 1], X, O, lane);
    team_sync(team, T);

    if (MODE == kForward) {
      for (int s = wt * 32 + lane; s < ns * 4; s += T * 32) {
        const int smp = s >> 2, ch = s & 3;
        const float v = O[ch * kLD + smp];
        if (ch == 0) st.occ_out[gs0 + smp] = v;
        else st.col_out[(gs0 + smp) * 3 + ch - 1] = v;
      }
      team_sync(team, T);
      continue;
    }

    // ---------------- render + loss (train) / external grads (backward) -----
    if (wt == 0) {
      // zero the pad samples' output grads
      if (lane >= ns) {
#pragma unroll
        for (int c = 0; c < 4; ++c) O[c * kLD + lane] = 0.f;
      }
      if (MODE == kTrain) {
        if (lane < nr) {
          const int r = r_begin + lane;
          const int sb = lane * S;
          const int64_t rg = int64_t(k) * st.R + r;
          RayTargets tg;
          tg.depth = st.tdepth[rg];
          tg.colour[0] = st.tcol[rg * 3 + 0];
          tg.colour[1] = st.tcol[rg * 3 + 1];
          tg.colour[2] = st.tcol[rg * 3 + 2];
          tg.mask = st.tmask[rg] != 0;
          tg.valid = st.valid[rg] != 0;
          tg.ok = st.ok[rg] != 0;
          RayLossGrad lg;
          if (S == 10) {  // register-resident chain, same operation order
            constexpr int NS = 10;
            float o[NS], cl[3][NS], tv[NS];
#pragma unroll
            for (int i = 0; i < NS; ++i) {
              o[i] = O[sb + i];
              tv[i] = tS[sb + i];
#pragma unroll
              for (int c = 0; c < 3; ++c) cl[c][i] = O[(1 + c) * kLD + sb + i];
            }
            lg = render_ray_fixed<NS>(o, cl, tv, tg, st.wc, st.wo);
#pragma unroll
            for (int i = 0; i < NS; ++i) {
              O[sb + i] = o[i];
#pragma unroll
              for (int c = 0; c < 3; ++c) O[(1 + c) * kLD + sb + i] = cl[c][i];
            }
          } else {
            auto occ = [&](int i) { return O[sb + i]; };
            auto col = [&](int i, int c) { return O[(1 + c) * kLD + sb + i]; };
            auto tt = [&](int i) { return tS[sb + i]; };
            render_ray_forward(S, occ, col, tt, [&](int i, float v) { Tsc[sb + i] = v; });
            const RayFwd f = render_ray_sums(S, occ, col, tt, [&](int i) { return Tsc[sb + i]; });
            lg = ray_loss_grad(f, tg, st.wc, st.wo);
            // backward writes dz (sigmoid'd) in place of the outputs; it walks
            // samples from the last to the first, reading only sample i >= cur.
            render_ray_backward(S, occ, col, tt, [&](int i) { return Tsc[sb + i]; }, lg.dO, lg.dD, lg.dC,
                                [&](int i, float d_occ, const float* d_col) {
                                  const float o = O[sb + i];
                                  O[sb + i] = __fmul_rn(__fmul_rn(d_occ, o), __fsub_rn(1.0f, o));
#pragma unroll
                                  for (int c = 0; c < 3; ++c) {
                                    const float cv = O[(1 + c) * kLD + sb + i];
                                    O[(1 + c) * kLD + sb + i] = __fmul_rn(__fmul_rn(d_col[c], cv), __fsub_rn(1.0f, cv));
                                  }
                                });
          }
          st.ray_terms[rg * 3 + 0] = lg.l_depth;
          st.ray_terms[rg * 3 + 1] = lg.l_colour;
          st.ray_terms[rg * 3 + 2] = lg.l_occ;
        }
      } else {  // kBackward: dz from caller's output grads (models.py:380-382)
        if (lane < ns) {
          const int64_t g = gs0 + lane;
          const float o = O[lane];
          O[lane] = (st.gocc[g] * o) * (1.0f - o);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const float cv = O[(1 + c) * kLD + lane];
            O[(1 + c) * kLD + lane] = (st.gcol[g * 3 + c] * cv) * (1.0f - cv);
          }
        }
      }
    }
    team_sync(team, T);

    // ---------------- backward ----------------
    {
      float* Alast = Abuf + (L - 2) * H * kLD;
      // output layer: dW (column slice of this warp) + db, then dz into Alast
      dw_acc<1, WG::NQL>(acc.wl, O, 0, Alast, o0, WG::NQL, lane);
      if (wt == 0 && lane < 4) {
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < kSB; q += 4) {
          const float4 v = ld4(O + lane * kLD + q);
          s += (v.x + v.y) + (v.z + v.w);
        }
        acc.bl += s;
      }
      __syncwarp();
      dx_layer<OW, 4, H>(sW + st.w_off[L - 1], O, Alast, o0, lane);
      team_sync(team, T);
    }
#pragma unroll
    for (int l = L - 2; l >= 1; --l) {
      float* Gl = Abuf + l * H * kLD;        // dz of layer l (rows o)
      float* Xl = Abuf + (l - 1) * H * kLD;  // input of layer l
      dw_acc<WG::NJ, WG::NQH>(acc.wh[l - 1 < 0 ? 0 : l - 1], Gl, o0, Xl, 0, WG::NQH, lane);
      acc.bh[l] += db_acc<OW>(Gl, o0, lane);
      team_sync(team, T);
      dx_layer<OW, H, H>(sW + st.w_off[l], Gl, Xl, o0, lane);
      team_sync(team, T);
    }
    dw_acc<WG::NJ, WG::NQ0>(acc.w0, Abuf, o0, E, 0, st.Dp / 8, lane);
    acc.bh[0] += db_acc<OW>(Abuf, o0, lane);
    team_sync(team, T);
  }

  if (MODE == kForward) return;

  // ---------------- gradient write-out ----------------
  // Destination: grads[k] when the model has one CTA, else partials[item].
  float* gdst = (st.P == 1) ? st.grads + int64_t(k) * st.block
                            : st.partials + (int64_t(k) * st.P + split) * st.block;
  // combine bias partial sums across the sample halves (OW == 16)
#pragma unroll
  for (int l = 0; l < L - 1; ++l) {
    if (OW == 16) acc.bh[l] += __shfl_xor_sync(0xffffffffu, acc.bh[l], 16);
  }
  auto emit = [&](float* dst, bool add) {
    const int r = lane >> 3, c = lane & 7;
    auto put = [&](int idx, float v) {
      if (add) dst[idx] += v;
      else dst[idx] = v;
    };
    // layer 0
#pragma unroll
    for (int j = 0; j < WG::NJ; ++j)
#pragma unroll
      for (int q = 0; q < WG::NQ0; ++q) {
        const int o = o0 + r + 4 * j, i = c + 8 * q;
        if (i < st.fi0) put(st.w_off[0] + o * st.fi0 + i, acc.w0[j][q]);
      }
    // hidden layers
#pragma unroll
    for (int h = 0; h < WG::NH; ++h)
#pragma unroll
      for (int j = 0; j < WG::NJ; ++j)
#pragma unroll
        for (int q = 0; q < WG::NQH; ++q) {
          const int o = o0 + r + 4 * j, i = c + 8 * q;
          put(st.w_off[h + 1] + o * H + i, acc.wh[h][j][q]);
        }
    // output layer
#pragma unroll
    for (int q = 0; q < WG::NQL; ++q) put(st.w_off[L - 1] + r * H + o0 + c + 8 * q, acc.wl[0][q]);
    // biases
#pragma unroll
    for (int l = 0; l < L - 1; ++l)
      if (lane < OW) put(st.b_off[l] + o0 + lane, acc.bh[l]);
    if (wt == 0 && lane < 4) put(st.b_off[L - 1] + lane, acc.bl);
  };

  if (NTEAMS == 1) {
    emit(gdst, false);
  } else if (st.block <= st.team_floats) {
    // each team writes its whole partial block into its own (now idle)
    // activation region; then all threads add the NTEAMS regions in team
    // order (deterministic, same sum order as the sequential variant below)
    float* mine = smem + st.w_floats + team * st.team_floats;
    emit(mine, false);
    __syncthreads();
    const float* r0 = smem + st.w_floats;
    for (int i = tid; i < st.block / 4; i += kThreads) {
      float4 v = ld4(r0 + 4 * i);
#pragma unroll
      for (int t = 1; t < NTEAMS; ++t) {
        const float4 u = ld4(r0 + t * st.team_floats + 4 * i);
        v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
      }
      st4(gdst + 4 * i, v);
    }
  } else {
    __syncthreads();  // every team is done with the weights: reuse sW as staging
    for (int t = 0; t < NTEAMS; ++t) {
      if (team == t) emit(sW, t > 0);
      __syncthreads();
    }
    for (int i = tid; i < st.block / 4; i += kThreads) st4(gdst + 4 * i, ld4(sW + 4 * i));
  }

  // ---------------- per-model finalisation ---------
  // A model split over P CTAs (fixed chunks of its own blocks, so the split
  // never depends on K) is summed by the CTA that finishes last (atomic
  // ticket), partials in chunk order -- deterministic and identical for the
  // vectorised and the sequential paths -- then finalised right here.
  bool finite = true;
  const float* gk = st.grads + int64_t(k) * st.block;
  if (st.P > 1) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&st.counters[k], 1) == st.P - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float* pb = st.partials + int64_t(k) * st.P * st.block;
    float* gw = st.grads + int64_t(k) * st.block;
    for (int i = tid; i < st.block / 4; i += kThreads) {
      float4 v = __ldcg(reinterpret_cast<const float4*>(pb + 4 * i));
      for (int u = 1; u < st.P; ++u) {
        const float4 w = __ldcg(reinterpret_cast<const float4*>(pb + int64_t(u) * st.block + 4 * i));
        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
      }
      st4(gw + 4 * i, v);
      finite &= isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
    }
    if (tid == 0) st.counters[k] = 0;  // ready for the next launch (graph replay)
  } else {
    __syncthreads();
    for (int i = tid; i < st.block / 4; i += kThreads) {
      const float4 v = ld4(gk + 4 * i);
      finite &= isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
    }
  }
  const bool all_finite = __syncthreads_and(finite);
  if (MODE == kBackward) return;
  // the team activation buffers are free now: stage per-ray terms there
  finalize_model(st, k, all_finite, true, smem + st.w_floats, NTEAMS * st.team_floats);
}

template <int H0, int L0, int H1, int L1, int MODE>
__global__ void __launch_bounds__(kThreads, (H0 <= 32 && H1 <= 32) ? 2 : 1) mlp_kernel(const __grid_constant__ KParams p) {
  extern __shared__ __align__(16) float smem[];
  const int b = blockIdx.x;
  if (p.n_stacks == 1 || b < p.s[1].item_base) {
    run_item<H0, L0, MODE>(p.s[0], b, smem);
  } else {
    if constexpr (H1 > 0) run_item<H1, L1, MODE>(p.s[1], b - p.s[1].item_base, smem);
  }
}

// Adam over every active model of every stack; stack s is skipped when any
// stack <= s reported a non-finite gradient, or any stack < s a non-finite
// loss (trainer.py:368-388 raises before training the next stack).
struct AdamStack {
  float* P; float* M; float* V;
  const float* G;
  int64_t* step;
  const uint8_t* upd;
  const float2* corr;
  int block, K, chunks, item_base;
  AdamConsts a;
  int32_t* status;
};
struct AdamParams {
  AdamStack s[2];
  int n_stacks;
  unsigned long long* trace;
};

__global__ void __launch_bounds__(256) adam_train_kernel(const __grid_constant__ AdamParams p, int block_offset) {
  const unsigned long long t_start = p.trace ? vm_gtime() : 0;
  // programmatic launch behind the partial reduce: wait for its gradients
  // (a no-op for an ordinary launch)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  struct Rec {  // schedule record at every exit
    const AdamParams& p;
    unsigned long long t;
    __device__ ~Rec() {
      if (p.trace && threadIdx.x == 0) vm_trace_rec(p.trace, 4, t);
    }
  } rec{p, t_start};
  int b = blockIdx.x + block_offset, si = 0;
  if (p.n_stacks > 1 && b >= p.s[1].item_base) si = 1;
  const AdamStack& s = p.s[si];
  b -= s.item_base;
  const int k = b / s.chunks, ch = b % s.chunks;
  const int64_t base = int64_t(k) * s.block;
  const int i = (ch * 256 + threadIdx.x) * 4;
  // the element loads are issued before the (dependent) status / mask / bias
  // correction reads, so one memory latency covers them all; nothing is
  // written unless the model updates
  const bool in = i < s.block;
  float4 pv, mv, vv, gv;
  if (in) {
    pv = ld4(s.P + base + i);
    mv = ld4(s.M + base + i);
    vv = ld4(s.V + base + i);
    gv = __ldcg(reinterpret_cast<const float4*>(s.G + base + i));
  }
  bool skip = s.status[0] != 0x7f7f7f7f;
  for (int j = 0; j < si; ++j) skip |= (p.s[j].status[0] != 0x7f7f7f7f) || (p.s[j].status[1] != 0x7f7f7f7f);
  if (k == 0 && ch == 0 && threadIdx.x == 0) s.status[2] = skip ? 0 : 1;
  if (skip || !s.upd[k]) return;
  const float2 c = s.corr[k];
  if (in) {
    adam_elem(pv.x, mv.x, vv.x, gv.x, c.x, c.y, s.a);
    adam_elem(pv.y, mv.y, vv.y, gv.y, c.x, c.y, s.a);
    adam_elem(pv.z, mv.z, vv.z, gv.z, c.x, c.y, s.a);
    adam_elem(pv.w, mv.w, vv.w, gv.w, c.x, c.y, s.a);
    st4(s.P + base + i, pv);
    st4(s.M + base + i, mv);
    st4(s.V + base + i, vv);
  }
  if (ch == 0 && threadIdx.x == 0) s.step[k] += 1;
#ifdef VM_TC_DEBUG
  if (threadIdx.x == 0) atomicAdd(&vm_tc_dbg[66], 1);
#endif
}

// ------------------------------------------------------------------ host side

struct Instance {
  int H, L;
};

inline size_t smem_bytes(const KStack& s) {
  const int nteams = kWarps / (s.H == 32 ? TeamCfg<32>::T : (s.H == 64 ? TeamCfg<64>::T : TeamCfg<128>::T));
  return size_t(s.w_floats + nteams * s.team_floats) * sizeof(float) + 64;
}

static int fill_stack(const VmStack& vs, KStack& ks, VmLayout& L) {
  int rc = compute_layout(vs.arch, L);
  if (rc) return rc;
  if (vs.arch.input_dim > kDpMax) return VM_ERR_UNSUPPORTED;
  std::memset(&ks, 0, sizeof(ks));
  ks.H = L.hidden_pad;
  ks.L = L.n_layers;
  ks.D = vs.arch.input_dim;
  ks.Dp = round_up(ks.D, 8);
  ks.fi0 = L.fi_pad[0];
  ks.block = int(L.block);
  ks.w_floats = round_up(ks.block, 32);
  ks.team_floats = (ks.Dp + (ks.L - 1) * ks.H + 4) * kLD + 2 * kSB;
  for (int l = 0; l < L.n_layers; ++l) {
    ks.w_off[l] = int(L.w_off[l]);
    ks.b_off[l] = int(L.b_off[l]);
  }
  ks.params = vs.params;
  ks.frozen = vs.frozen;
  ks.step = vs.step;
  ks.corr1 = vs.corr1;
  ks.corr2 = vs.corr2;
  ks.corr_len = vs.corr_len;
  ks.beta1 = vs.beta1;
  ks.beta2 = vs.beta2;
  ks.K = vs.count;
  return VM_OK;
}

using KernelFn = void (*)(KParams);

template <int MODE>
static KernelFn pick_kernel(int H0, int L0, int H1, int L1) {
#define VM_SINGLE(h, l) \
  if (H1 == 0 && H0 == h && L0 == l) return mlp_kernel<h, l, 0, 0, MODE>;
#define VM_PAIR(h0, l0, h1, l1) \
  if (H0 == h0 && L0 == l0 && H1 == h1 && L1 == l1) return mlp_kernel<h0, l0, h1, l1, MODE>;
  VM_SINGLE(32, 2) VM_SINGLE(32, 3) VM_SINGLE(32, 4) VM_SINGLE(32, 5)
  VM_SINGLE(64, 2) VM_SINGLE(64, 3) VM_SINGLE(64, 4)
  VM_SINGLE(128, 2) VM_SINGLE(128, 3) VM_SINGLE(128, 4)
  if constexpr (MODE == kTrain) {
    VM_PAIR(32, 4, 128, 4) VM_PAIR(32, 4, 32, 4) VM_PAIR(32, 3, 32, 3) VM_PAIR(32, 4, 64, 4)
  }
#undef VM_SINGLE
#undef VM_PAIR
  return nullptr;
}

static int launch_mlp(KernelFn fn, const KParams& p, int grid, size_t smem, cudaStream_t s) {
  if (smem > 227 * 1024) {
    set_error("vm: model too large for shared memory (block + activation tiles > 227 KB)");
    return VM_ERR_UNSUPPORTED;
  }
  VM_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(smem)));
  void* args[] = {const_cast<KParams*>(&p)};
  VM_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(fn), dim3(grid), dim3(kThreads), args, smem, s));
  return VM_OK;
}

// Work split: a model's ray blocks are cut into fixed chunks of
// VM_KF_CHUNK blocks (default 8: two per 2-warp team of a CTA), one CTA per
// chunk.  The chunking depends only on the model's own ray count, never on
// K, so a model's gradient summation order -- and therefore its bits -- does
// not depend on which other models share the launch (vectorised ==
// sequential, test_trainer.py:117-132), while the grid is a few hundred small
// CTAs that the block scheduler spreads over all 148 SMs (two per SM) and
// that fill the SMs the tensor-core kernel leaves free.  A tensor-core stack
// is one CTA per 128-row tile instead.
int chunk_blocks() {
  static const int v = [] {
    const char* e = std::getenv("VM_KF_CHUNK");
    const int c = e ? std::atoi(e) : 8;
    return c > 0 ? c : 8;
  }();
  return v;
}
static int choose_splits(const KStack* ks, int n, int* P) {
  for (int i = 0; i < n; ++i) {
    if (ks[i].tc) {
      const int g = tck::kTM / ks[i].S;
      P[i] = std::max(1, (ks[i].R + g - 1) / g);
      continue;
    }
    const int nblk = (ks[i].R + ks[i].G - 1) / ks[i].G;
    P[i] = std::max(1, (nblk + chunk_blocks() - 1) / chunk_blocks());
  }
  return VM_OK;
}

}  // namespace vm

using namespace vm;

namespace {
// Optional per-launch CUDA-event timing of the fused kernel (bench.py reads
// it to report the kernel's roofline fraction from the timed region itself).
struct KernelProfiler {
  bool on = false;
  long kernels = 0;  // every kernel launched by vm_train_step / vm_sample while on
  std::vector<cudaEvent_t> ev;  // start/stop pairs
  std::vector<int> tag;         // per pair: 0 = MLP phase, 1 = FFMA kernel (KF), 2 = tensor-core branch (KT),
                                // 3 = partial reduce + Adam
  size_t used = 0;
  cudaEvent_t get() {
    if (used == ev.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    return ev[used++];
  }
  void pair(cudaEvent_t& a, cudaEvent_t& b, int t) {
    a = get();
    b = get();
    if (tag.size() < used / 2) tag.resize(used / 2);
    tag[used / 2 - 1] = t;
  }
} g_prof;

struct TrainPlan {
  KParams kp;
  AdamParams ap;
  int grid, adam_grid;
  size_t smem;
  size_t ws_bytes;
  // workspace offsets
  size_t off_grads[2], off_part[2], off_terms[2], off_cnt[2], off_upd[2], off_corr[2], off_img[2];
  size_t off_queue;
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// The specialised hidden-32 kernel (vm_kf32.cu) is the default for the
// object stacks; VM_KF32=0 selects the generic FFMA kernel (A/B, parity).
bool kf32_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VM_KF32");
    return !(e && e[0] == '0');
  }();
  return on;
}

// VM_KH=1 runs hidden-32 object stacks on the warp-level tensor path (KH32,
// 3xTF32 mma.sync) instead of the FP32 FFMA kernel KF32.  Off by default:
// measured on B200 at config 2 it is no faster standalone (65.6 vs 65.1 us,
// ncu) and its one-CTA-per-SM footprint slows the concurrent KT phase
// (0.183 vs 0.175 ms/step); see DESIGN.md "KH32".
bool kh32_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VM_KH");
    return e && e[0] == '1';
  }();
  return on;
}

// Hidden-128 forward-only evaluation (vm_forward: inference grids and view
// rays) on the tensor cores; VM_TC_FWD=0 keeps it on the FFMA forward kernel.
int tc_fwd_mode() {  // 0: FFMA forward, 1: one tile in flight, 2 (default): two
  static const int m = [] {
    const char* e = std::getenv("VM_TC_FWD");
    return e ? std::atoi(e) : 2;
  }();
  return m;
}
bool tc_fwd_enabled() { return tc_fwd_mode() != 0; }

// The tensor-core path is the default for hidden-128 stacks; VM_TC=0 selects
// the FFMA kernel for them (A/B measurements and the parity cross-check).
bool tc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VM_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

int plan_train(const VmStack* stacks, const VmBatch* batches, int n, TrainPlan& pl) {
  VM_REQUIRE(n >= 1 && n <= 2, "vm_train_step: 1 or 2 stacks supported");
  std::memset(&pl, 0, sizeof(pl));
  pl.kp.n_stacks = n;
  pl.ap.n_stacks = n;
  size_t off = 0;
  int item_base = 0, model_base = 0, adam_base = 0;
  int P[2] = {1, 1};
  for (int i = 0; i < n; ++i) {
    VmLayout L;
    int rc = fill_stack(stacks[i], pl.kp.s[i], L);
    if (rc) {
      set_error("vm_train_step: unsupported architecture");
      return rc;
    }
    KStack& ks = pl.kp.s[i];
    const VmBatch& b = batches[i];
    VM_REQUIRE(b.n_models == stacks[i].count, "vm_train_step: batch leading axis != params.count");
    VM_REQUIRE(b.input_dim == stacks[i].arch.input_dim, "vm_train_step: encoding dim mismatch");
    VM_REQUIRE(b.n_points >= 1 && b.n_points <= kSB, "vm_train_step: points per ray must be in [1, 32]");
    VM_REQUIRE(b.encoded != nullptr || (b.points != nullptr && b.pe_scale != nullptr),
               "vm_train_step: encoded input or points + pe_scale required");
    ks.R = b.n_rays;
    ks.S = b.n_points;
    ks.G = kSB / b.n_points;
    ks.enc = b.encoded;
    ks.pts = b.encoded ? nullptr : b.points;
    ks.pe_scale = b.pe_scale;
    ks.n_freq = (stacks[i].arch.input_dim % 6 == 3) ? (stacks[i].arch.input_dim - 3) / 6 : stacks[i].arch.input_dim / 6;
    ks.include_input = stacks[i].arch.input_dim % 6 == 3;
    ks.t = b.t;
    ks.tdepth = b.target_depth;
    ks.tcol = b.target_colour;
    ks.tmask = b.target_mask;
    ks.valid = b.valid_depth;
    ks.ok = b.ray_ok;
    ks.chunk = chunk_blocks();
    ks.model_rays = b.model_rays;
    ks.items = b.model_rays ? b.work_items : nullptr;
    ks.n_items = ks.items ? b.n_work_items : 0;
    VM_REQUIRE(!ks.items || ks.n_items >= 0, "vm_train_step: bad work-item count");
    ks.tc = tc_enabled() && ks.H == 128 && ks.L == 4 && ks.D <= tck::kK0 && ks.S <= 32 ? 1 : 0;
    {
      int64_t st64[64];
      int len[64];
      ks.ls_sep = ks.tc && pairwise_leaves(ks.R, st64, len, 64) <= 64 ? 1 : 0;
    }
  }
  choose_splits(pl.kp.s, n, P);
  for (int i = 0; i < n; ++i) {
    KStack& ks = pl.kp.s[i];
    ks.P = P[i];
    ks.item_base = item_base;
    ks.model_base = model_base;
    item_base += ks.items ? ks.n_items : ks.K * ks.P;
    model_base += ks.K;
    const size_t K = size_t(ks.K);
    pl.off_grads[i] = off; off = align_up(off + K * ks.block * 4, 256);
    pl.off_part[i] = off;  off = align_up(off + (ks.P > 1 ? K * ks.P * ks.block * 4 : 0), 256);
    pl.off_terms[i] = off; off = align_up(off + K * size_t(ks.R) * 3 * 4, 256);
    pl.off_cnt[i] = off;   off = align_up(off + K * 4, 256);
    pl.off_upd[i] = off;   off = align_up(off + K, 256);
    pl.off_corr[i] = off;  off = align_up(off + K * 8, 256);
    pl.off_img[i] = off;   off = align_up(off + (ks.tc ? K * tck::Img<128, 4>::total * 4 : 0), 256);
    if (!ks.tc) pl.smem = std::max(pl.smem, smem_bytes(ks));
    AdamStack& as = pl.ap.s[i];
    as.P = stacks[i].params;
    as.M = stacks[i].m;
    as.V = stacks[i].v;
    as.step = stacks[i].step;
    as.block = ks.block;
    as.K = ks.K;
    as.chunks = (ks.block / 4 + 255) / 256;
    as.item_base = adam_base;
    as.a = adam_consts(stacks[i]);
    adam_base += ks.K * as.chunks;
  }
  pl.off_queue = off;
  off = align_up(off + 4, 256);
  pl.grid = item_base;
  pl.adam_grid = adam_base;
  pl.ws_bytes = off;
  return VM_OK;
}
struct StepInit {
  int32_t* status;
  int n_status;
  int* cnt[2];
  int n_cnt[2];
  int* queue;
  unsigned long long* trace;
};
__global__ void step_init_kernel(const __grid_constant__ StepInit in) {
  const unsigned long long t0 = in.trace ? vm_gtime() : 0;
  for (int i = threadIdx.x; i < in.n_status; i += blockDim.x) in.status[i] = 0x7f7f7f7f;
  for (int j = 0; j < 2; ++j)
    for (int i = threadIdx.x; i < in.n_cnt[j]; i += blockDim.x) in.cnt[j][i] = 0;
  if (threadIdx.x == 0) {
    *in.queue = 0;
    if (in.trace) vm_trace_rec(in.trace, 8, t0);
  }
}

// VM_PDL=0 disables programmatic dependent launch (A/B).
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Partial reduce of a tensor-core stack (its tiles' weight-gradient blocks;
// FFMA stacks reduce in-kernel).  Runs on the tensor-core branch's stream so
// it overlaps the FFMA kernel.
int launch_reduce(const TrainPlan& pl, int i, cudaStream_t s) {
  {
    const KStack& ks = pl.kp.s[i];
    if (ks.P <= 1 || ks.K == 0 || !ks.tc) return VM_OK;
    const int cf = red_chunk_floats(ks.P);
    const int grid = ks.K * ((ks.block + cf - 1) / cf);
    const int red_smem = ks.R * 3 * 4;
    if (red_smem > 48 * 1024)
      VM_CUDA(cudaFuncSetAttribute(reduce_partials_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, red_smem));
    // programmatic dependent launch (Blackwell/Hopper): the reduce grid is
    // scheduled while KT drains and released by griddepcontrol.wait, hiding
    // the launch gap on the step's critical path
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kRedThreads);
    cfg.dynamicSmemBytes = red_smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    VM_CUDA(cudaLaunchKernelEx(&cfg, reduce_partials_kernel, pl.kp, i));
    if (g_prof.on) g_prof.kernels += 1;
  }
  return VM_OK;
}

// One Adam launch over every stack.  Adam of stack i reads the status words
// of stacks < i (trainer.py:368-388 raise order).
// Adam over the CTA range [b0, b1) of the plan's Adam grid (stack order).
int launch_adam(const TrainPlan& pl, cudaStream_t s, int b0 = 0, int b1 = -1) {
  if (b1 < 0) b1 = pl.adam_grid;
  if (b1 <= b0) return VM_OK;
  adam_train_kernel<<<b1 - b0, 256, 0, s>>>(pl.ap, b0);
  VM_CUDA(cudaGetLastError());
  if (g_prof.on) g_prof.kernels += 1;
  return VM_OK;
}
}  // namespace

extern "C" int vm_work_items(const int32_t* model_rays, int32_t n_models, int32_t n_points, int32_t* items,
                             int32_t capacity, int32_t* n_items) {
  VM_REQUIRE(model_rays && n_items && n_models >= 0, "vm_work_items: null argument");
  VM_REQUIRE(n_points >= 1 && n_points <= kSB, "vm_work_items: points per ray must be in [1, 32]");
  const int G = kSB / n_points, chunk = chunk_blocks();
  int64_t n = 0;
  for (int k = 0; k < n_models; ++k) {
    VM_REQUIRE(model_rays[k] >= 0, "vm_work_items: negative ray count");
    const int nblk = (model_rays[k] + G - 1) / G;
    const int pk = std::max(1, (nblk + chunk - 1) / chunk);
    for (int c = 0; c < pk; ++c, ++n) {
      if (items && n < capacity) {
        items[2 * n] = k;
        items[2 * n + 1] = c;
      }
    }
  }
  VM_REQUIRE(n <= INT32_MAX, "vm_work_items: too many items");
  *n_items = int32_t(n);
  VM_REQUIRE(!items || n <= capacity, "vm_work_items: capacity too small");
  return VM_OK;
}

// Whether the fused kernels (KF32 / generic FFMA, KT) take every stack of
// this call; otherwise the layered path (vm_layered.cu) trains the stacks the
// fused kernels lack.
static bool fused_supported(const VmStack* stacks, const VmBatch* batches, int n) {
  if (layered_forced()) return false;
  TrainPlan pl;
  if (plan_train(stacks, batches, n, pl)) return false;
  KParams kf;
  std::memset(&kf, 0, sizeof(kf));
  for (int i = 0; i < n; ++i)
    if (!pl.kp.s[i].tc) kf.s[kf.n_stacks++] = pl.kp.s[i];
  if (kf.n_stacks == 0) return true;
  if (kf32_enabled() && kf32_supported(kf)) return true;
  return pick_kernel<kTrain>(kf.s[0].H, kf.s[0].L, kf.n_stacks > 1 ? kf.s[1].H : 0,
                             kf.n_stacks > 1 ? kf.s[1].L : 0) != nullptr &&
         pl.smem <= 227 * 1024;
}

// 0: every stack fused; 1: stack 0 fused, stack 1 layered; 2: all layered
// (a layered stack 0 would have to precede a fused stack 1, whose kernels
// read stack 0's status words inside the same fused launch sequence).
static int train_route(const VmStack* stacks, const VmBatch* batches, int n) {
  if (fused_supported(stacks, batches, n)) return 0;
  if (n == 2 && fused_supported(stacks, batches, 1)) return 1;
  return 2;
}

static size_t fused_bytes(const VmStack* stacks, const VmBatch* batches, int n) {
  TrainPlan pl;
  if (plan_train(stacks, batches, n, pl)) return 0;
  return pl.ws_bytes;
}

extern "C" size_t vm_train_workspace_bytes(const VmStack* stacks, const VmBatch* batches, int n_stacks) {
  switch (train_route(stacks, batches, n_stacks)) {
    case 0: return fused_bytes(stacks, batches, n_stacks);
    case 1: return align_up(fused_bytes(stacks, batches, 1), 256) + layered_train_bytes(stacks, batches, 2, 1);
    default: return layered_train_bytes(stacks, batches, n_stacks, 0);
  }
}

// VM_TRACE=1: every vm_train_step records (kind 1 = FFMA item, 2 = KT tile,
// SM id, start/end globaltimer ns) into a device buffer read by vm_trace_read.
namespace {
unsigned long long* g_trace = nullptr;
}  // namespace

// The trace buffer (allocated on first use when VM_TRACE=1, else null); the
// record counter is reset by vm_trace_read, so a read returns every record
// since the previous one (e.g. one replayed step graph, sampler included).
unsigned long long* vm::trace_ptr() {
  static const bool on = [] {
    const char* e = std::getenv("VM_TRACE");
    return e && e[0] == '1';
  }();
  if (!on) return nullptr;
  if (!g_trace) {
    if (cudaMalloc(&g_trace, sizeof(unsigned long long) * (1 + 4 * (1 << 16))) != cudaSuccess) return nullptr;
    cudaMemset(g_trace, 0, sizeof(unsigned long long));
  }
  return g_trace;
}
namespace {
unsigned long long* trace_buffer(cudaStream_t) { return vm::trace_ptr(); }
}  // namespace

static int train_fused(const VmStack* stacks, const VmBatch* batches, int n_stacks, VmLossWeights w,
                       float* losses, int32_t* status, void* workspace, size_t workspace_bytes,
                       void* stream) {
  TrainPlan pl;
  int rc = plan_train(stacks, batches, n_stacks, pl);
  if (rc) return rc;
  VM_REQUIRE(workspace_bytes >= pl.ws_bytes, "vm_train_step: workspace too small");
  cudaStream_t s = cudaStream_t(stream);
  char* ws = static_cast<char*>(workspace);
  // one init kernel: status words to the "no failure" pattern, the chunk
  // tickets of the in-kernel partial reductions (the workspace may have held
  // another plan's data) and the persistent kernel's item counter
  {
    StepInit in;
    std::memset(&in, 0, sizeof(in));
    in.status = status;
    in.n_status = 4 * n_stacks;
    for (int i = 0; i < n_stacks; ++i)
      if (!pl.kp.s[i].tc && pl.kp.s[i].K > 0) {
        in.cnt[i] = reinterpret_cast<int*>(ws + pl.off_cnt[i]);
        in.n_cnt[i] = pl.kp.s[i].K;
      }
    in.queue = reinterpret_cast<int*>(ws + pl.off_queue);
    in.trace = trace_ptr();
    step_init_kernel<<<1, 256, 0, s>>>(in);
    VM_CUDA(cudaGetLastError());
    if (g_prof.on) g_prof.kernels += 1;
  }
  int loss_off = 0;
  for (int i = 0; i < n_stacks; ++i) {
    KStack& ks = pl.kp.s[i];
    ks.grads = reinterpret_cast<float*>(ws + pl.off_grads[i]);
    ks.partials = reinterpret_cast<float*>(ws + pl.off_part[i]);
    ks.ray_terms = reinterpret_cast<float*>(ws + pl.off_terms[i]);
    ks.counters = reinterpret_cast<int*>(ws + pl.off_cnt[i]);
    ks.upd = reinterpret_cast<uint8_t*>(ws + pl.off_upd[i]);
    ks.corr = reinterpret_cast<float2*>(ws + pl.off_corr[i]);
    ks.losses = losses + int64_t(loss_off) * 3;
    ks.status = status + 4 * i;
    ks.wc = w.colour;
    ks.wo = w.occupancy;
    loss_off += ks.K;
    AdamStack& as = pl.ap.s[i];
    as.G = ks.grads;
    as.upd = ks.upd;
    as.corr = ks.corr;
    as.status = ks.status;
  }
  if (pl.grid == 0) return VM_OK;
  // FFMA kernel over the stacks KT does not take
  KParams kf;
  std::memset(&kf, 0, sizeof(kf));
  // The FFMA object kernel runs as a persistent grid (two CTAs per SM) pulling
  // work items from a counter: measured 0.171 vs 0.182 ms per config-2 step
  // against one CTA per item; VM_KF_PERSIST=0 restores the latter.
  static const bool kf_persist = [] {
    const char* e = std::getenv("VM_KF_PERSIST");
    return !(e && e[0] == '0');
  }();
  if (kf_persist) kf.queue = reinterpret_cast<int*>(ws + pl.off_queue);
  kf.trace = pl.kp.trace = pl.ap.trace = trace_buffer(s);
  int ff_grid = 0;
  for (int i = 0; i < n_stacks; ++i) {
    if (pl.kp.s[i].tc) continue;
    kf.s[kf.n_stacks++] = pl.kp.s[i];
  }
  KernelFn fn = nullptr;
  const bool use_kf32 = kf.n_stacks > 0 && kf32_enabled() && kf32_supported(kf);
  for (int i = 0; i < kf.n_stacks; ++i) {
    KStack& ks = kf.s[i];
    // only the specialised kernel walks work-item tables; the generic one
    // trains the padding rows too (zero rows: identical results)
    if (!use_kf32) {
      ks.items = nullptr;
      ks.n_items = 0;
    }
    ks.item_base = ff_grid;
    ff_grid += ks.items ? ks.n_items : ks.K * ks.P;
  }
  const bool use_kh32 = use_kf32 && kh32_enabled() && kh32_supported(kf);
  if (kf.n_stacks > 0 && !use_kf32) {
    fn = pick_kernel<kTrain>(kf.s[0].H, kf.s[0].L, kf.n_stacks > 1 ? kf.s[1].H : 0, kf.n_stacks > 1 ? kf.s[1].L : 0);
  }
  if (kf.n_stacks > 0 && !fn && !use_kf32) {
    if (n_stacks == 2) {  // no fused instantiation for this pair: run stacks back to back
      // (Adam of stack 1 still honours stack 0's status because both read it)
      set_error("vm_train_step: unsupported stack pair");
      return VM_ERR_UNSUPPORTED;
    }
    set_error("vm_train_step: no kernel for this architecture");
    return VM_ERR_UNSUPPORTED;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr, kf0 = nullptr, kf1 = nullptr, kt0 = nullptr, kt1 = nullptr;
  if (g_prof.on) {
    g_prof.pair(e0, e1, 0);
    VM_CUDA(cudaEventRecord(e0, s));
  }
  // The tensor-core stacks run on a side stream, concurrently with the FFMA
  // kernel (fork/join with events; both are captured when `s` is capturing).
  // The FFMA kernel is launched right after the fork (then the FFMA stacks'
  // Adam, on the caller's stream); the branch builds KT's pre-split weight
  // image (tc_prep_kernel) and runs KT, whose one-tile-per-SM CTAs take the
  // SMs the first FFMA wave leaves and those it frees, then the partial
  // reduce; the remaining Adam runs after the join.
  // side stream + fork/join events: one set per (host thread, device), so
  // concurrent callers on different threads or devices never share them
  struct SideRes {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, kt_done = nullptr, ls_done = nullptr, kf_done = nullptr;
    cudaStream_t side2 = nullptr;  // loss sums of the tensor-core stacks
  };
  static thread_local SideRes side_res[64];
  int dev = 0;
  VM_CUDA(cudaGetDevice(&dev));
  VM_REQUIRE(dev >= 0 && dev < 64, "vm_train_step: device ordinal out of range");
  cudaStream_t& side = side_res[dev].side;
  cudaEvent_t& ev_fork = side_res[dev].fork;
  cudaEvent_t& ev_join = side_res[dev].join;
  cudaEvent_t& ev_kt = side_res[dev].kt_done;
  cudaEvent_t& ev_ls = side_res[dev].ls_done;
  cudaEvent_t& ev_kf = side_res[dev].kf_done;
  cudaStream_t& side2 = side_res[dev].side2;
  bool forked = false;
  cudaStream_t ts = s;
  using TI = tck::Img<128, 4>;
  auto launch_prep = [&](int i, cudaStream_t st) -> int {
    const KStack& ks = pl.kp.s[i];
    float* img = reinterpret_cast<float*>(ws + pl.off_img[i]);
    tck::tc_prep_kernel<128, 4><<<dim3(TI::n_chunks * 4, ks.K), 256, 0, st>>>(ks, img);
    VM_CUDA(cudaGetLastError());
    if (g_prof.on) g_prof.kernels += 1;
    return VM_OK;
  };
  // Adam of the leading FFMA stacks can run on the caller's stream as soon
  // as KF is done, overlapping the tensor-core branch (their updates never
  // depend on a later stack's status); the rest runs after the join.
  int adam_split = 0;
  for (int i = 0; i < n_stacks && !pl.kp.s[i].tc; ++i)
    adam_split = (i + 1 < n_stacks) ? pl.ap.s[i + 1].item_base : pl.adam_grid;
  bool any_tc = false;
  for (int i = 0; i < n_stacks; ++i) any_tc |= pl.kp.s[i].tc && pl.kp.s[i].K > 0;
  if (!any_tc) adam_split = 0;
  auto launch_kf = [&]() -> int {
    if (!fn && !use_kf32) return VM_OK;
    if (g_prof.on) {
      g_prof.pair(kf0, kf1, 1);
      VM_CUDA(cudaEventRecord(kf0, s));
    }
    const int r = use_kf32 ? (use_kh32 ? launch_kh32(kf, ff_grid, s) : launch_kf32(kf, ff_grid, s))
                           : launch_mlp(fn, kf, ff_grid, pl.smem, s);
    if (r) return r;
    if (g_prof.on) {
      g_prof.kernels += 1;
      VM_CUDA(cudaEventRecord(kf1, s));
    }
    rc = launch_adam(pl, s, 0, adam_split);
    if (rc) return rc;
    if (forked) VM_CUDA(cudaEventRecord(ev_kf, s));
    return VM_OK;
  };
  // launch order: the FFMA kernel goes first (measured 0.195 vs 0.207 ms per
  // graph-replayed config-2 step); VM_KT_FIRST=1 launches KT first instead
  // VM_KT_FIRST=2: KT's weight image is built on the caller's stream before
  // the fork, so KT and KF become ready together and KT (launched first)
  // takes its SMs before KF's CTAs fill the rest
  static const int kt_first_mode = [] {
    const char* e = std::getenv("VM_KT_FIRST");
    return e ? std::atoi(e) : 0;
  }();
  const bool kf_first = kt_first_mode == 0;
  const bool prep_before_fork = kt_first_mode == 2;
  if (prep_before_fork)
    for (int i = 0; i < n_stacks; ++i)
      if (pl.kp.s[i].tc && pl.kp.s[i].K > 0) {
        rc = launch_prep(i, s);
        if (rc) return rc;
      }
  bool kf_done = false;
  for (int i = 0; i < n_stacks; ++i) {
    const KStack& ks = pl.kp.s[i];
    if (!ks.tc || ks.K == 0) continue;
    static const bool no_fork = [] {
      const char* e = std::getenv("VM_NO_FORK");
      return e && e[0] == '1';
    }();
    if (!forked && (fn || use_kf32) && !no_fork) {
      if (!side || !ev_kt) {  // first use may be inside a graph capture: relax the capture mode for the creation
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        VM_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
        if (!side) {
          VM_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
          VM_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
          VM_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        }
        if (!ev_kt) {
          VM_CUDA(cudaEventCreateWithFlags(&ev_kt, cudaEventDisableTiming));
          VM_CUDA(cudaEventCreateWithFlags(&ev_kf, cudaEventDisableTiming));
          VM_CUDA(cudaEventCreateWithFlags(&ev_ls, cudaEventDisableTiming));
          VM_CUDA(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
        }
        VM_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
      }
      VM_CUDA(cudaEventRecord(ev_fork, s));
      VM_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
      forked = true;
      ts = side;
      if (kf_first && !kf_done) {
        rc = launch_kf();
        if (rc) return rc;
        kf_done = true;
      }
    }
    if (g_prof.on && !kt0) {
      g_prof.pair(kt0, kt1, 2);
      VM_CUDA(cudaEventRecord(kt0, ts));
    }
    if (!prep_before_fork) {
      rc = launch_prep(i, ts);
      if (rc) return rc;
    }
    float* img = reinterpret_cast<float*>(ws + pl.off_img[i]);
    const int smem_tc = tck::Smem<128, 4>::total;
    VM_CUDA(cudaFuncSetAttribute(tck::tc_train_kernel<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tc));
    tck::tc_train_kernel<128, 4><<<ks.K * ks.P, tck::kTCThreads, smem_tc, ts>>>(pl.kp, i, img);
    VM_CUDA(cudaGetLastError());
    if (g_prof.on) g_prof.kernels += 1;
    if (forked && ks.P > 1) VM_CUDA(cudaEventRecord(ev_kt, ts));
    rc = launch_reduce(pl, i, ts);
    if (rc) return rc;
  }
  // the tensor-core stacks' Adam right behind their reduce on the branch
  // (programmatic launch; it waits for KF32 + the FFMA stacks' Adam through
  // ev_kf, since it reads their status words), so the step's tail does not
  // pay the join before it
  bool adam_on_branch = false;
  if (forked && kf_done && adam_split < pl.adam_grid && pdl_enabled()) {
    VM_CUDA(cudaStreamWaitEvent(ts, ev_kf, 0));
    // the MLP phase (profile tag 0) ends here: KF32 + its Adam and KT + reduce done
    if (g_prof.on) VM_CUDA(cudaEventRecord(e1, ts));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.adam_grid - adam_split);
    cfg.blockDim = dim3(256);
    cfg.stream = ts;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    VM_CUDA(cudaLaunchKernelEx(&cfg, adam_train_kernel, pl.ap, adam_split));
    if (g_prof.on) g_prof.kernels += 1;
    adam_on_branch = true;
  }
  // loss sums of the split tensor-core models: on a second branch once KT is
  // done, concurrently with their partial reduce and Adam (only the host
  // report needs them; Adam needs the reduce); joined after Adam
  bool ls_forked = false;
  for (int i = 0; i < n_stacks; ++i) {
    const KStack& ks = pl.kp.s[i];
    if (!ks.ls_sep || ks.K == 0 || ks.P <= 1) continue;
    cudaStream_t ls = s;
    if (forked) {
      VM_CUDA(cudaStreamWaitEvent(side2, ev_kt, 0));
      ls = side2;
      ls_forked = true;
    }
    LeafTable lt;
    int64_t st64[64];
    lt.n = pairwise_leaves(ks.R, st64, lt.len, 64);  // <= 64: ls_sep
    for (int l = 0; l < lt.n; ++l) lt.start[l] = int(st64[l]);
    lt.n_ops = 0;
    combine_program(ks.R, lt);  // 2 * leaves - 1 <= 127 ops, stack depth <= 7 (64 leaves)
    const int ls_smem = ks.R * 4;
    if (ls_smem > 48 * 1024)
      VM_CUDA(cudaFuncSetAttribute(loss_sums_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ls_smem));
    loss_sums_kernel<<<dim3(ks.K, 3), 128, ls_smem, ls>>>(pl.kp, i, lt);
    VM_CUDA(cudaGetLastError());
    if (g_prof.on) g_prof.kernels += 1;
  }
  if (kt1) VM_CUDA(cudaEventRecord(kt1, ts));
  if (!kf_done) {
    rc = launch_kf();
    if (rc) return rc;
  }
  if (forked) {
    VM_CUDA(cudaEventRecord(ev_join, side));
    VM_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
  }
  if (g_prof.on && !adam_on_branch) VM_CUDA(cudaEventRecord(e1, s));
  cudaEvent_t r0 = nullptr, r1 = nullptr;
  if (g_prof.on) {
    g_prof.pair(r0, r1, 3);
    VM_CUDA(cudaEventRecord(r0, s));
  }
  if (!adam_on_branch) {
    rc = launch_adam(pl, s, adam_split);
    if (rc) return rc;
  }
  if (ls_forked) {
    VM_CUDA(cudaEventRecord(ev_ls, side2));
    VM_CUDA(cudaStreamWaitEvent(s, ev_ls, 0));
  }
  if (r1) VM_CUDA(cudaEventRecord(r1, s));
  return VM_OK;
}

extern "C" int vm_train_step(const VmStack* stacks, const VmBatch* batches, int n_stacks, VmLossWeights w,
                             float* losses, int32_t* status, void* workspace, size_t workspace_bytes,
                             void* stream) {
  VM_REQUIRE(stacks && batches && n_stacks >= 1 && n_stacks <= VM_MAX_STACKS,
             "vm_train_step: 1 or 2 stacks supported");
  const cudaStream_t s = cudaStream_t(stream);
  switch (train_route(stacks, batches, n_stacks)) {
    case 0:
      return train_fused(stacks, batches, n_stacks, w, losses, status, workspace, workspace_bytes, stream);
    case 1: {
      const size_t b0 = align_up(fused_bytes(stacks, batches, 1), 256);
      VM_REQUIRE(workspace_bytes >= b0, "vm_train_step: workspace too small");
      int rc = train_fused(stacks, batches, 1, w, losses, status, workspace, b0, stream);
      if (rc) return rc;
      return train_layered(stacks, batches, 2, 1, w, losses, status, static_cast<char*>(workspace) + b0,
                           workspace_bytes - b0, s);
    }
    default:
      return train_layered(stacks, batches, n_stacks, 0, w, losses, status, workspace, workspace_bytes, s);
  }
}

namespace {
int run_fwd_bwd(const VmStack* st, const float* encoded, int64_t n_samples, const float* gocc,
                const float* gcol, float* occ, float* col, float* grads, bool backward, cudaStream_t s,
                float* img_ws = nullptr) {
  VM_REQUIRE(st && encoded && n_samples >= 0, "vm_forward/backward: bad arguments");
  KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  VmLayout L;
  int rc = fill_stack(*st, kp.s[0], L);
  if (rc == VM_ERR_UNSUPPORTED || (!rc && !(kp.s[0].H == 128 && kp.s[0].L == 4 && !backward && tc_enabled() &&
                                            tc_fwd_enabled() && kp.s[0].D <= tck::kK0) &&
                                   !(backward ? pick_kernel<kBackward>(kp.s[0].H, kp.s[0].L, 0, 0)
                                              : pick_kernel<kForward>(kp.s[0].H, kp.s[0].L, 0, 0)))) {
    // no fused kernel for this architecture: one kernel sequence per layer
    return layered_fwd_bwd(*st, encoded, n_samples, gocc, gcol, occ, col, grads, backward, s);
  }
  if (rc) {
    set_error("vm_forward/backward: unsupported architecture");
    return rc;
  }
  kp.n_stacks = 1;
  KStack& ks = kp.s[0];
  ks.N = n_samples;
  ks.S = 1;
  ks.G = 1;
  ks.R = 0;
  ks.enc = encoded;
  ks.gocc = gocc;
  ks.gcol = gcol;
  ks.occ_out = occ;
  ks.col_out = col;
  ks.grads = grads;
  const int nblk = int((n_samples + kSB - 1) / kSB);
  if (backward) {
    ks.P = 1;  // one CTA per model reduces every block of that model
  } else {
    // forward only (no reduction): enough CTAs to fill the GPU even for one
    // model (inference grids / rays), >= 1 block each
    ks.P = std::max(1, std::min(nblk, std::max(64, 148 * 8 / std::max(ks.K, 1))));
  }
  if (ks.K == 0 || n_samples == 0) {
    if (backward && ks.K > 0) VM_CUDA(cudaMemsetAsync(grads, 0, size_t(ks.K) * ks.block * 4, s));
    return VM_OK;
  }
  if (!backward && tc_enabled() && tc_fwd_enabled() && ks.H == 128 && ks.L == 4 && ks.D <= tck::kK0) {
    // hidden-128 forward (background grids / view rays) on the tensor cores:
    // the weight image (3xTF32 pre-split chunks) in a stream-ordered
    // temporary, then the persistent tile loop
    using TI = tck::Img<128, 4>;
    float* img = img_ws;
    if (!img) VM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&img), sizeof(float) * TI::total * size_t(ks.K), s));
    tck::tc_prep_kernel<128, 4><<<dim3(TI::n_chunks * 4, ks.K), 256, 0, s>>>(ks, img);
    VM_CUDA(cudaGetLastError());
    static int sms = 0;
    if (!sms) VM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int64_t tiles = (n_samples + tck::kTM - 1) / tck::kTM;
    // two tiles in flight per CTA when each CTA gets at least two (VM_TC_FWD=1: one)
    const bool two = tc_fwd_mode() == 2 && tiles >= 2 * int64_t(sms);
    const int64_t groups = two ? (tiles + 1) / 2 : tiles;
    const int gx = int(std::max<int64_t>(1, std::min<int64_t>(groups, (sms + ks.K - 1) / ks.K)));
    if (two) {
      const int smem = tck::FwdSmem<128, 4, 2>::total;
      VM_CUDA(cudaFuncSetAttribute(tck::tc_forward_kernel<128, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smem));
      tck::tc_forward_kernel<128, 4, 2><<<dim3(gx, ks.K), tck::kTCThreads, smem, s>>>(ks, img, n_samples, occ, col);
    } else {
      const int smem = tck::FwdSmem<128, 4, 1>::total;
      VM_CUDA(cudaFuncSetAttribute(tck::tc_forward_kernel<128, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smem));
      tck::tc_forward_kernel<128, 4, 1><<<dim3(gx, ks.K), tck::kTCThreads, smem, s>>>(ks, img, n_samples, occ, col);
    }
    VM_CUDA(cudaGetLastError());
    if (!img_ws) VM_CUDA(cudaFreeAsync(img, s));
    return VM_OK;
  }
  KernelFn fn = backward ? pick_kernel<kBackward>(ks.H, ks.L, 0, 0) : pick_kernel<kForward>(ks.H, ks.L, 0, 0);
  if (!fn) {
    set_error("vm_forward/backward: no kernel for this architecture");
    return VM_ERR_UNSUPPORTED;
  }
  return launch_mlp(fn, kp, ks.K * ks.P, smem_bytes(ks), s);
}
}  // namespace

extern "C" int vm_forward(const VmStack* st, const float* encoded, int64_t n_samples, float* occ, float* col,
                          void* stream) {
  return run_fwd_bwd(st, encoded, n_samples, nullptr, nullptr, occ, col, nullptr, false, cudaStream_t(stream));
}

size_t vm::fwd_image_bytes(const VmArch& a) {
  // one model's pre-split image (the inference entry points evaluate one model view)
  return (tc_enabled() && tc_fwd_enabled() && a.hidden > 64 && a.hidden <= 128 && a.n_layers == 4 &&
          a.input_dim <= tck::kK0)
             ? sizeof(float) * tck::Img<128, 4>::total
             : 0;
}

int vm::forward_ws(const VmStack* st, const float* encoded, int64_t n_samples, float* occ, float* col, float* img,
                   cudaStream_t s) {
  return run_fwd_bwd(st, encoded, n_samples, nullptr, nullptr, occ, col, nullptr, false, s,
                     st && st->count == 1 ? img : nullptr);
}

extern "C" int vm_backward(const VmStack* st, const float* encoded, int64_t n_samples, const float* grad_occ,
                           const float* grad_col, float* grads, void* stream) {
  return run_fwd_bwd(st, encoded, n_samples, grad_occ, grad_col, nullptr, nullptr, grads, true,
                     cudaStream_t(stream));
}

extern "C" int vm_trace_read(unsigned long long* out, int max_records, int* n_records) {
  VM_REQUIRE(out && n_records, "vm_trace_read: null argument");
  if (!g_trace) {
    *n_records = 0;
    return VM_OK;
  }
  VM_CUDA(cudaDeviceSynchronize());
  unsigned long long n = 0;
  VM_CUDA(cudaMemcpy(&n, g_trace, sizeof(n), cudaMemcpyDeviceToHost));
  n = std::min<unsigned long long>(n, std::min(max_records, 1 << 16));
  VM_CUDA(cudaMemcpy(out, g_trace + 1, sizeof(unsigned long long) * 4 * n, cudaMemcpyDeviceToHost));
  VM_CUDA(cudaMemset(g_trace, 0, sizeof(unsigned long long)));
  *n_records = int(n);
  return VM_OK;
}

extern "C" int vm_tc_debug_read(int* out) {
#ifdef VM_TC_DEBUG
  static cudaStream_t ds = nullptr;
  if (!ds) cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking);
  VM_CUDA(cudaMemcpyFromSymbolAsync(out, vm_tc_dbg, sizeof(int) * 512, 0, cudaMemcpyDeviceToHost, ds));
  VM_CUDA(cudaStreamSynchronize(ds));
  return VM_OK;
#else
  (void)out;
  return VM_ERR_UNSUPPORTED;
#endif
}

extern "C" int vm_profile_enable(int on) {
  g_prof.on = on != 0;
  g_prof.used = 0;
  g_prof.kernels = 0;
  return VM_OK;
}

extern "C" void vm_profile_count_kernels(int n) {
  if (g_prof.on) g_prof.kernels += n;
}

extern "C" int vm_profile_kernels(long* n) {
  *n = g_prof.kernels;
  return VM_OK;
}

extern "C" int vm_profile_read_tag(int tag, int* launches, double* total_ms) {
  double t = 0.0;
  int n = 0;
  for (size_t i = 0; i + 1 < g_prof.used; i += 2) {
    if (i / 2 >= g_prof.tag.size() || g_prof.tag[i / 2] != tag) continue;
    VM_CUDA(cudaEventSynchronize(g_prof.ev[i + 1]));
    float ms = 0.f;
    VM_CUDA(cudaEventElapsedTime(&ms, g_prof.ev[i], g_prof.ev[i + 1]));
    t += ms;
    ++n;
  }
  *launches = n;
  *total_ms = t;
  return VM_OK;
}

extern "C" int vm_profile_read(int* launches, double* total_ms) {
  return vm_profile_read_tag(0, launches, total_ms);
}

extern "C" int vm_train_grid(const VmStack* stacks, const VmBatch* batches, int n_stacks, int* ctas,
                             int* smem_bytes) {
  TrainPlan pl;
  int rc = plan_train(stacks, batches, n_stacks, pl);
  if (rc) return rc;
  *ctas = pl.grid;
  *smem_bytes = int(pl.smem);
  return VM_OK;
}
