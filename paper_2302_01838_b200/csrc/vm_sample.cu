// KS: ray/sample generation for the per-object training batch.
//
// Restates, on the device and bit-exactly:
//   objects.py:323-352  sample_training_pixels (keyframe index, pixel, mask bit)
//   trainer.py:269-318  _assemble_batch (gathers, f64 ray geometry, padded box)
//   render.py:76-139    camera_dirs / ray_box_intersect
//   render.py:142-227   depth-guided stratified + Gaussian surface sampling
//   models.py:286-308   positional encoding (f64, cast to f32)
//   rng.py:24-34        keyed SeedSequence -> PCG64 streams; numpy's
//                       Generator.integers (32-bit Lemire), .random() and
//                       .standard_normal() (256-layer ziggurat) draw layouts.
// The file is compiled with -fmad=false so every f64 expression rounds like
// the numpy expression it restates (verified in tests/test_gpu_sampler.py).
//
// Stream layouts (per object, per step):
//   PIXELS  key (seed,3,obj,step): [ceil(R/2) words kf Lemire halves, absent
//           if n_kf==1][2R words uv]
//   SAMPLES key (seed,4,obj,step): [nc*R u_strat][ns*R normals, variable
//           length][S*R u_fallback]
// Normals are resolved in parallel: every window position is classified as a
// ziggurat fast accept or not, slow positions are resolved speculatively, and
// one thread walks only the slow list to place them (about 2% of positions).
#include "vm_common.cuh"
#define VM_ZIG_QUAL __device__
#include "ziggurat_tables.h"

#include <cstring>

namespace vm {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
  return (u128(2549297995355413924ULL) << 64) | u128(4865540595714422341ULL);
}

__device__ __forceinline__ uint64_t pcg_out(u128 s) {
  const uint64_t hi = uint64_t(s >> 64), lo = uint64_t(s);
  const uint64_t x = hi ^ lo;
  const unsigned rot = unsigned(hi >> 58);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

// State after `delta` LCG steps (Brown, "Random number generation with
// arbitrary strides").
__device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// Jump tables: advancing by 2^k steps is s -> A[k]*s + G[k]*inc with
// A[k] = M^(2^k), G[k] = sum_{i<2^k} M^i (mod 2^128); filled once on the host.
constexpr int kJumpBits = 48;
__constant__ u128 c_jumpA[kJumpBits];
__constant__ u128 c_jumpG[kJumpBits];

__device__ __forceinline__ u128 pcg_jump(u128 s, u128 inc, uint64_t delta) {
#pragma unroll 1
  for (int k = 0; k < kJumpBits; ++k) {
    if (!__any_sync(__activemask(), (delta >> k) != 0)) break;  // warp-uniform exit
    if ((delta >> k) & 1) s = c_jumpA[k] * s + c_jumpG[k] * inc;
  }
  return s;
}

struct Stream {
  u128 state0, inc;
  // Cursor positioned so that next() returns word `pos`.
  __device__ __forceinline__ u128 at(uint64_t pos) const { return pcg_jump(state0, inc, pos); }
};

__device__ __forceinline__ uint64_t next_word(u128& s, u128 inc) {
  s = s * pcg_mult() + inc;
  return pcg_out(s);
}

__device__ __forceinline__ double word_to_double(uint64_t w) { return double(w >> 11) * (1.0 / 9007199254740992.0); }

// SeedSequence(parts).generate_state(8) -> PCG64 seeding (numpy bit_generator.pyx, pcg64.c).
__device__ Stream seed_stream(uint64_t seed, uint64_t purpose, uint64_t obj, uint64_t step) {
  uint32_t ent[8];
  int n = 0;
  const uint64_t parts[4] = {seed, purpose, obj, step};
  for (int i = 0; i < 4; ++i) {
    uint64_t v = parts[i];
    if (v == 0) {
      ent[n++] = 0;
    } else {
      while (v) {
        ent[n++] = uint32_t(v);
        v >>= 32;
      }
    }
  }
  uint32_t hc = 0x43b0d7e5u;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [](uint32_t x, uint32_t y) {
    const uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int e = 4; e < n; ++e)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[e]));
  uint32_t hb = 0x8b51f9ddu, w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= 0x58f38dedu;
    v *= hb;
    w[i] = v ^ (v >> 16);
  }
  uint64_t u[4];
  for (int i = 0; i < 4; ++i) u[i] = uint64_t(w[2 * i]) | (uint64_t(w[2 * i + 1]) << 32);
  const u128 initstate = (u128(u[0]) << 64) | u128(u[1]);
  const u128 initseq = (u128(u[2]) << 64) | u128(u[3]);
  Stream st;
  st.inc = (initseq << 1) | 1;
  u128 s = st.inc;  // 0 * mult + inc
  s += initstate;
  s = s * pcg_mult() + st.inc;
  st.state0 = s;
  return st;
}

struct Zig {
  const uint64_t* ki;
  const double* wi;
  const double* fi;
};

__device__ __forceinline__ double zig_fast(uint64_t r, const Zig& z, bool& fast) {
  const int idx = int(r & 0xff);
  r >>= 8;
  const int sign = int(r & 1);
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
  double x = double(rabs) * z.wi[idx];
  if (sign) x = -x;
  fast = rabs < z.ki[idx];
  return x;
}

// Resolve an attempt starting at absolute word `p` whose first word is not a
// fast accept.  Returns consumed words; `accepted` false means the normal
// restarts at p + consumed.
__device__ int zig_slow(const Stream& st, uint64_t p, const Zig& z, double& value, bool& accepted) {
  u128 s = st.at(p);
  uint64_t r = next_word(s, st.inc);
  const int idx = int(r & 0xff);
  r >>= 8;
  const int sign = int(r & 1);
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
  double x = double(rabs) * z.wi[idx];
  if (sign) x = -x;
  const double zr = 3.6541528853610087963519472518;
  const double zinv = 0.27366123732975827203338247596;
  if (idx == 0) {
    int used = 1;
    for (;;) {
      const double xx = -zinv * log1p(-word_to_double(next_word(s, st.inc)));
      const double yy = -log1p(-word_to_double(next_word(s, st.inc)));
      used += 2;
      if (yy + yy > xx * xx) {
        value = ((rabs >> 8) & 0x1) ? -(zr + xx) : zr + xx;
        accepted = true;
        return used;
      }
    }
  }
  const double u = word_to_double(next_word(s, st.inc));
  accepted = ((z.fi[idx - 1] - z.fi[idx]) * u + z.fi[idx]) < exp(-0.5 * x * x);
  value = x;
  return 2;
}

__device__ __forceinline__ double np_min_d(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a <= b ? a : b;
}
__device__ __forceinline__ double np_max_d(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a >= b ? a : b;
}

struct KS {
  const VmSampleObject* objs;
  const VmKeyframe* kfs;
  const float4* rgbd;
  const uint8_t* mask;
  VmSampleParams p;
  int S, N, W, SC;  // samples/ray, normals/object, window, slow capacity
  // outputs
  float* t32;
  float* tdepth;
  float* tcol;
  uint8_t* tmask;
  uint8_t* valid;
  uint8_t* ok;
  float* points;    // [K,R,S,3] f32 (encode == 0)
  double* p64;      // [K,R,S,3] f64 workspace (encode == 1)
  // workspace written by the per-object prep kernel
  Stream* streams;  // [K][2] PIXELS, SAMPLES
  int* kf;          // [K,R] keyframe index per ray
  int64_t* bases;   // [K][2] first uv word (PIXELS), first u_fallback word (SAMPLES)
  double* nrm;      // [K,N] resolved normals
  int* status;      // [K] fallback flags (diagnostics)
  int64_t* aux_kf;
  int64_t* aux_u;
  int64_t* aux_v;
  double* aux_t64;
  unsigned long long* trace;  // VM_TRACE schedule records, or null
};

// schedule record of one CTA at every exit of a sampler kernel
struct TraceOnExit {
  unsigned long long* tr;
  int kind;
  unsigned long long t;
  __device__ TraceOnExit(unsigned long long* tr_, int kind_) : tr(tr_), kind(kind_), t(tr_ ? vm_gtime() : 0) {}
  __device__ ~TraceOnExit() {
    if (tr && threadIdx.x == 0) vm_trace_rec(tr, kind, t);
  }
};

// Block-wide exclusive scan of one int per thread (blockDim.x == 256).
__device__ int block_exclusive_scan(int v, int* scratch, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < 8 ? scratch[lane] : 0;
    for (int o = 1; o < 8; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < 8) scratch[8 + lane] = w;
  }
  __syncthreads();
  total = scratch[8 + 7];
  const int before = warp ? scratch[8 + warp - 1] : 0;
  const int excl = before + x - v;
  __syncthreads();
  return excl;
}

constexpr int kST = 256;
constexpr int kRT = 128;  // per-ray kernel block size

__device__ __forceinline__ bool object_live(const VmSampleObject& ob) { return ob.active && ob.n_kf > 0; }
__device__ __forceinline__ int object_rays(const VmSampleObject& ob, const VmSampleParams& P) {
  return (ob.n_rays > 0 && ob.n_rays < P.n_rays) ? ob.n_rays : P.n_rays;
}

// ---- per object: stream seeds, keyframe index per ray, normal resolution.
__global__ void __launch_bounds__(kST) sample_prep_kernel(const __grid_constant__ KS ks) {
  TraceOnExit rec(ks.trace, 5);
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint64_t s_ki[256];
  __shared__ double s_wi[256], s_fi[256];
  __shared__ Stream s_pix, s_smp;
  __shared__ int s_scan[16], s_flag, s_nseg, s_nov, s_end;
  __shared__ int64_t s_kfwords;

  const int k = blockIdx.x, tid = threadIdx.x;
  const VmSampleObject ob = ks.objs[k];
  if (!object_live(ob)) return;
  const VmSampleParams& P = ks.p;
  // rays this object draws (config 3: fewer than the batch width; the PIXELS
  // and SAMPLES streams are laid out for exactly this many draws)
  const int R = object_rays(ob, P), nc = P.n_stratified, N = P.n_surface * R, W = ks.W;

  double* xs = reinterpret_cast<double*>(sm);                  // [W]
  double* ov_val = xs + W;                                     // [SC]
  int* slow = reinterpret_cast<int*>(ov_val + ks.SC);          // [SC]
  int* seg_j = slow + ks.SC;                                   // [SC+1]
  int* seg_off = seg_j + ks.SC + 1;                            // [SC+1]
  int* ov_j = seg_off + ks.SC + 1;                             // [SC]
  uint8_t* fastf = reinterpret_cast<uint8_t*>(ov_j + ks.SC);   // [W]

  for (int i = tid; i < 256; i += kST) {
    s_ki[i] = vm_zig_ki[i];
    s_wi[i] = __longlong_as_double(static_cast<long long>(vm_zig_wi[i]));
    s_fi[i] = __longlong_as_double(static_cast<long long>(vm_zig_fi[i]));
  }
  const uint64_t step = P.step_dev ? uint64_t(*P.step_dev + P.step_offset) : uint64_t(P.step);
  if (tid == 0) s_pix = seed_stream(P.seed, 3, uint64_t(ob.object_id), step);
  if (tid == 32) s_smp = seed_stream(P.seed, 4, uint64_t(ob.object_id), step);
  if (tid == 64) s_flag = 0;
  __syncthreads();
  const Zig zig{s_ki, s_wi, s_fi};
  const Stream pix = s_pix, smp = s_smp;
  if (tid == 0) {
    ks.streams[2 * k] = pix;
    ks.streams[2 * k + 1] = smp;
  }

  // ---------------- keyframe index per ray (objects.py:336) ----------------
  int* kf_out = ks.kf + int64_t(k) * P.n_rays;
  const int n_kf = ob.n_kf;
  if (n_kf == 1) {
    for (int r = tid; r < R; r += kST) kf_out[r] = 0;
    if (tid == 0) s_kfwords = 0;
  } else {
    const uint32_t n = uint32_t(n_kf);
    const uint32_t thr = uint32_t((uint64_t(1) << 32) - n) % n;
    bool rej = false;
    // two rays (low/high half) per 64-bit word; consecutive words per thread
    for (int w = tid; w < (R + 1) / 2; w += kST) {
      u128 s = pix.at(uint64_t(w));
      const uint64_t word = next_word(s, pix.inc);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 2 * w + h;
        if (r >= R) break;
        const uint32_t x = h ? uint32_t(word >> 32) : uint32_t(word);
        const uint64_t m = uint64_t(x) * n;
        const uint32_t left = uint32_t(m);
        if (left < n && left < thr) rej = true;
        kf_out[r] = int(m >> 32);
      }
    }
    if (__syncthreads_or(rej)) {
      if (tid == 0) {  // rare: replay the buffered Lemire draws sequentially
        u128 s = pix.state0;
        uint64_t buf = 0, words = 0;
        bool have = false;
        for (int r = 0; r < R;) {
          uint32_t x;
          if (have) {
            x = uint32_t(buf >> 32);
            have = false;
          } else {
            buf = next_word(s, pix.inc);
            ++words;
            x = uint32_t(buf);
            have = true;
          }
          const uint64_t m = uint64_t(x) * n;
          const uint32_t left = uint32_t(m);
          if (left < n && left < thr) continue;
          kf_out[r++] = int(m >> 32);
        }
        s_kfwords = int64_t(words);
        s_flag |= 1;
      }
    } else if (tid == 0) {
      s_kfwords = (R + 1) / 2;
    }
  }

  // ---------------- normals (render.py:185) ----------------
  const uint64_t nbase = uint64_t(nc) * R;
  int total = 0;
  {
    const int per = (W + kST - 1) / kST;
    const int p0 = tid * per, p1 = min(W, p0 + per);
    int cnt = 0;
    if (p0 < p1) {
      u128 s = smp.at(nbase + p0);
      for (int p = p0; p < p1; ++p) {
        bool f;
        xs[p] = zig_fast(next_word(s, smp.inc), zig, f);
        fastf[p] = f;
        cnt += !f;
      }
    }
    int off = block_exclusive_scan(cnt, s_scan, total);
    if (total > ks.SC) {
      if (tid == 0) s_flag |= 2;
    } else {
      for (int p = p0; p < p1; ++p)
        if (!fastf[p]) slow[off++] = p;
    }
    __syncthreads();
    if (!(s_flag & 2)) {  // speculative slow-path resolution, one thread per slow position
      for (int i = tid; i < total; i += kST) {
        double v;
        bool acc;
        const int used = zig_slow(smp, nbase + slow[i], zig, v, acc);
        ov_val[i] = v;
        ov_j[i] = acc ? used : -used;  // +consumed (accepted) / -consumed (rejected)
      }
    }
    __syncthreads();
    if (tid == 0 && !(s_flag & 2)) {
      // walk the slow list: seg_j/seg_off = segment starts/offsets of fast
      // normals; slow[]/ov_val[] are compacted in place to the accepted slow
      // normals (index, value).
      int pos = 0, j = 0, nseg = 1, nov = 0;
      seg_j[0] = 0;
      seg_off[0] = 0;
      for (int i = 0; i < total && j < N; ++i) {
        const int s = slow[i];
        if (s < pos) continue;
        if (j + (s - pos) >= N) break;
        j += s - pos;
        const int r = ov_j[i];
        if (r > 0) {
          ov_val[nov] = ov_val[i];
          slow[nov] = j;
          ++nov;
          ++j;
          pos = s + r;
        } else {
          pos = s - r;
        }
        seg_j[nseg] = j;
        seg_off[nseg] = pos - j;
        ++nseg;
      }
      const int end = pos + (N - j);
      if (end > W) s_flag |= 2;
      s_nseg = nseg;
      s_nov = nov;
      s_end = end;
    }
    __syncthreads();
  }
  double* nrm = ks.nrm + int64_t(k) * ks.N;
  if (s_flag & 2) {
    if (tid == 0) {  // window overflow (practically unreachable): sequential replay
      u128 s = smp.at(nbase);
      uint64_t used = 0;
      for (int j = 0; j < N; ++j) {
        for (;;) {
          bool f;
          const double x = zig_fast(next_word(s, smp.inc), zig, f);
          if (f) {
            nrm[j] = x;
            ++used;
            break;
          }
          double v;
          bool acc;
          const int u = zig_slow(smp, nbase + used, zig, v, acc);
          used += u;
          s = smp.at(nbase + used);
          if (acc) {
            nrm[j] = v;
            break;
          }
        }
      }
      s_end = int(used);
    }
  } else {
    const int nseg = s_nseg, nov = s_nov;
    for (int j = tid; j < N; j += kST) {
      int lo = 0, hi = nseg - 1;  // last segment with seg_j <= j
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (seg_j[mid] <= j) lo = mid;
        else hi = mid - 1;
      }
      int a = 0, b = nov - 1, hit = -1;  // accepted-slow override
      while (a <= b) {
        const int mid = (a + b) >> 1;
        if (slow[mid] == j) {
          hit = mid;
          break;
        }
        if (slow[mid] < j) a = mid + 1;
        else b = mid - 1;
      }
      nrm[j] = hit >= 0 ? ov_val[hit] : xs[j + seg_off[lo]];
    }
  }
  __syncthreads();
  if (tid == 0) {
    ks.bases[2 * k] = s_kfwords;
    ks.bases[2 * k + 1] = int64_t(nbase) + s_end;
    ks.status[k] = s_flag;
  }
}

// ---- per ray: pixel, gathers, f64 geometry, depth-guided samples, outputs.
__global__ void __launch_bounds__(kRT) sample_rays_kernel(const __grid_constant__ KS ks, int n_objects) {
  TraceOnExit rec(ks.trace, 6);
  const VmSampleParams& P = ks.p;
  const int R = P.n_rays, S = ks.S, nc = P.n_stratified, nsf = P.n_surface;
  const int64_t rg = blockIdx.x * int64_t(kRT) + threadIdx.x;
  if (rg >= int64_t(n_objects) * R) return;
  const int k = int(rg / R), r = int(rg % R);
  const VmSampleObject& ob = ks.objs[k];
  // zero batch (trainer.py:190-200, :272-273); rows past the object's own
  // ray count are the same zero rows (config-3 padding, ray_ok = 0)
  if (!object_live(ob) || r >= object_rays(ob, P)) {
    for (int i = 0; i < S; ++i) {
      ks.t32[rg * S + i] = 0.f;
      if (ks.points)
        for (int c = 0; c < 3; ++c) ks.points[(rg * S + i) * 3 + c] = 0.f;
      if (ks.p64)
        for (int c = 0; c < 3; ++c) ks.p64[(rg * S + i) * 3 + c] = 0.0;
      if (ks.aux_t64) ks.aux_t64[rg * S + i] = 0.0;
    }
    ks.tdepth[rg] = 0.f;
    for (int c = 0; c < 3; ++c) ks.tcol[rg * 3 + c] = 0.f;
    ks.tmask[rg] = 0;
    ks.valid[rg] = 0;
    ks.ok[rg] = 0;
    if (ks.aux_kf) {
      ks.aux_kf[rg] = 0;
      ks.aux_u[rg] = 0;
      ks.aux_v[rg] = 0;
    }
    return;
  }
  const Stream pix = ks.streams[2 * k], smp = ks.streams[2 * k + 1];
  const uint64_t uv_base = uint64_t(ks.bases[2 * k]), fb_base = uint64_t(ks.bases[2 * k + 1]);
  const int kfi = ks.kf[rg];
  const VmKeyframe& kf = ks.kfs[ob.kf_begin + kfi];
  u128 s = pix.at(uv_base + 2 * uint64_t(r));
  const double du = word_to_double(next_word(s, pix.inc));
  const double dv = word_to_double(next_word(s, pix.inc));
  int64_t u = kf.u0 + int64_t(floor(du * double(kf.u1 - kf.u0)));
  int64_t v = kf.v0 + int64_t(floor(dv * double(kf.v1 - kf.v0)));
  u = u < int64_t(kf.u1 - 1) ? u : int64_t(kf.u1 - 1);
  v = v < int64_t(kf.v1 - 1) ? v : int64_t(kf.v1 - 1);
  const int64_t tix = kf.texel_off + (v - kf.v0) * (kf.u1 - kf.u0) + (u - kf.u0);
  const float4 px = ks.rgbd[tix];
  const bool in_mask = ks.mask[tix] != 0;

  // rays (trainer.py:289-297): camera dirs, rotate, normalise
  const double d0 = (double(u) - P.cx) / P.fx;
  const double d1 = (double(v) - P.cy) / P.fy;
  const double to_t = sqrt((d0 * d0 + d1 * d1) + 1.0);
  double dir[3], org[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    // einsum "rij,rj->ri": (R[i][0]*d0 + R[i][2]*1.0) + R[i][1]*d1
    dir[i] = (kf.pose[4 * i + 0] * d0 + kf.pose[4 * i + 2] * 1.0) + kf.pose[4 * i + 1] * d1;
    org[i] = kf.pose[4 * i + 3];
  }
  const double dn = sqrt((dir[0] * dir[0] + dir[1] * dir[1]) + dir[2] * dir[2]);
#pragma unroll
  for (int i = 0; i < 3; ++i) dir[i] = dir[i] / dn;
  const double z = double(px.w);
  const bool valid = z > 0.0;
  const double surf = z * to_t;

  // ray_box_intersect (render.py:111-139) on the padded box
  double tin = -INFINITY, tout = INFINITY;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double lo, hi;
    if (dir[i] == 0.0) {
      const bool inside = (org[i] >= ob.box_min[i]) && (org[i] <= ob.box_max[i]);
      lo = inside ? -INFINITY : INFINITY;
      hi = inside ? INFINITY : -INFINITY;
    } else {
      const double inv = 1.0 / dir[i];
      const double ta = (ob.box_min[i] - org[i]) * inv;
      const double tb = (ob.box_max[i] - org[i]) * inv;
      lo = np_min_d(ta, tb);
      hi = np_max_d(ta, tb);
    }
    tin = i == 0 ? lo : np_max_d(tin, lo);
    tout = i == 0 ? hi : np_min_d(tout, hi);
  }
  const double t_entry = np_max_d(tin, 0.0);
  const bool hit = (tout >= t_entry) && (tout >= 0.0);
  const double near_ = hit ? np_max_d(t_entry, P.t_near) : P.t_near;
  const double far_ = (hit && tout > near_) ? tout : P.t_far;

  // sample_along_rays (render.py:149-227)
  const double lo = near_;
  const double far2 = np_max_d(far_, lo);
  const bool has_depth = valid && (surf > lo);
  const bool near_block = valid && !has_depth;
  const bool over = in_mask && has_depth && (surf > far2 + P.three_std);
  const bool guided = in_mask && has_depth && !over;
  const double upper = in_mask ? far2 : (has_depth ? np_min_d(surf, far2) : far2);
  const bool ray_ok = (guided || upper > lo) && !near_block && !over;
  double t[32];
  if (guided) {
    u128 q = smp.at(uint64_t(nc) * r);
    for (int i = 0; i < nc; ++i) {
      const double us = word_to_double(next_word(q, smp.inc));
      t[i] = lo + ((double(i) + us) / double(nc)) * (surf - lo);
    }
    const double band_hi = np_min_d(surf + P.three_std, far2);
    const double* nz = ks.nrm + int64_t(k) * ks.N + int64_t(r) * nsf;
    for (int i = 0; i < nsf; ++i) {
      const double a = surf + P.surface_std * nz[i];
      t[nc + i] = np_min_d(np_max_d(a, lo), band_hi);
    }
  } else {
    u128 q = smp.at(fb_base + uint64_t(S) * r);
    const double hi_f = np_max_d(upper, lo);
    for (int i = 0; i < S; ++i) {
      const double uf = word_to_double(next_word(q, smp.inc));
      t[i] = lo + ((double(i) + uf) / double(S)) * (hi_f - lo);
    }
  }
  for (int i = 1; i < S; ++i) {  // ascending insertion sort
    const double x = t[i];
    int j = i - 1;
    while (j >= 0 && t[j] > x) {
      t[j + 1] = t[j];
      --j;
    }
    t[j + 1] = x;
  }

  ks.tdepth[rg] = float(surf);
  ks.tcol[rg * 3 + 0] = px.x;
  ks.tcol[rg * 3 + 1] = px.y;
  ks.tcol[rg * 3 + 2] = px.z;
  ks.tmask[rg] = in_mask;
  ks.valid[rg] = valid;
  ks.ok[rg] = ray_ok;
  if (ks.aux_kf) {
    ks.aux_kf[rg] = kfi;
    ks.aux_u[rg] = u;
    ks.aux_v[rg] = v;
  }
  for (int i = 0; i < S; ++i) {
    const int64_t sg = rg * S + i;
    ks.t32[sg] = float(t[i]);
    if (ks.aux_t64) ks.aux_t64[sg] = t[i];
    double pn[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) pn[c] = ((org[c] + t[i] * dir[c]) - ob.center[c]) / ob.half[c];
    if (ks.points) {
#pragma unroll
      for (int c = 0; c < 3; ++c) ks.points[sg * 3 + c] = float(pn[c]);
    }
    if (ks.p64) {
#pragma unroll
      for (int c = 0; c < 3; ++c) ks.p64[sg * 3 + c] = pn[c];
    }
  }
}

// positional_encode (models.py:286-308) from the f64 normalised points:
// one thread per (sample, band); band -1 writes the raw point.
__global__ void encode_kernel(int64_t n_samples, int n_freq, int include, int D, int S, int64_t samples_per_obj,
                              const VmSampleObject* __restrict__ objs, const double* __restrict__ p64,
                              float* __restrict__ enc, int R) {
  const int nb = n_freq + (include ? 1 : 0);
  const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (idx >= n_samples * nb) return;
  const int64_t smp = idx / nb;
  const int b = int(idx % nb) - (include ? 1 : 0);
  float* out = enc + smp * D;
  const int64_t obj = smp / samples_per_obj;
  const int nr = (objs[obj].n_rays > 0 && objs[obj].n_rays < R) ? objs[obj].n_rays : R;
  const bool live = objs[obj].active && objs[obj].n_kf > 0 && (smp % samples_per_obj) / S < nr;
  const double* p = p64 + smp * 3;
  if (b < 0) {
    for (int c = 0; c < 3; ++c) out[c] = live ? float(p[c]) : 0.f;
    return;
  }
  const int base = (include ? 3 : 0) + 6 * b;
  if (!live) {
    for (int c = 0; c < 6; ++c) out[base + c] = 0.f;
    return;
  }
  const double coef = (3.141592653589793 * double(1u << b)) / objs[obj].pe_scale;
  for (int c = 0; c < 3; ++c) {
    const double a = coef * p[c];
    out[base + c] = float(sin(a));
    out[base + 3 + c] = float(cos(a));
  }
}

struct SamplePlan {
  int S, N, W, SC;
  size_t smem;
  size_t off_streams, off_kf, off_bases, off_nrm, off_status, off_p64, bytes;
};

SamplePlan plan_sample(int n_objects, const VmSampleParams& p) {
  SamplePlan pl;
  pl.S = p.n_stratified + p.n_surface;
  pl.N = p.n_surface * p.n_rays;
  pl.W = pl.N + pl.N / 16 + 64;
  pl.SC = pl.W / 8 + 64;
  pl.smem = size_t(pl.W) * 8 + size_t(pl.SC) * 8 + size_t(pl.SC) * 4 * 2 + size_t(pl.SC + 1) * 4 * 2 +
            size_t(pl.W) + 16;
  size_t off = 0;
  auto take = [&](size_t b) {
    const size_t o = off;
    off = (off + b + 255) / 256 * 256;
    return o;
  };
  pl.off_streams = take(size_t(n_objects) * 2 * sizeof(Stream));
  pl.off_kf = take(size_t(n_objects) * p.n_rays * 4);
  pl.off_bases = take(size_t(n_objects) * 2 * 8);
  pl.off_nrm = take(size_t(n_objects) * pl.N * 8 + 8);
  pl.off_status = take(size_t(n_objects) * 4 + 4);
  pl.off_p64 = take(p.encode ? size_t(n_objects) * p.n_rays * pl.S * 3 * 8 : 0);
  pl.bytes = off;
  return pl;
}

// Host: jump tables A[k] = M^(2^k), G[k] = 1 + M + ... + M^(2^k - 1) (mod 2^128).
int ensure_jump_tables() {
  static bool ready = false;
  if (ready) return VM_OK;
  const u128 M = (u128(2549297995355413924ULL) << 64) | u128(4865540595714422341ULL);
  u128 A[kJumpBits], G[kJumpBits];
  u128 a = M, g = 1;
  for (int k = 0; k < kJumpBits; ++k) {
    A[k] = a;
    G[k] = g;
    g = g * (a + 1);  // sum_{i<2^(k+1)} M^i = (1 + M^(2^k)) * sum_{i<2^k} M^i
    a = a * a;
  }
  VM_CUDA(cudaMemcpyToSymbol(c_jumpA, A, sizeof(A)));
  VM_CUDA(cudaMemcpyToSymbol(c_jumpG, G, sizeof(G)));
  ready = true;
  return VM_OK;
}

}  // namespace
}  // namespace vm

using namespace vm;

extern "C" void vm_profile_count_kernels(int n);

namespace vm {
__global__ void step_advance_kernel(int64_t* c, int64_t inc, unsigned long long* tr) {
  const unsigned long long t0 = tr ? vm_gtime() : 0;
  *c += inc;
  if (tr) vm_trace_rec(tr, 9, t0);
}
}  // namespace vm

namespace vm {
// End of a step graph: the step's result words (losses + status) stored
// straight into mapped pinned host memory (no copy-engine transfer: a few
// hundred bytes of posted writes) and the device step counter advanced.
__global__ void step_finish_kernel(const int32_t* __restrict__ src, int32_t* host_dst, int n, int64_t* c,
                                   int64_t inc, unsigned long long* tr) {
  const unsigned long long t0 = tr ? vm_gtime() : 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) host_dst[i] = __ldcg(src + i);
  __threadfence_system();
  if (threadIdx.x == 0) {
    *c += inc;
    if (tr) vm_trace_rec(tr, 9, t0);
  }
}
}  // namespace vm

extern "C" int vm_step_finish(const int32_t* words, int32_t* host_words, int32_t n_words, int64_t* counter,
                              int64_t inc, void* stream) {
  VM_REQUIRE(n_words >= 0 && (n_words == 0 || (words && host_words)) && counter, "vm_step_finish: bad arguments");
  int32_t* dst = nullptr;
  if (n_words > 0) VM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dst), host_words, 0));
  step_finish_kernel<<<1, 256, 0, cudaStream_t(stream)>>>(words, dst, n_words, counter, inc, trace_ptr());
  VM_CUDA(cudaGetLastError());
  return VM_OK;
}

// Launch an instantiated CUDA graph (the Mapper's captured step) on `stream`
// without the Python-side replay wrapper.
extern "C" int vm_graph_launch(void* graph_exec, void* stream) {
  VM_REQUIRE(graph_exec, "vm_graph_launch: null graph");
  VM_CUDA(cudaGraphLaunch(cudaGraphExec_t(graph_exec), cudaStream_t(stream)));
  return VM_OK;
}

extern "C" int vm_step_advance(int64_t* counter, int64_t inc, void* stream) {
  step_advance_kernel<<<1, 1, 0, cudaStream_t(stream)>>>(counter, inc, trace_ptr());
  VM_CUDA(cudaGetLastError());
  return VM_OK;
}

extern "C" size_t vm_sample_workspace_bytes(int n_objects, const VmSampleParams* params) {
  if (!params || n_objects < 0) return 0;
  return plan_sample(n_objects, *params).bytes;
}

extern "C" int vm_sample(const VmSampleObject* objects, int n_objects, const VmKeyframe* keyframes,
                         const float* rgbd, const uint8_t* mask, const VmSampleParams* params, VmBatch* out,
                         VmSampleAux* aux, void* workspace, size_t workspace_bytes, void* stream) {
  VM_REQUIRE(params && out && n_objects >= 0, "vm_sample: null argument");
  const VmSampleParams& p = *params;
  VM_REQUIRE(p.n_rays >= 1 && p.n_stratified >= 1 && p.n_surface >= 0, "vm_sample: bad sampling config");
  VM_REQUIRE(p.n_stratified + p.n_surface <= 32, "vm_sample: at most 32 points per ray");
  VM_REQUIRE(p.fx > 0 && p.fy > 0, "vm_sample: bad intrinsics");
  SamplePlan pl = plan_sample(n_objects, p);
  VM_REQUIRE(workspace_bytes >= pl.bytes, "vm_sample: workspace too small");
  VM_REQUIRE(pl.smem <= 220 * 1024, "vm_sample: too many rays per object for one CTA");
  if (n_objects == 0) return VM_OK;
  if (p.encode) VM_REQUIRE(out->encoded != nullptr, "vm_sample: encoded output missing");
  else VM_REQUIRE(out->points != nullptr, "vm_sample: points output missing");
  int rc = ensure_jump_tables();
  if (rc) return rc;
  char* ws = static_cast<char*>(workspace);
  KS ks;
  std::memset(&ks, 0, sizeof(ks));
  ks.objs = objects;
  ks.kfs = keyframes;
  ks.rgbd = reinterpret_cast<const float4*>(rgbd);
  ks.mask = mask;
  ks.p = p;
  ks.S = pl.S;
  ks.N = pl.N;
  ks.W = pl.W;
  ks.SC = pl.SC;
  ks.t32 = const_cast<float*>(out->t);
  ks.tdepth = const_cast<float*>(out->target_depth);
  ks.tcol = const_cast<float*>(out->target_colour);
  ks.tmask = const_cast<uint8_t*>(out->target_mask);
  ks.valid = const_cast<uint8_t*>(out->valid_depth);
  ks.ok = const_cast<uint8_t*>(out->ray_ok);
  ks.points = p.encode ? nullptr : const_cast<float*>(out->points);
  ks.p64 = p.encode ? reinterpret_cast<double*>(ws + pl.off_p64) : nullptr;
  ks.streams = reinterpret_cast<Stream*>(ws + pl.off_streams);
  ks.kf = reinterpret_cast<int*>(ws + pl.off_kf);
  ks.bases = reinterpret_cast<int64_t*>(ws + pl.off_bases);
  ks.nrm = reinterpret_cast<double*>(ws + pl.off_nrm);
  ks.status = reinterpret_cast<int*>(ws + pl.off_status);
  ks.trace = trace_ptr();
  if (aux) {
    ks.aux_kf = aux->kf_idx;
    ks.aux_u = aux->u;
    ks.aux_v = aux->v;
    ks.aux_t64 = aux->t64;
  }
  cudaStream_t s = cudaStream_t(stream);
  VM_CUDA(cudaFuncSetAttribute(sample_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem)));
  sample_prep_kernel<<<n_objects, kST, pl.smem, s>>>(ks);
  VM_CUDA(cudaGetLastError());
  const int64_t n_rays = int64_t(n_objects) * p.n_rays;
  sample_rays_kernel<<<unsigned((n_rays + kRT - 1) / kRT), kRT, 0, s>>>(ks, n_objects);
  VM_CUDA(cudaGetLastError());
  vm_profile_count_kernels(2);
  if (p.encode) {
    const int D = (p.include_input ? 3 : 0) + 6 * p.n_freq;
    const int64_t spo = int64_t(p.n_rays) * pl.S;
    const int64_t n = int64_t(n_objects) * spo;
    const int nb = p.n_freq + (p.include_input ? 1 : 0);
    const int64_t work = n * nb;
    encode_kernel<<<unsigned((work + 255) / 256), 256, 0, s>>>(n, p.n_freq, p.include_input, D, pl.S, spo, objects,
                                                               ks.p64, const_cast<float*>(out->encoded), p.n_rays);
    VM_CUDA(cudaGetLastError());
    vm_profile_count_kernels(1);
  }
  return VM_OK;
}
