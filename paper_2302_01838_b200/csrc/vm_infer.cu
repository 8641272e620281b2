// Forward-only inference for meshing and novel views:
//   query_grid  (meshing.py:64-97)   occupancy of one model on a regular grid
//   _eval_field (meshing.py:453-476) occupancy/colour at per-ray samples
//   render_view (meshing.py:485-579) coarse + refined background, objects
//                                    composited by depth per pixel
// The MLP evaluation reuses the fused FFMA forward kernel (vm_forward, one
// model viewed as a 1-model stack); everything around it -- grid and ray
// sample generation, the f32 positional encoding exactly as the reference's
// inference path computes it (f32 points, f32 centre/half, f32 band
// coefficients), ray/box selection, per-ray compositing and the per-pixel
// depth competition -- runs in the kernels below.  Large point sets are
// processed in chunks through one workspace (no host round trips except the
// hit count of an object's ray selection).
#include <algorithm>
#include <cmath>

#include "vm_common.cuh"

namespace vm {
namespace {

constexpr int kIT = 256;

inline unsigned blocks_for(int64_t n) { return unsigned((n + kIT - 1) / kIT); }

// numpy pairwise summation (f64 / f32) for n <= 128: 8 accumulators, see
// vm_common.cuh pairwise_sum_leaf.
template <typename T, typename F>
__device__ T pw_leaf(const F& get, int n) {
  if (n < 8) {
    T r = T(-0.0);
    for (int i = 0; i < n; ++i) r = r + get(i);
    return r;
  }
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = get(j);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = r[j] + get(i + j);
  T res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res = res + get(i);
  return res;
}

template <typename T, typename F>
__device__ T pw_sum(const F& get, int i0, int n) {
  if (n <= 128) return pw_leaf<T>([&](int i) { return get(i0 + i); }, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pw_sum<T>(get, i0, n2) + pw_sum<T>(get, i0 + n2, n - n2);
}

// np.linspace(lo, hi, num)[i] (numpy 2: i * step + start, last = stop)
__device__ __forceinline__ double linspace_at(double lo, double hi, int num, int i) {
  if (num == 1) return lo;
  if (i == num - 1) return hi;
  const double step = __ddiv_rn(__dsub_rn(hi, lo), double(num - 1));
  return __dadd_rn(__dmul_rn(double(i), step), lo);
}

// meshgrid(ij) of the three linspaces, flattened C-order, cast to f32
__global__ void grid_points_kernel(double3 bmin, double3 bmax, int rx, int ry, int rz, int64_t start, int64_t n,
                                   float* __restrict__ pts) {
  const int64_t i = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (i >= n) return;
  const int64_t f = start + i;
  const int iz = int(f % rz), iy = int((f / rz) % ry), ix = int(f / (int64_t(ry) * rz));
  pts[3 * i + 0] = float(linspace_at(bmin.x, bmax.x, rx, ix));
  pts[3 * i + 1] = float(linspace_at(bmin.y, bmax.y, ry, iy));
  pts[3 * i + 2] = float(linspace_at(bmin.z, bmax.z, rz, iz));
}

// positional_encode (models.py:286-308) on f32 points as query_grid /
// _eval_field call it: centre/half cast to f32, p = (x - c) / h in f32, the
// band coefficient pi * 2^i / scale formed in f64 and used as an f32 scalar,
// sin/cos in f32.
struct PE32 {
  float c[3], h[3], coef[16];
  int n_freq, include, D;
};

__global__ void encode_f32_kernel(const float* __restrict__ pts, int64_t n, PE32 pe, float* __restrict__ enc) {
  const int64_t i = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (i >= n) return;
  float p[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) p[c] = __fdiv_rn(__fsub_rn(pts[3 * i + c], pe.c[c]), pe.h[c]);
  float* out = enc + i * pe.D;
  int f = 0;
  if (pe.include) {
#pragma unroll
    for (int c = 0; c < 3; ++c) out[c] = p[c];
    f = 3;
  }
  for (int b = 0; b < pe.n_freq; ++b) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float a = __fmul_rn(pe.coef[b], p[c]);
      float sn, cs;
      sincosf(a, &sn, &cs);
      out[f + 6 * b + c] = sn;
      out[f + 6 * b + 3 + c] = cs;
    }
  }
}

// pixel rays of a camera (render_view, meshing.py:516-526): directions
// d_cam @ R^T normalised, and the z-depth -> ray-distance scale |d_cam|
struct Cam {
  double fx, fy, cx, cy;
  double R[9], o[3];
  int w, h;
};

__global__ void view_rays_kernel(Cam cam, double* __restrict__ dirs, double* __restrict__ scale) {
  const int64_t i = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (i >= int64_t(cam.w) * cam.h) return;
  const int u = int(i % cam.w), v = int(i / cam.w);
  const double d0 = __ddiv_rn(__dsub_rn(double(u), cam.cx), cam.fx);
  const double d1 = __ddiv_rn(__dsub_rn(double(v), cam.cy), cam.fy);
  scale[i] = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), 1.0));
  double d[3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    d[r] = __dadd_rn(__dadd_rn(__dmul_rn(d0, cam.R[3 * r + 0]), __dmul_rn(d1, cam.R[3 * r + 1])), cam.R[3 * r + 2]);
  const double nn = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
#pragma unroll
  for (int r = 0; r < 3; ++r) dirs[3 * i + r] = __ddiv_rn(d[r], nn);
}

// ray_box_intersect (render.py:111-139) + render_view's selection
// t0 = max(t0, t_near); hit & (t1 > t0) (meshing.py:562-565).  Selected
// rays are compacted (order irrelevant: results are scattered back by index).
__global__ void ray_box_select_kernel(double3 o, const double* __restrict__ dirs, int64_t n, double3 bmin,
                                      double3 bmax, double t_near, int* __restrict__ sel, int* __restrict__ count,
                                      double* __restrict__ lo, double* __restrict__ hi) {
  const int64_t i = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (i >= n) return;
  const double oo[3] = {o.x, o.y, o.z}, mn[3] = {bmin.x, bmin.y, bmin.z}, mx[3] = {bmax.x, bmax.y, bmax.z};
  double tin = -INFINITY, tout = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double d = dirs[3 * i + a];
    double l, h;
    if (d == 0.0) {
      const bool inside = oo[a] >= mn[a] && oo[a] <= mx[a];
      l = inside ? -INFINITY : INFINITY;
      h = inside ? INFINITY : -INFINITY;
    } else {
      const double inv = 1.0 / d;
      const double ta = (mn[a] - oo[a]) * inv, tb = (mx[a] - oo[a]) * inv;
      l = fmin(ta, tb);
      h = fmax(ta, tb);
      if (ta != ta || tb != tb) l = h = NAN;
    }
    tin = a == 0 ? l : (tin != tin || l != l ? NAN : fmax(tin, l));
    tout = a == 0 ? h : (tout != tout || h != h ? NAN : fmin(tout, h));
  }
  const double t_entry = tin != tin ? tin : fmax(tin, 0.0);
  const bool hit = (tout >= t_entry) && (tout >= 0.0);
  const double t0 = t_entry != t_entry ? t_entry : fmax(t_entry, t_near);
  if (hit && tout > t0) {
    const int j = atomicAdd(count, 1);
    sel[j] = int(i);
    lo[j] = t0;
    hi[j] = tout;
  }
}

// _midpoints (meshing.py:479-482) and the sample points origin + t * dir,
// cast to f32 as _eval_field does (meshing.py:468)
__global__ void ray_points_kernel(double3 o, const double* __restrict__ dirs, const int* __restrict__ sel,
                                  const double* __restrict__ lo, const double* __restrict__ hi, double lo_c,
                                  double hi_c, int64_t r0, int64_t n, int S, float* __restrict__ pts,
                                  double* __restrict__ t) {
  const int64_t i = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (i >= n * S) return;
  const int64_t r = r0 + i / S;
  const int s = int(i % S);
  const int64_t ray = sel ? sel[r] : r;
  const double l = lo ? lo[r] : lo_c, h = hi ? hi[r] : hi_c;
  const double centre = __ddiv_rn(__dadd_rn(double(s), 0.5), double(S));
  const double tt = __dadd_rn(l, __dmul_rn(centre, __dsub_rn(h, l)));
  t[i] = tt;
  const double oo[3] = {o.x, o.y, o.z};
#pragma unroll
  for (int c = 0; c < 3; ++c) pts[3 * i + c] = float(__dadd_rn(oo[c], __dmul_rn(tt, dirs[3 * ray + c])));
}

// render_rays (render.py:230-246) on inference samples: f32 occupancy /
// colour, f64 t (so depth is f64, as in render_view)
__global__ void composite_kernel(const float* __restrict__ occ, const float* __restrict__ col,
                                 const double* __restrict__ t, int64_t n, int S, float* __restrict__ opacity,
                                 double* __restrict__ depth, float* __restrict__ colour, int64_t out0) {
  const int64_t r = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (r >= n) return;
  const float* o = occ + r * S;
  float w[128];
  float tr = 1.0f;
  for (int i = 0; i < S; ++i) {
    w[i] = __fmul_rn(o[i], tr);
    tr = __fmul_rn(tr, __fsub_rn(1.0f, o[i]));
  }
  opacity[out0 + r] = pw_sum<float>([&](int i) { return w[i]; }, 0, S);
  depth[out0 + r] = pw_sum<double>([&](int i) { return double(w[i]) * t[r * S + i]; }, 0, S);
  for (int c = 0; c < 3; ++c) {
    float acc = __fmul_rn(w[0], col[(r * S) * 3 + c]);
    for (int i = 1; i < S; ++i) acc = __fadd_rn(acc, __fmul_rn(w[i], col[(r * S + i) * 3 + c]));
    colour[(out0 + r) * 3 + c] = acc;
  }
}

// refinement window around the coarse depth (meshing.py:540-543)
__global__ void refine_window_kernel(const double* __restrict__ depth, int64_t n, double t_near, double t_far,
                                     double rw, double* __restrict__ lo, double* __restrict__ hi) {
  const int64_t i = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (i >= n) return;
  const double c = fmin(fmax(depth[i], t_near + rw), t_far - rw);
  lo[i] = fmax(c - rw, t_near);
  hi[i] = fmin(c + rw, t_far);
}

// background choice + per-pixel state init (meshing.py:547-556)
__global__ void bg_select_kernel(int64_t n, const float* __restrict__ c_op, const double* __restrict__ c_dep,
                                 const float* __restrict__ c_col, const double* __restrict__ r_dep,
                                 const float* __restrict__ r_col, int refined, double* __restrict__ depth,
                                 double* __restrict__ colour, int* __restrict__ instance, double* __restrict__ best) {
  const int64_t i = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (i >= n) return;
  const bool use = refined && c_op[i] >= 0.5f;
  depth[i] = use ? r_dep[i] : c_dep[i];
#pragma unroll
  for (int c = 0; c < 3; ++c) colour[3 * i + c] = double(use ? r_col[3 * i + c] : c_col[3 * i + c]);
  instance[i] = 0;
  best[i] = INFINITY;
}

// depth competition of one object over its selected rays (meshing.py:569-574)
__global__ void object_winner_kernel(int64_t n, const int* __restrict__ sel, const float* __restrict__ op,
                                     const double* __restrict__ dep, const float* __restrict__ col, float thr,
                                     int object_id, double* __restrict__ best, double* __restrict__ depth,
                                     double* __restrict__ colour, int* __restrict__ instance) {
  const int64_t j = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (j >= n) return;
  const int i = sel[j];
  if (op[j] >= thr && dep[j] < best[i]) {
    best[i] = dep[j];
    depth[i] = dep[j];
#pragma unroll
    for (int c = 0; c < 3; ++c) colour[3 * i + c] = double(col[3 * j + c]);
    instance[i] = object_id;
  }
}

// z-depth, clipped colour, f32 outputs (meshing.py:576-581)
__global__ void view_finish_kernel(int64_t n, const double* __restrict__ depth, const double* __restrict__ scale,
                                   const double* __restrict__ colour, float* __restrict__ rgb,
                                   float* __restrict__ z) {
  const int64_t i = blockIdx.x * int64_t(kIT) + threadIdx.x;
  if (i >= n) return;
  z[i] = float(depth[i] / scale[i]);
#pragma unroll
  for (int c = 0; c < 3; ++c) rgb[3 * i + c] = float(fmin(fmax(colour[3 * i + c], 0.0), 1.0));
}

PE32 make_pe(const double* center, const double* half, double pe_scale, int n_freq, int include, int D) {
  PE32 pe{};
  for (int c = 0; c < 3; ++c) {
    pe.c[c] = float(center[c]);
    pe.h[c] = float(half[c]);
  }
  for (int b = 0; b < n_freq && b < 16; ++b) pe.coef[b] = float((M_PI * std::ldexp(1.0, b)) / pe_scale);
  pe.n_freq = n_freq;
  pe.include = include;
  pe.D = D;
  return pe;
}

int arch_pe(const VmArch& a, int& n_freq, int& include) {
  include = a.input_dim % 6 == 3 ? 1 : 0;
  n_freq = (a.input_dim - 3 * include) / 6;
  if (n_freq > 16 || 3 * include + 6 * n_freq != a.input_dim) return VM_ERR_SHAPE;
  return VM_OK;
}

// one model of a stack as a 1-model stack view
VmStack model_view(const VmStack& st, int index, int64_t block) {
  VmStack v = st;
  v.count = 1;
  v.capacity = 1;
  v.params = st.params + int64_t(index) * block;
  v.m = v.v = nullptr;
  v.step = nullptr;
  v.frozen = nullptr;
  return v;
}

}  // namespace
}  // namespace vm

using namespace vm;

extern "C" size_t vm_infer_workspace_bytes(const VmArch* arch, int64_t chunk) {
  if (!arch || chunk <= 0) return 0;
  // points f32 [chunk,3] + encoded f32 [chunk,D] + occ [chunk] + col [chunk,3] + t f64 [chunk]
  // + the tensor-core forward's weight image (hidden-128 models)
  return size_t(chunk) * (12 + 4 * size_t(arch->input_dim) + 4 + 12 + 8) + 1024 + fwd_image_bytes(*arch) + 256;
}

namespace {
struct InferWs {
  float *pts, *enc, *occ, *col, *img;
  double* t;
};
InferWs carve(void* ws, int64_t chunk, int D, size_t img_bytes) {
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t b) {
    char* r = p;
    p += (b + 255) / 256 * 256;
    return r;
  };
  InferWs w;
  w.t = reinterpret_cast<double*>(take(size_t(chunk) * 8));
  w.pts = reinterpret_cast<float*>(take(size_t(chunk) * 12));
  w.enc = reinterpret_cast<float*>(take(size_t(chunk) * 4 * D));
  w.occ = reinterpret_cast<float*>(take(size_t(chunk) * 4));
  w.col = reinterpret_cast<float*>(take(size_t(chunk) * 12));
  w.img = img_bytes ? reinterpret_cast<float*>(take(img_bytes)) : nullptr;
  return w;
}
}  // namespace

extern "C" int vm_forward(const VmStack* st, const float* encoded, int64_t n_samples, float* occ, float* col,
                          void* stream);

extern "C" int vm_query_grid(const VmStack* stack, int32_t model_index, const double* box_min,
                             const double* box_max, double pe_scale, const int32_t* resolution, float* occ_out,
                             void* workspace, size_t workspace_bytes, int64_t chunk, void* stream) {
  VM_REQUIRE(stack && box_min && box_max && resolution && occ_out && workspace, "vm_query_grid: null argument");
  VM_REQUIRE(model_index >= 0 && model_index < stack->count, "vm_query_grid: model index out of range");
  VM_REQUIRE(resolution[0] >= 2 && resolution[1] >= 2 && resolution[2] >= 2,
             "vm_query_grid: grid resolution must be >= 2 per axis");
  VM_REQUIRE(pe_scale > 0, "vm_query_grid: scale must be positive");
  VM_REQUIRE(workspace_bytes >= vm_infer_workspace_bytes(&stack->arch, chunk), "vm_query_grid: workspace too small");
  VmLayout L;
  VM_REQUIRE(compute_layout(stack->arch, L) == VM_OK, "vm_query_grid: unsupported architecture");
  int nf, inc;
  VM_REQUIRE(arch_pe(stack->arch, nf, inc) == VM_OK, "vm_query_grid: input_dim is not a PE width");
  double c[3], h[3];
  for (int i = 0; i < 3; ++i) {
    c[i] = 0.5 * (box_min[i] + box_max[i]);
    h[i] = 0.5 * (box_max[i] - box_min[i]);
    VM_REQUIRE(h[i] > 0, "vm_query_grid: half_extent must be positive");
  }
  const PE32 pe = make_pe(c, h, pe_scale, nf, inc, stack->arch.input_dim);
  const VmStack view = model_view(*stack, model_index, L.block);
  cudaStream_t s = cudaStream_t(stream);
  const InferWs w = carve(workspace, chunk, stack->arch.input_dim, fwd_image_bytes(stack->arch));
  const int64_t total = int64_t(resolution[0]) * resolution[1] * resolution[2];
  const double3 bmin = make_double3(box_min[0], box_min[1], box_min[2]);
  const double3 bmax = make_double3(box_max[0], box_max[1], box_max[2]);
  for (int64_t start = 0; start < total; start += chunk) {
    const int64_t n = std::min(chunk, total - start);
    grid_points_kernel<<<blocks_for(n), kIT, 0, s>>>(bmin, bmax, resolution[0], resolution[1], resolution[2], start,
                                                     n, w.pts);
    encode_f32_kernel<<<blocks_for(n), kIT, 0, s>>>(w.pts, n, pe, w.enc);
    VM_CUDA(cudaGetLastError());
    const int rc = forward_ws(&view, w.enc, n, occ_out + start, w.col, w.img, s);
    if (rc) return rc;
  }
  return VM_OK;
}

extern "C" int vm_eval_rays(const VmStack* stack, int32_t model_index, const double* box_min, const double* box_max,
                            double pe_scale, const double* origin, const double* dirs, const int32_t* sel,
                            int64_t n_rays, const double* lo, const double* hi, double lo_const, double hi_const,
                            int32_t n_samples, float* opacity, double* depth, float* colour, void* workspace,
                            size_t workspace_bytes, int64_t chunk, void* stream) {
  VM_REQUIRE(stack && box_min && box_max && origin && dirs && opacity && depth && colour && workspace,
             "vm_eval_rays: null argument");
  VM_REQUIRE(model_index >= 0 && model_index < stack->count, "vm_eval_rays: model index out of range");
  VM_REQUIRE(n_samples >= 1 && n_samples <= 128, "vm_eval_rays: 1..128 samples per ray");
  VM_REQUIRE(chunk >= n_samples, "vm_eval_rays: chunk smaller than one ray");
  VM_REQUIRE(workspace_bytes >= vm_infer_workspace_bytes(&stack->arch, chunk), "vm_eval_rays: workspace too small");
  VmLayout L;
  VM_REQUIRE(compute_layout(stack->arch, L) == VM_OK, "vm_eval_rays: unsupported architecture");
  int nf, inc;
  VM_REQUIRE(arch_pe(stack->arch, nf, inc) == VM_OK, "vm_eval_rays: input_dim is not a PE width");
  double c[3], h[3];
  for (int i = 0; i < 3; ++i) {
    c[i] = 0.5 * (box_min[i] + box_max[i]);
    h[i] = 0.5 * (box_max[i] - box_min[i]);
  }
  const PE32 pe = make_pe(c, h, pe_scale, nf, inc, stack->arch.input_dim);
  const VmStack view = model_view(*stack, model_index, L.block);
  cudaStream_t s = cudaStream_t(stream);
  const InferWs w = carve(workspace, chunk, stack->arch.input_dim, fwd_image_bytes(stack->arch));
  const double3 o = make_double3(origin[0], origin[1], origin[2]);
  const int64_t rays_per = chunk / n_samples;
  for (int64_t r0 = 0; r0 < n_rays; r0 += rays_per) {
    const int64_t n = std::min(rays_per, n_rays - r0);
    const int64_t ns = n * n_samples;
    ray_points_kernel<<<blocks_for(ns), kIT, 0, s>>>(o, dirs, sel, lo, hi, lo_const, hi_const, r0, n, n_samples,
                                                     w.pts, w.t);
    encode_f32_kernel<<<blocks_for(ns), kIT, 0, s>>>(w.pts, ns, pe, w.enc);
    VM_CUDA(cudaGetLastError());
    int rc = forward_ws(&view, w.enc, ns, w.occ, w.col, w.img, cudaStream_t(stream));
    if (rc) return rc;
    composite_kernel<<<blocks_for(n), kIT, 0, s>>>(w.occ, w.col, w.t, n, n_samples, opacity, depth, colour, r0);
    VM_CUDA(cudaGetLastError());
  }
  return VM_OK;
}

extern "C" int vm_view_rays(const double* intr, int32_t width, int32_t height, const double* pose, double* dirs,
                            double* scale, void* stream) {
  VM_REQUIRE(intr && pose && dirs && scale && width > 0 && height > 0, "vm_view_rays: bad arguments");
  Cam cam{};
  cam.fx = intr[0];
  cam.fy = intr[1];
  cam.cx = intr[2];
  cam.cy = intr[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) cam.R[3 * r + c] = pose[4 * r + c];
    cam.o[r] = pose[4 * r + 3];
  }
  cam.w = width;
  cam.h = height;
  const int64_t n = int64_t(width) * height;
  view_rays_kernel<<<blocks_for(n), kIT, 0, cudaStream_t(stream)>>>(cam, dirs, scale);
  VM_CUDA(cudaGetLastError());
  return VM_OK;
}

extern "C" int vm_ray_box_select(const double* origin, const double* dirs, int64_t n, const double* box_min,
                                 const double* box_max, double t_near, int32_t* sel, int32_t* count, double* lo,
                                 double* hi, void* stream) {
  VM_REQUIRE(origin && dirs && box_min && box_max && sel && count && lo && hi, "vm_ray_box_select: null argument");
  cudaStream_t s = cudaStream_t(stream);
  VM_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t), s));
  if (n == 0) return VM_OK;
  ray_box_select_kernel<<<blocks_for(n), kIT, 0, s>>>(make_double3(origin[0], origin[1], origin[2]), dirs, n,
                                                      make_double3(box_min[0], box_min[1], box_min[2]),
                                                      make_double3(box_max[0], box_max[1], box_max[2]), t_near, sel,
                                                      count, lo, hi);
  VM_CUDA(cudaGetLastError());
  return VM_OK;
}

extern "C" int vm_view_compose(int32_t op, int64_t n, const void* a0, const void* a1, const void* a2,
                               const void* a3, const void* a4, const void* a5, double p0, double p1, double p2,
                               int32_t i0, void* o0, void* o1, void* o2, void* o3, void* stream) {
  cudaStream_t s = cudaStream_t(stream);
  if (n <= 0) return VM_OK;
  switch (op) {
    case 0:  // refine window: a0 = coarse depth; p = t_near, t_far, window -> o0 = lo, o1 = hi
      refine_window_kernel<<<blocks_for(n), kIT, 0, s>>>((const double*)a0, n, p0, p1, p2, (double*)o0, (double*)o1);
      break;
    case 1:  // background choice: a0..a4 = coarse op/depth/colour, refined depth/colour; i0 = refined?
      bg_select_kernel<<<blocks_for(n), kIT, 0, s>>>(n, (const float*)a0, (const double*)a1, (const float*)a2,
                                                     (const double*)a3, (const float*)a4, i0, (double*)o0,
                                                     (double*)o1, (int*)o2, (double*)o3);
      break;
    case 2:  // object winner: a0 = sel, a1..a3 = opacity/depth/colour; p0 = threshold; i0 = object id
      object_winner_kernel<<<blocks_for(n), kIT, 0, s>>>(n, (const int*)a0, (const float*)a1, (const double*)a2,
                                                         (const float*)a3, float(p0), i0, (double*)o0, (double*)o1,
                                                         (double*)o2, (int*)o3);
      break;
    case 3:  // finish: a0 = depth along, a1 = scale, a2 = colour -> o0 = rgb f32, o1 = z f32
      view_finish_kernel<<<blocks_for(n), kIT, 0, s>>>(n, (const double*)a0, (const double*)a1, (const double*)a2,
                                                       (float*)o0, (float*)o1);
      break;
    default:
      VM_REQUIRE(false, "vm_view_compose: unknown op");
  }
  VM_CUDA(cudaGetLastError());
  return VM_OK;
}
