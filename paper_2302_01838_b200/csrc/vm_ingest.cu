// Per-frame ingestion on the device:
//   decode   datasets.py:160-175   8-bit BGR / 16-bit depth / 16-bit instance
//                                  ids -> f32 RGB, f32 metres, int32 ids
//   stats    objects.py:188-201    per-instance pixel counts, valid-depth
//                                  counts and 2D bbox (one pass, atomics)
//   lift     objects.py:160-167    backprojection of every valid pixel of
//            objects.py:202-203    each kept instance (and of the stride-
//            objects.py:220-230    subsampled frame for scene_bounds) into a
//                                  per-(instance, axis) segment
//   trim     geometry.py:49-70     AABB.from_points: per-axis np.quantile
//                                  ('linear') after a segmented sort (CUB),
//                                  or min/max for <= 10 points, then the
//                                  min_extent widening
// The host keeps association, bookkeeping and keyframe decisions
// (objects.py:233-277, trainer.py:226-265): a handful of detections/frame.
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <vector>

#include "vm_common.cuh"

namespace vm {
namespace {

constexpr int kGT = 256;
constexpr int kMaxId = 65535;        // 16-bit instance masks (datasets.py: mask/%06d.png)
constexpr int kSlots = kMaxId + 1;

inline unsigned nblocks(int64_t n) { return unsigned((n + kGT - 1) / kGT); }

__global__ void decode_kernel(const uint8_t* __restrict__ bgr, const uint16_t* __restrict__ d16,
                              const uint16_t* __restrict__ m16, int64_t n, float depth_scale, float* __restrict__ rgb, float* __restrict__ depth,
                              int32_t* __restrict__ mask) {
  const int64_t i = blockIdx.x * int64_t(kGT) + threadIdx.x;
  if (i >= n) return;
  // rgb_bgr[:, :, ::-1].astype(np.float32) / 255.0  (f32 division)
  if (bgr) {
#pragma unroll
    for (int c = 0; c < 3; ++c) rgb[3 * i + c] = __fdiv_rn(float(bgr[3 * i + 2 - c]), 255.0f);
  }
  // depth_raw.astype(np.float32) / depth_scale  (f32 division by the f32 scalar)
  if (d16) depth[i] = __fdiv_rn(float(d16[i]), depth_scale);
  if (m16) mask[i] = int32_t(m16[i]);
}

struct Tables {
  int* cnt_all;     // [kSlots] pixels per id
  int* cnt_valid;   // [kSlots] pixels with depth > 0 per id
  int* u0; int* v0; int* u1; int* v1;  // [kSlots] bbox (half-open)
  int* seg;         // [kSlots] segment of a kept id, -1 otherwise
  int* n_scene;     // [1] stride-subsampled valid pixels
  int* present;     // [kSlots] compacted ids present in the frame
  int* n_present;   // [1]
  int* bad;         // [1] ids outside [0, 65535]
};

__global__ void stats_kernel(const float* __restrict__ depth, const int32_t* __restrict__ mask, int W, int H,
                             int stride, Tables t) {
  const int64_t i = blockIdx.x * int64_t(kGT) + threadIdx.x;
  if (i >= int64_t(W) * H) return;
  const int u = int(i % W), v = int(i / W);
  const float z = depth[i];
  if (z > 0.f && u % stride == 0 && v % stride == 0) atomicAdd(t.n_scene, 1);
  const int id = mask[i];
  if (id == 0) return;
  if (id < 0 || id > kMaxId) {
    atomicExch(t.bad, 1);
    return;
  }
  if (atomicAdd(&t.cnt_all[id], 1) == 0) t.present[atomicAdd(t.n_present, 1)] = id;
  if (z > 0.f) atomicAdd(&t.cnt_valid[id], 1);
  atomicMin(&t.u0[id], u);
  atomicMin(&t.v0[id], v);
  atomicMax(&t.u1[id], u + 1);
  atomicMax(&t.v1[id], v + 1);
}

struct Cam {
  double fx, fy, cx, cy, R[9], t[3];
};

// backproject (objects.py:160-167): x = (u - cx) / fx * z, y likewise,
// world = [x y z] @ R^T + t
__device__ __forceinline__ void lift(const Cam& c, int u, int v, float zf, double p[3]) {
  const double z = double(zf);
  const double x = __dmul_rn(__ddiv_rn(__dsub_rn(double(u), c.cx), c.fx), z);
  const double y = __dmul_rn(__ddiv_rn(__dsub_rn(double(v), c.cy), c.fy), z);
#pragma unroll
  for (int r = 0; r < 3; ++r)
    p[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, c.R[3 * r]), __dmul_rn(y, c.R[3 * r + 1])),
                               __dmul_rn(z, c.R[3 * r + 2])),
                     c.t[r]);
}

__global__ void scatter_kernel(const float* __restrict__ depth, const int32_t* __restrict__ mask, int W, int H,
                               int stride, Cam cam, Tables t, const int* __restrict__ seg_off, int scene_seg,
                               int* __restrict__ fill, int64_t total, double* __restrict__ keys) {
  const int64_t i = blockIdx.x * int64_t(kGT) + threadIdx.x;
  if (i >= int64_t(W) * H) return;
  const float z = depth[i];
  if (!(z > 0.f)) return;
  const int u = int(i % W), v = int(i / W);
  const int id = mask[i];
  const int s = (id > 0 && id <= kMaxId) ? t.seg[id] : -1;
  const bool scene = scene_seg >= 0 && u % stride == 0 && v % stride == 0;
  if (s < 0 && !scene) return;
  double p[3];
  lift(cam, u, v, z, p);
  if (s >= 0) {
    const int64_t j = seg_off[s] + atomicAdd(&fill[s], 1);
#pragma unroll
    for (int a = 0; a < 3; ++a) keys[a * total + j] = p[a];
  }
  if (scene) {
    const int64_t j = seg_off[scene_seg] + atomicAdd(&fill[scene_seg], 1);
#pragma unroll
    for (int a = 0; a < 3; ++a) keys[a * total + j] = p[a];
  }
}

// np.quantile(x, q) (method 'linear') on a sorted segment: v = (n-1) q,
// lerp(x[floor v], x[floor v + 1], v - floor v) with numpy's two-sided form
__device__ double quantile_sorted(const double* x, int64_t n, double q) {
  const double vi = __dmul_rn(double(n - 1), q);
  int64_t lo = int64_t(floor(vi)), hi = lo + 1;
  double prev_idx = floor(vi);
  if (vi >= double(n - 1)) {
    lo = hi = n - 1;
    prev_idx = -1.0;  // numpy sets previous_indexes = -1 before forming gamma
  } else if (vi < 0.0) {
    lo = hi = 0;
    prev_idx = 0.0;
  }
  const double a = x[lo], b = x[hi];
  const double gamma = __dsub_rn(vi, prev_idx);
  const double diff = __dsub_rn(b, a);
  return gamma >= 0.5 ? __dsub_rn(b, __dmul_rn(diff, __dsub_rn(1.0, gamma))) : __dadd_rn(a, __dmul_rn(diff, gamma));
}

// AABB.from_points (geometry.py:49-70) per segment and axis
__global__ void box_kernel(const double* __restrict__ sorted, const int* __restrict__ seg_off, int nseg,
                           int64_t total, double trim, double scene_trim, int scene_seg, double min_extent,
                           double* __restrict__ boxes) {
  const int j = blockIdx.x * kGT + threadIdx.x;
  if (j >= 3 * nseg) return;
  const int a = j / nseg, s = j % nseg;
  const int64_t b0 = seg_off[s], n = seg_off[s + 1] - seg_off[s];
  const double* x = sorted + a * total + b0;
  const double tr = s == scene_seg ? scene_trim : trim;
  double lo, hi;
  if (tr > 0.0 && n > 10) {
    lo = quantile_sorted(x, n, tr);
    hi = quantile_sorted(x, n, __dsub_rn(1.0, tr));
  } else {
    lo = x[0];
    hi = x[n - 1];
  }
  if (__dsub_rn(hi, lo) < min_extent) {
    lo = __dsub_rn(lo, __dmul_rn(0.5, min_extent));
    hi = __dadd_rn(hi, __dmul_rn(0.5, min_extent));
  }
  boxes[6 * s + a] = lo;
  boxes[6 * s + 3 + a] = hi;
}

__global__ void set_seg_kernel(const int* __restrict__ ids, int n, int* __restrict__ seg) {
  const int i = blockIdx.x * kGT + threadIdx.x;
  if (i < n) seg[ids[i]] = i;
}

struct WsPlan {
  size_t tables, keys, sorted, offs, fill, ids, boxes, cub, bytes;
  size_t cub_bytes;
};

WsPlan plan_ws(int W, int H) {
  const int64_t n = int64_t(W) * H;
  WsPlan p{};
  size_t off = 0;
  auto take = [&](size_t b) {
    const size_t o = off;
    off = (off + b + 255) / 256 * 256;
    return o;
  };
  p.tables = take(sizeof(int) * (size_t(kSlots) * 7 + 16));
  // every valid pixel lands in at most one instance segment plus the scene
  // segment: 2n points x 3 axes
  p.keys = take(sizeof(double) * size_t(2 * n) * 3);
  p.sorted = take(sizeof(double) * size_t(2 * n) * 3);
  p.offs = take(sizeof(int) * (2 * size_t(kSlots) + 8) * 3);
  p.fill = take(sizeof(int) * (size_t(kSlots) + 2));
  p.ids = take(sizeof(int) * (size_t(kSlots) + 2));
  p.boxes = take(sizeof(double) * 6 * (size_t(kSlots) + 2));
  // CUB temp storage for the largest possible call
  size_t cub_bytes = 0;
  cub::DeviceSegmentedSort::SortKeys(nullptr, cub_bytes, (const double*)nullptr, (double*)nullptr, int64_t(6 * n),
                                     int64_t(3 * (kSlots + 1)), (const int*)nullptr, (const int*)nullptr);
  p.cub_bytes = cub_bytes;
  p.cub = take(cub_bytes + 256);
  p.bytes = off;
  return p;
}

Tables carve_tables(char* base) {
  int* t = reinterpret_cast<int*>(base);
  Tables tb;
  tb.cnt_all = t;
  tb.cnt_valid = t + kSlots;
  tb.u0 = t + 2 * kSlots;
  tb.v0 = t + 3 * kSlots;
  tb.u1 = t + 4 * kSlots;
  tb.v1 = t + 5 * kSlots;
  tb.seg = t + 6 * kSlots;
  tb.present = nullptr;  // set by the caller (ids buffer)
  tb.n_scene = t + 7 * kSlots;
  tb.n_present = t + 7 * kSlots + 1;
  tb.bad = t + 7 * kSlots + 2;
  return tb;
}

}  // namespace
}  // namespace vm

using namespace vm;

extern "C" int vm_decode_frame(const uint8_t* bgr, const uint16_t* depth16, const uint16_t* mask16, int32_t width,
                               int32_t height, double depth_scale, float* rgb, float* depth, int32_t* mask,
                               void* stream) {
  VM_REQUIRE(width > 0 && height > 0 && depth_scale > 0, "vm_decode_frame: bad arguments");
  VM_REQUIRE((!bgr || rgb) && (!depth16 || depth) && (!mask16 || mask), "vm_decode_frame: missing output");
  const int64_t n = int64_t(width) * height;
  decode_kernel<<<nblocks(n), kGT, 0, cudaStream_t(stream)>>>(bgr, depth16, mask16, n, float(depth_scale), rgb,
                                                              depth, mask);
  VM_CUDA(cudaGetLastError());
  return VM_OK;
}

extern "C" size_t vm_ingest_workspace_bytes(int32_t width, int32_t height) {
  if (width <= 0 || height <= 0) return 0;
  return plan_ws(width, height).bytes;
}

extern "C" int vm_ingest_frame(const float* depth, const int32_t* mask, int32_t width, int32_t height,
                               const double* intr, const double* pose, int32_t min_pixels, double trim,
                               int32_t scene_stride, double scene_trim, VmDetection* out, int32_t capacity,
                               int32_t* n_out, double* scene_box, int32_t* scene_ok, void* workspace,
                               size_t workspace_bytes, void* stream) {
  VM_REQUIRE(depth && mask && intr && pose && out && n_out && scene_box && scene_ok && workspace,
             "vm_ingest_frame: null argument");
  VM_REQUIRE(width > 0 && height > 0 && scene_stride >= 1, "vm_ingest_frame: bad frame size / stride");
  VM_REQUIRE(trim >= 0.0 && trim < 0.5 && scene_trim >= 0.0 && scene_trim < 0.5,
             "vm_ingest_frame: trim must be in [0, 0.5)");
  const WsPlan pl = plan_ws(width, height);
  VM_REQUIRE(workspace_bytes >= pl.bytes, "vm_ingest_frame: workspace too small");
  cudaStream_t s = cudaStream_t(stream);
  char* ws = static_cast<char*>(workspace);
  Tables tb = carve_tables(ws + pl.tables);
  int* ids = reinterpret_cast<int*>(ws + pl.ids);
  tb.present = ids;
  const int64_t n = int64_t(width) * height;
  // counts / seg (-1) / bbox sentinels
  VM_CUDA(cudaMemsetAsync(tb.cnt_all, 0, sizeof(int) * 2 * kSlots, s));
  VM_CUDA(cudaMemsetAsync(tb.u0, 0x7f, sizeof(int) * 2 * kSlots, s));
  VM_CUDA(cudaMemsetAsync(tb.u1, 0, sizeof(int) * 2 * kSlots, s));
  VM_CUDA(cudaMemsetAsync(tb.seg, 0xff, sizeof(int) * kSlots, s));
  VM_CUDA(cudaMemsetAsync(tb.n_scene, 0, sizeof(int) * 16, s));
  stats_kernel<<<nblocks(n), kGT, 0, s>>>(depth, mask, width, height, scene_stride, tb);
  VM_CUDA(cudaGetLastError());
  int head[3];
  VM_CUDA(cudaMemcpyAsync(head, tb.n_scene, sizeof(int) * 3, cudaMemcpyDeviceToHost, s));
  VM_CUDA(cudaStreamSynchronize(s));
  VM_REQUIRE(head[2] == 0, "vm_ingest_frame: instance id outside [0, 65535]");
  const int n_scene = head[0], n_present = head[1];
  // per present id: count, valid count, bbox (one small gather on the host side)
  std::vector<int> present(n_present);
  std::vector<int> stats(size_t(6) * kSlots);
  if (n_present) {
    VM_CUDA(cudaMemcpyAsync(present.data(), ids, sizeof(int) * n_present, cudaMemcpyDeviceToHost, s));
    VM_CUDA(cudaMemcpyAsync(stats.data(), tb.cnt_all, sizeof(int) * 6 * kSlots, cudaMemcpyDeviceToHost, s));
    VM_CUDA(cudaStreamSynchronize(s));
  }
  std::sort(present.begin(), present.end());  // np.unique order
  std::vector<int> kept;
  std::vector<int> offs(1, 0);
  for (int id : present) {
    if (stats[size_t(kSlots) + id] < min_pixels) continue;
    kept.push_back(id);
    offs.push_back(offs.back() + stats[size_t(kSlots) + id]);
  }
  const bool want_scene = n_scene >= 16;  // scene_bounds returns None below 16 points
  const int scene_seg = want_scene ? int(kept.size()) : -1;
  if (want_scene) offs.push_back(offs.back() + n_scene);
  const int nseg = int(offs.size()) - 1;
  const int64_t total = offs.back();
  VM_REQUIRE(int64_t(kept.size()) <= int64_t(capacity), "vm_ingest_frame: detection capacity too small");
  *n_out = int32_t(kept.size());
  *scene_ok = want_scene ? 1 : 0;
  if (nseg == 0) return VM_OK;
  int* seg_off = reinterpret_cast<int*>(ws + pl.offs);
  int* fill = reinterpret_cast<int*>(ws + pl.fill);
  double* keys = reinterpret_cast<double*>(ws + pl.keys);
  double* sorted = reinterpret_cast<double*>(ws + pl.sorted);
  double* boxes = reinterpret_cast<double*>(ws + pl.boxes);
  // segment begin/end offsets of the 3*nseg sort segments (axis-major)
  std::vector<int> beg(3 * nseg), end(3 * nseg);
  for (int a = 0; a < 3; ++a)
    for (int g = 0; g < nseg; ++g) {
      beg[a * nseg + g] = int(a * total + offs[g]);
      end[a * nseg + g] = int(a * total + offs[g + 1]);
    }
  VM_REQUIRE(3 * total < int64_t(INT32_MAX), "vm_ingest_frame: frame too large");
  int* d_beg = seg_off + (nseg + 1);
  int* d_end = d_beg + 3 * nseg;
  VM_CUDA(cudaMemcpyAsync(seg_off, offs.data(), sizeof(int) * (nseg + 1), cudaMemcpyHostToDevice, s));
  VM_CUDA(cudaMemcpyAsync(d_beg, beg.data(), sizeof(int) * 3 * nseg, cudaMemcpyHostToDevice, s));
  VM_CUDA(cudaMemcpyAsync(d_end, end.data(), sizeof(int) * 3 * nseg, cudaMemcpyHostToDevice, s));
  if (!kept.empty()) {
    VM_CUDA(cudaMemcpyAsync(ids, kept.data(), sizeof(int) * kept.size(), cudaMemcpyHostToDevice, s));
    set_seg_kernel<<<nblocks(int64_t(kept.size())), kGT, 0, s>>>(ids, int(kept.size()), tb.seg);
  }
  VM_CUDA(cudaMemsetAsync(fill, 0, sizeof(int) * (nseg + 1), s));
  Cam cam{};
  cam.fx = intr[0];
  cam.fy = intr[1];
  cam.cx = intr[2];
  cam.cy = intr[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) cam.R[3 * r + c] = pose[4 * r + c];
    cam.t[r] = pose[4 * r + 3];
  }
  scatter_kernel<<<nblocks(n), kGT, 0, s>>>(depth, mask, width, height, scene_stride, cam, tb, seg_off, scene_seg,
                                            fill, total, keys);
  VM_CUDA(cudaGetLastError());
  size_t cub_bytes = pl.cub_bytes;
  VM_CUDA(cub::DeviceSegmentedSort::SortKeys(ws + pl.cub, cub_bytes, keys, sorted, int64_t(3 * total),
                                             int64_t(3 * nseg), d_beg, d_end, s));
  box_kernel<<<nblocks(3 * nseg), kGT, 0, s>>>(sorted, seg_off, nseg, total, trim, scene_trim, scene_seg, 1e-3,
                                               boxes);
  VM_CUDA(cudaGetLastError());
  std::vector<double> hb(size_t(6) * nseg);
  VM_CUDA(cudaMemcpyAsync(hb.data(), boxes, sizeof(double) * 6 * nseg, cudaMemcpyDeviceToHost, s));
  VM_CUDA(cudaStreamSynchronize(s));
  for (size_t k = 0; k < kept.size(); ++k) {
    const int id = kept[k];
    VmDetection& d = out[k];
    d.instance_id = id;
    d.n_pixels = stats[id];
    d.n_valid = stats[size_t(kSlots) + id];
    d.u0 = stats[2 * size_t(kSlots) + id];
    d.v0 = stats[3 * size_t(kSlots) + id];
    d.u1 = stats[4 * size_t(kSlots) + id];
    d.v1 = stats[5 * size_t(kSlots) + id];
    for (int a = 0; a < 3; ++a) {
      d.box_min[a] = hb[6 * k + a];
      d.box_max[a] = hb[6 * k + 3 + a];
    }
  }
  if (want_scene)
    for (int a = 0; a < 6; ++a) scene_box[a] = hb[6 * size_t(scene_seg) + a];
  return VM_OK;
}
