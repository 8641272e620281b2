// VOBJ v1 checkpoint sections straight from / into the device arena
// (checkpoint.py:51-84).  One launch gathers a stack's live
// parameters and Adam moments from the padded model-major arena into the
// exact byte order of the reference's stack section -- per layer weights
// [K, fan_out, fan_in] then biases [K, fan_out]; then per layer m_w, v_w,
// m_b, v_b -- so the host writes it with a single D2H copy; the inverse
// launch scatters a loaded section back into the arena (padding untouched).
#include "vm_common.cuh"

namespace vm {
namespace {

constexpr int kCT = 256;
constexpr int kMaxSeg = 6 * VM_MAX_LAYERS;

struct Seg {
  int which;              // 0 params, 1 Adam m, 2 Adam v arena (per-model stride `block`)
  int64_t off;            // float offset inside a model block
  int64_t out0;           // first float of this segment in the packed section
  int fo, fi, fi_pad;     // rows, live columns, arena row length
};

struct PackPlan {
  Seg seg[kMaxSeg];
  int n;
  int K;
  int64_t block;
  int64_t total;
};

__global__ void pack_kernel(const __grid_constant__ PackPlan p, float* __restrict__ packed, float* __restrict__ arena_p,
                            float* __restrict__ arena_m, float* __restrict__ arena_v, int unpack) {
  const int64_t i = blockIdx.x * int64_t(kCT) + threadIdx.x;
  if (i >= p.total) return;
  int s = 0;
  while (s + 1 < p.n && p.seg[s + 1].out0 <= i) ++s;
  const Seg& g = p.seg[s];
  const int64_t r = i - g.out0;
  const int64_t per = int64_t(g.fo) * g.fi;
  const int64_t k = r / per, e = r % per;
  const int64_t o = e / g.fi, c = e % g.fi;
  const int64_t a = k * p.block + g.off + o * g.fi_pad + c;
  float* base = g.which == 0 ? arena_p : (g.which == 1 ? arena_m : arena_v);
  if (unpack) base[a] = packed[i];
  else packed[i] = base[a];
}

int plan_pack(const VmStack& st, PackPlan& p) {
  VmLayout L;
  if (compute_layout(st.arch, L)) return VM_ERR_UNSUPPORTED;
  p = PackPlan{};
  p.K = st.count;
  p.block = L.block;
  int64_t out = 0;
  auto add = [&](int which, int64_t off, int fo, int fi, int fi_pad) {
    Seg& g = p.seg[p.n++];
    g.which = which;
    g.off = off;
    g.out0 = out;
    g.fo = fo;
    g.fi = fi;
    g.fi_pad = fi_pad;
    out += int64_t(st.count) * fo * fi;
  };
  for (int l = 0; l < L.n_layers; ++l) {
    add(0, L.w_off[l], L.fo[l], L.fi[l], L.fi_pad[l]);
    add(0, L.b_off[l], 1, L.fo[l], L.fo_pad[l]);  // biases as one row of fan_out
  }
  for (int l = 0; l < L.n_layers; ++l) {
    add(1, L.w_off[l], L.fo[l], L.fi[l], L.fi_pad[l]);
    add(2, L.w_off[l], L.fo[l], L.fi[l], L.fi_pad[l]);
    add(1, L.b_off[l], 1, L.fo[l], L.fo_pad[l]);
    add(2, L.b_off[l], 1, L.fo[l], L.fo_pad[l]);
  }
  p.total = out;
  return VM_OK;
}

}  // namespace
}  // namespace vm

using namespace vm;

extern "C" int64_t vm_pack_floats(const VmStack* st) {
  PackPlan p;
  if (!st || plan_pack(*st, p)) return -1;
  return p.total;
}

extern "C" int vm_pack_stack(const VmStack* st, float* packed, int32_t unpack, void* stream) {
  VM_REQUIRE(st && packed && st->params && st->m && st->v, "vm_pack_stack: null argument");
  PackPlan p;
  VM_REQUIRE(plan_pack(*st, p) == VM_OK, "vm_pack_stack: unsupported architecture");
  if (p.total == 0) return VM_OK;
  pack_kernel<<<unsigned((p.total + kCT - 1) / kCT), kCT, 0, cudaStream_t(stream)>>>(
      p, packed, st->params, st->m, st->v, unpack ? 1 : 0);
  VM_CUDA(cudaGetLastError());
  return VM_OK;
}
