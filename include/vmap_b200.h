/*
 * vmap_b200.h -- C ABI of the B200-native vMAP object-mapping step.
 *
 * The reference (`vobj`, /root/reference/pkg/src/vobj) is a pure-Python
 * package; its "operator API" is the set of module-level functions its
 * trainer calls.  Each entry point below replaces one of them and keeps its
 * argument meaning and error behaviour (the Python mirror in
 * paper_2302_01838_b200/ raises the same exception types from the codes).
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer owned by the caller (torch tensors in
 *     the Python host); nothing is allocated inside except where a call says
 *     so.  `stream` is a cudaStream_t passed as void*.
 *   - Calls are asynchronous on `stream`; device-side failures (non-finite
 *     gradients) are reported through a caller-provided device status word.
 *   - Return codes: VM_OK, VM_ERR_SHAPE (bad arguments), VM_ERR_CUDA (launch
 *     error; see vm_last_error()), VM_ERR_UNSUPPORTED (arch outside the
 *     compiled kernel set).
 *   - Not reentrant per stack (single writer).  Different host
 *     threads may drive different stacks/devices concurrently: the library's
 *     internal side stream and fork/join events (vm_train_step's tensor-core
 *     branch) are per (host thread, device).
 *
 * Parameter storage: one model-major arena per stack,
 *   arena[capacity][block],  block = sum over layers of (fo_pad*fi_pad + fo_pad)
 * with layer l's weight matrix at w_off[l] (row-major [fo_pad][fi_pad]) and
 * its bias at b_off[l].  Padded rows/columns are zero and stay zero.  The
 * reference's per-layer views `weights[l]: [capacity, fo, fi]`
 * (models.py:69-71) are strided views of this arena.
 */
#ifndef VMAP_B200_H
#define VMAP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VM_OK 0
#define VM_ERR_SHAPE 1
#define VM_ERR_CUDA 3
#define VM_ERR_UNSUPPORTED 4

#define VM_MAX_LAYERS 8
#define VM_MAX_STACKS 2

/* models.py:19-55 ModelArch (output_dim is always 4: occupancy + RGB). */
typedef struct VmArch {
  int32_t n_layers;   /* >= 2 */
  int32_t hidden;     /* >= 1 (fused kernels: <= 128; wider: the layered path) */
  int32_t input_dim;  /* 3*include_input + 6*n_freq (fused kernels: <= 40) */
  int32_t reserved;
} VmArch;

/* Arena layout of one model block, filled by vm_model_layout(). */
typedef struct VmLayout {
  int32_t n_layers;
  int32_t hidden_pad;                 /* 32, 64, 128, else hidden rounded up to 32 */
  int32_t fo[VM_MAX_LAYERS], fi[VM_MAX_LAYERS];         /* true dims */
  int32_t fo_pad[VM_MAX_LAYERS], fi_pad[VM_MAX_LAYERS]; /* arena dims */
  int64_t w_off[VM_MAX_LAYERS], b_off[VM_MAX_LAYERS];   /* float offsets */
  int64_t block;                      /* floats per model */
  int64_t n_params;                   /* true parameter count per model */
} VmLayout;

/* StackedModelParams + OptimState (models.py:58-126). */
typedef struct VmStack {
  VmArch arch;
  int32_t count;          /* live models K */
  int32_t capacity;
  float* params;          /* [capacity*block] */
  float* m;               /* Adam first moment, same layout */
  float* v;               /* Adam second moment */
  int64_t* step;          /* [capacity] Adam step counters */
  const uint8_t* frozen;  /* [capacity] */
  /* Bias corrections f32(1 - beta^t) computed in f64 on the host exactly as
     models.py:434-436 does; index t-1.  For t > corr_len the device computes
     f32(1 - pow(beta, t)) in f64 from beta1/beta2 below. */
  const float* corr1;
  const float* corr2;
  int32_t corr_len;
  /* f32 constants as numpy forms them (models.py:444-457):
     beta1f = f32(b1), omb1 = f32(1-b1), beta2f, omb2 = f32(1-b2), eps, lr. */
  float beta1f, omb1, beta2f, omb2, eps, lr;
  double beta1, beta2;    /* the python-float betas (bias corrections past corr_len) */
} VmStack;

/* RaySampleBatch (trainer.py:162-173), stacked on a leading model axis.
   Either `encoded` [K,R,S,D] (reference layout) or `points` [K,R,S,3]
   (box-normalised sample points; positional encoding fused in-kernel with
   `pe_scale` [K]) must be given.

   Mixed per-object ray counts (BASELINE config 3): `model_rays`
   [K] (device, optional) gives the rays model k drew (<= n_rays); its rows
   r >= model_rays[k] are zero padding with ray_ok = 0 -- exactly the
   reference's _zero_batch rows (trainer.py:190-200), which contribute
   nothing to losses (render.py:301-308) or gradients (render.py:324-333).
   The FFMA object kernel skips them; `work_items` [2*n_work_items] (device,
   (model, chunk) pairs from vm_work_items) lets its grid cover only the live
   chunks (NULL: a K x max-chunks grid whose dead chunks exit at once). */
typedef struct VmBatch {
  int32_t n_models, n_rays, n_points, input_dim;
  const float* encoded;
  const float* points;
  const float* pe_scale;
  const float* t;              /* [K,R,S] */
  const float* target_depth;   /* [K,R] */
  const float* target_colour;  /* [K,R,3] */
  const uint8_t* target_mask;  /* [K,R] */
  const uint8_t* valid_depth;  /* [K,R] */
  const uint8_t* ray_ok;       /* [K,R] */
  const int32_t* model_rays;   /* [K] live rays per model, or NULL (all n_rays) */
  const int32_t* work_items;   /* [2*n_work_items] (model, chunk), or NULL */
  int32_t n_work_items, reserved;
} VmBatch;

/* LossWeights (render.py:61-64). */
typedef struct VmLossWeights { float colour, occupancy; } VmLossWeights;

/* Status words written by vm_train_step (device int32[4*n_stacks]; the call
   initialises them to the sentinel 0x7f7f7f7f = "none"):
   [4s+0] first model index with a non-finite gradient among the models Adam
          would update, else sentinel (models.py:423-428 FloatingPointError)
   [4s+1] first model index with a non-finite loss, else sentinel
          (trainer.py:404-407)
   [4s+2] 1 if Adam ran for stack s, else 0
   [4s+3] reserved */

/* ---- layout ---------------------------------------------------------- */
int vm_model_layout(const VmArch* arch, VmLayout* out);

/* ---- fused training step: replaces trainer.py:480-506 train_on_batch for
   1..VM_MAX_STACKS stacks in one launch sequence (Mapper.train_step runs the
   object stack then the background stack, trainer.py:364-390).  Stack s is
   skipped (no Adam) when an earlier stack reported a non-finite gradient or
   loss, matching the reference's raise-before-next-stack order. ----------- */
size_t vm_train_workspace_bytes(const VmStack* stacks, const VmBatch* batches, int n_stacks);
/* Work items of the FFMA object kernel for per-model ray counts
   `model_rays` (host [n_models]): (model, chunk) pairs written to `items`
   (host, 2*capacity int32; may be NULL to query), count in *n_items.  The
   chunking depends only on each model's own ray count (vectorised ==
   sequential bits). */
int vm_work_items(const int32_t* model_rays, int32_t n_models, int32_t n_points, int32_t* items,
                  int32_t capacity, int32_t* n_items);
/* Stacks without a fused kernel (hidden > 128, input_dim > 40, n_points > 32
   (up to 64), layer counts other than the fused instantiations) are trained by
   the layered path: the same math one layer at a time (per-layer batched FP32
   GEMMs, the per-ray render chain, Adam), with the same status words, skip
   rules and vectorised == sequential bits; it requires `encoded`.  In a
   two-stack call with a fused stack 0 only stack 1 takes it.  VM_LAYERED=1
   forces it for every stack (cross-check). */
int vm_train_step(const VmStack* stacks, const VmBatch* batches, int n_stacks,
                  VmLossWeights weights, float* losses /* [sum K][3] */,
                  int32_t* status /* device [4*n_stacks] */,
                  void* workspace, size_t workspace_bytes, void* stream);

/* ---- models.py:311-355 forward: occupancy/colour for N samples per model.
   encoded [K,N,D] -> occ [K,N], col [K,N,3]. -------------------------------- */
int vm_forward(const VmStack* st, const float* encoded, int64_t n_samples,
               float* occ, float* col, void* stream);

/* ---- models.py:358-398 backward: parameter gradients given output grads.
   Recomputes the forward from `encoded` (the activation cache is the input).
   grads: [K][block] arena layout. ------------------------------------------- */
int vm_backward(const VmStack* st, const float* encoded, int64_t n_samples,
                const float* grad_occ, const float* grad_col, float* grads, void* stream);

/* ---- models.py:401-467 adam_step over the stacked arena.  update_mask may be
   NULL.  status: device int32[1], set to the first active model index with a
   non-finite gradient (and then NOTHING is updated), else -1. --------------- */
int vm_adam(const VmStack* st, const float* grads, const uint8_t* update_mask,
            int32_t* status, void* stream);

/* ---- render.py:230-281 occupancy rendering (bit-exact f32 op order). ------ */
int vm_render_forward(int64_t n_rays, int32_t n_points, const float* occ, const float* col,
                      const float* t, float* opacity, float* depth, float* colour,
                      float* weights, float* trans, void* stream);
int vm_render_backward(int64_t n_rays, int32_t n_points, const float* occ, const float* col,
                       const float* t, const float* weights, const float* trans,
                       const float* grad_opacity, const float* grad_depth,
                       const float* grad_colour, float* d_occ, float* d_col, void* stream);
/* ---- render.py:284-333 L1 losses (pairwise-summed over rays) and grads. ---
 * The per-ray terms live in a stream-ordered temporary (cudaMallocAsync /
 * cudaFreeAsync on `stream`, 12 B per ray): the one entry point here that
 * allocates; vm_train_step takes them from its caller's workspace. */
int vm_losses(int32_t n_models, int32_t n_rays, const float* opacity, const float* depth,
              const float* colour, const float* target_depth, const float* target_colour,
              const uint8_t* target_mask, const uint8_t* valid_depth, const uint8_t* ray_ok,
              VmLossWeights w, float* l_depth, float* l_colour, float* l_occ, float* l_total,
              float* grad_opacity, float* grad_depth, float* grad_colour, void* stream);

/* ---- sampler: objects.py:323-352 + trainer.py:269-318 + render.py:76-227 --- */
/* Keyframe crop texels live in one arena: texel (u,v) of keyframe j is
   rgbd[kf.texel_off + (v-v0)*(u1-u0) + (u-u0)] (float4: r,g,b,depth z) and
   mask[kf.texel_off + same] (uint8). */
typedef struct VmKeyframe {
  int64_t texel_off;
  int32_t u0, v0, u1, v1;      /* half-open bbox in image pixels */
  double pose[12];             /* camera-to-world rows 0..2 of the 4x4 */
} VmKeyframe;

typedef struct VmSampleObject {
  int64_t object_id;           /* RNG key part (objects.py:335, trainer.py:304) */
  int32_t kf_begin, n_kf;      /* keyframes [kf_begin, kf_begin+n_kf) */
  int32_t active;              /* 0 -> zero batch (trainer.py:272-273, :336-338) */
  int32_t n_rays;              /* rays this object draws (<= params n_rays; 0: params n_rays);
                                  rows beyond are zero padding (config 3) */
  double box_min[3], box_max[3];   /* padded AABB (geometry.py:40-42) */
  double center[3], half[3];       /* of the padded AABB */
  double pe_scale;
} VmSampleObject;

typedef struct VmSampleParams {
  uint64_t seed;
  int64_t step;
  int32_t n_rays, n_stratified, n_surface, encode; /* encode: 1 -> write encoded, 0 -> points */
  int32_t n_freq, include_input, reserved0, reserved1;
  double fx, fy, cx, cy;
  int32_t width, height;
  double t_near, t_far, surface_std, three_std; /* three_std = 3.0*surface_std (python f64) */
  /* If non-NULL the RNG step key is (*step_dev + step_offset) read on the
     device (CUDA-graph replay); otherwise `step`. */
  const int64_t* step_dev;
  int64_t step_offset;
} VmSampleParams;

/* Debug/parity outputs of the sampler (optional, may be NULL). */
typedef struct VmSampleAux {
  int64_t* kf_idx; int64_t* u; int64_t* v;    /* [K,R] */
  double* t64;                                 /* [K,R,S] f64 sorted samples */
} VmSampleAux;

size_t vm_sample_workspace_bytes(int n_objects, const VmSampleParams* p);
int vm_sample(const VmSampleObject* objects /* device [K] */, int n_objects,
              const VmKeyframe* keyframes /* device */, const float* rgbd /* float4 texels */,
              const uint8_t* mask, const VmSampleParams* params, VmBatch* out /* device ptrs */,
              VmSampleAux* aux, void* workspace, size_t workspace_bytes, void* stream);

/* ---- forward-only inference (meshing.py) --------------------
   Host pointers for the small double[3] arguments (box corners, origin);
   device pointers for arrays.  Point sets are processed in chunks of `chunk`
   samples through `workspace` (vm_infer_workspace_bytes(arch, chunk)). */
size_t vm_infer_workspace_bytes(const VmArch* arch, int64_t chunk);
/* query_grid (meshing.py:64-97): occupancy of model `model_index` on the
   np.linspace grid over [box_min, box_max] (meshgrid 'ij', C order) ->
   occ_out [rx*ry*rz] (device). */
int vm_query_grid(const VmStack* stack, int32_t model_index, const double* box_min, const double* box_max,
                  double pe_scale, const int32_t* resolution /* host [3] */, float* occ_out, void* workspace,
                  size_t workspace_bytes, int64_t chunk, void* stream);
/* _eval_field + render_rays (meshing.py:453-482, render.py:230-246) for rays
   origin + t dirs[sel[r]] at the S bin midpoints of [lo[r], hi[r]] (or the
   constants when lo/hi are NULL; sel NULL = identity) -> per ray opacity
   (f32), depth (f64, as render_view forms it) and colour (f32). */
int vm_eval_rays(const VmStack* stack, int32_t model_index, const double* box_min, const double* box_max,
                 double pe_scale, const double* origin, const double* dirs, const int32_t* sel, int64_t n_rays,
                 const double* lo, const double* hi, double lo_const, double hi_const, int32_t n_samples,
                 float* opacity, double* depth, float* colour, void* workspace, size_t workspace_bytes,
                 int64_t chunk, void* stream);
/* pixel rays of a camera (meshing.py:516-526): dirs [H*W,3] f64 unit,
   scale [H*W] = |d_cam|; intr = (fx, fy, cx, cy) host, pose 4x4 host. */
int vm_view_rays(const double* intr, int32_t width, int32_t height, const double* pose, double* dirs,
                 double* scale, void* stream);
/* ray_box_intersect + render_view's t0 = max(t0, t_near), hit & t1 > t0
   (render.py:111-139, meshing.py:562-565): compacted ray indices `sel`,
   their [lo, hi] and the count (device int32). */
int vm_ray_box_select(const double* origin, const double* dirs, int64_t n, const double* box_min,
                      const double* box_max, double t_near, int32_t* sel, int32_t* count, double* lo, double* hi,
                      void* stream);
/* render_view's per-pixel steps (meshing.py:538-581): op 0 refine window,
   1 background choice + state init, 2 one object's depth competition,
   3 z-depth + clipped colour outputs (see vm_infer.cu). */
int vm_view_compose(int32_t op, int64_t n, const void* a0, const void* a1, const void* a2, const void* a3,
                    const void* a4, const void* a5, double p0, double p1, double p2, int32_t i0, void* o0,
                    void* o1, void* o2, void* o3, void* stream);

/* ---- per-frame ingestion (trainer.py:226-265) ---------- */
/* Dataset.frame's conversion (datasets.py:160-175) on the device: 8-bit BGR
   -> f32 RGB / 255, 16-bit depth -> f32 / depth_scale, 16-bit ids -> int32.
   Any of the three inputs may be NULL. */
int vm_decode_frame(const uint8_t* bgr, const uint16_t* depth16, const uint16_t* mask16, int32_t width,
                    int32_t height, double depth_scale, float* rgb, float* depth, int32_t* mask, void* stream);

/* One lifted instance (objects.py:68-83 Detection without the mask crop). */
typedef struct VmDetection {
  int32_t instance_id, n_pixels, n_valid, reserved;
  int32_t u0, v0, u1, v1;                 /* half-open 2D bbox of the whole mask */
  double box_min[3], box_max[3];          /* AABB.from_points(trim) of the valid pixels */
} VmDetection;

size_t vm_ingest_workspace_bytes(int32_t width, int32_t height);
/* extract_detections (objects.py:170-217) + scene_bounds (:220-230) for one
   device frame (depth f32, mask int32 in [0, 65535]): detections of the ids
   with >= min_pixels valid-depth pixels in ascending id order (host `out`),
   and the trimmed box of the stride-subsampled valid depth (*scene_ok = 0
   when fewer than 16 points).  intr = (fx, fy, cx, cy), pose 4x4 (host).
   Synchronises `stream` (the detections are returned on the host). */
int vm_ingest_frame(const float* depth, const int32_t* mask, int32_t width, int32_t height, const double* intr,
                    const double* pose, int32_t min_pixels, double trim, int32_t scene_stride, double scene_trim,
                    VmDetection* out, int32_t capacity, int32_t* n_out, double* scene_box /* host [6] */,
                    int32_t* scene_ok, void* workspace, size_t workspace_bytes, void* stream);

/* ---- VOBJ v1 checkpoint stack sections (checkpoint.py:51-84; 8f #3) ------
   vm_pack_stack gathers the live parameters + Adam moments of `st` from the
   padded device arena into the reference's section order (per layer W
   [K,fo,fi], b [K,fo]; then per layer m_w, v_w, m_b, v_b), `packed` being
   vm_pack_floats(st) device floats; unpack = 1 scatters it back. */
int64_t vm_pack_floats(const VmStack* st);
int vm_pack_stack(const VmStack* st, float* packed, int32_t unpack, void* stream);

/* ---- profiling: event-time every fused-kernel launch of vm_train_step ---- */
int vm_profile_enable(int on);                          /* resets the launch log */
int vm_profile_read(int* launches, double* total_ms);   /* syncs on the events; MLP phase */
/* tag: 0 = MLP phase (fork .. join), 1 = FFMA kernel KF, 2 = tensor-core branch (KT + its partial reduce), 3 = Adam */
int vm_profile_read_tag(int tag, int* launches, double* total_ms);
int vm_profile_kernels(long* n);                        /* kernels launched since enable */
/* VM_TRACE=1 in the environment: each vm_train_step records its FFMA work
 * items (kind 1) and KT tiles (kind 2) as (kind, SM id, start ns, end ns);
 * reads the last step's records (syncs the device). */
int vm_trace_read(unsigned long long* out, int max_records, int* n_records);
void vm_profile_count_kernels(int n);                   /* internal: launch counter */
/* CTA count and dynamic smem the fused kernel would use for these stacks. */
int vm_train_grid(const VmStack* stacks, const VmBatch* batches, int n_stacks, int* ctas, int* smem_bytes);

/* Device step counter used by graph-replayed steps: *counter += inc. */
int vm_step_advance(int64_t* counter, int64_t inc, void* stream);
/* Launch an instantiated CUDA graph (cudaGraphExec_t) on a stream. */
int vm_graph_launch(void* graph_exec, void* stream);
/* End of a captured step: copy n_words result words (losses + status) into
 * pinned host memory by device stores (no copy-engine transfer) and advance
 * the device step counter by inc. */
int vm_step_finish(const int32_t* words, int32_t* host_words, int32_t n_words, int64_t* counter, int64_t inc,
                   void* stream);

/* ---- misc ---------------------------------------------------------------- */
const char* vm_last_error(void);
const char* vm_version(void);
/* FP32 FFMA throughput probe (roofline denominator): returns achieved
   TFLOP/s measured with events around `iters` dependent-chain FFMAs. */
int vm_ffma_peak(int iters, float* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VMAP_B200_H */
