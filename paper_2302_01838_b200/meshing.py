"""Forward-only inference on the B200: occupancy grids and composed views
(drop-in for vobj/meshing.py:64-97 `query_grid` and :453-579 `_eval_field` /
`render_view`).

Every point evaluation runs on the device: grid / ray sample generation, the
f32 positional encoding exactly as the reference's inference path forms it,
the fused FFMA MLP forward (vm_forward) and the per-ray compositing
(csrc/vm_infer.cu).  Only the final arrays are copied to the host (numpy, as
the reference returns them).  Marching cubes, metrics and the other meshing
helpers stay out of scope (scikit-image / KD-tree host code).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .geometry import AABB
from .models import StackedModelParams, vm_stack
from .render import CameraIntrinsics


@dataclass
class OccupancyGrid:
    """meshing.py:40-54."""

    bound: AABB
    values: np.ndarray  # [rx, ry, rz] float32

    @property
    def resolution(self) -> tuple[int, int, int]:
        return self.values.shape

    @property
    def spacing(self) -> np.ndarray:
        res = np.array(self.values.shape, dtype=np.float64)
        return (self.bound.max - self.bound.min) / (res - 1)


@dataclass
class RenderedView:
    """meshing.py:447-450."""

    rgb: np.ndarray       # [H, W, 3] float32 in [0, 1]
    depth: np.ndarray     # [H, W] float32 z-depth
    instance: np.ndarray  # [H, W] int32 object id (0 = background)


def _d3(x) -> C.Array:
    a = (C.c_double * 3)()
    a[:] = [float(v) for v in np.asarray(x, np.float64).reshape(3)]
    return a


class _Workspace:
    """Per-device inference scratch (points, encodings, outputs of one chunk)."""

    def __init__(self):
        self.buf = None

    def get(self, arch, chunk: int, device) -> tuple[int, int]:
        lib = _lib.load()
        va = arch.vm_arch()
        n = lib.vm_infer_workspace_bytes(C.byref(va), chunk)
        if self.buf is None or self.buf.numel() < n or self.buf.device != device:
            self.buf = torch.empty(n, dtype=torch.uint8, device=device)
        return self.buf.data_ptr(), self.buf.numel()


_WS = _Workspace()


def query_grid(params: StackedModelParams, model_index: int, bound: AABB, pe_scale: float,
               resolution, chunk: int | None = None, as_tensor: bool = False) -> OccupancyGrid:
    """meshing.py:64-97: occupancy of one model on the inclusive np.linspace
    grid over `bound` ('ij' order).  Returns numpy values (or the device
    tensor with `as_tensor`)."""
    if isinstance(resolution, int):
        resolution = (resolution, resolution, resolution)
    resolution = tuple(int(r) for r in resolution)
    if any(r < 2 for r in resolution):
        raise ValueError(f"grid resolution must be >= 2 per axis, got {resolution}")
    if not 0 <= model_index < params.count:
        raise IndexError(f"model index {model_index} out of range for count {params.count}")
    dev = params.arena.device
    n = int(np.prod(resolution))
    if chunk is None:
        chunk = 1 << 21
    chunk = max(32, min(int(chunk), n))
    out = torch.empty(n, dtype=torch.float32, device=dev)
    ws, wsn = _WS.get(params.arch, chunk, dev)
    st = vm_stack(params)
    res = (C.c_int32 * 3)(*resolution)
    _lib.check(_lib.load().vm_query_grid(C.byref(st), int(model_index), _d3(bound.min), _d3(bound.max),
                                         float(pe_scale), res, out.data_ptr(), ws, wsn, chunk, _lib.stream_ptr()),
               "query_grid")
    vals = out.reshape(resolution)
    return OccupancyGrid(bound=bound, values=vals if as_tensor else vals.cpu().numpy())


def _eval_rays(params, model_index, box: AABB, pe_scale, origin, dirs, sel, n, lo, hi, lo_c, hi_c, S, chunk):
    dev = dirs.device
    op = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    dep = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    col = torch.empty((max(n, 1), 3), dtype=torch.float32, device=dev)
    if n:
        chunk = max(int(chunk), S)
        ws, wsn = _WS.get(params.arch, chunk, dev)
        st = vm_stack(params)
        _lib.check(_lib.load().vm_eval_rays(
            C.byref(st), int(model_index), _d3(box.min), _d3(box.max), float(pe_scale), _d3(origin), dirs.data_ptr(),
            _lib.ptr(sel), n, _lib.ptr(lo), _lib.ptr(hi), float(lo_c), float(hi_c), int(S), op.data_ptr(),
            dep.data_ptr(), col.data_ptr(), ws, wsn, chunk, _lib.stream_ptr()), "eval_rays")
    return op, dep, col


def render_view(obj_params: StackedModelParams, bg_params: StackedModelParams, object_map,
                intrinsics: CameraIntrinsics, pose: np.ndarray, *, t_near: float = 0.0, t_far: float = 8.0,
                samples_object: int = 48, samples_background: int = 48, samples_refine: int = 32,
                refine_window: float = 0.25, bound_pad: float = 0.10, threshold: float = 0.5,
                chunk: int = 1 << 21) -> RenderedView:
    """meshing.py:485-579: coarse + refined background, then every object
    over its padded-box interval; per pixel the nearest object with opacity
    >= threshold wins (ascending id breaks ties), the background fills the
    rest."""
    lib = _lib.load()
    dev = bg_params.arena.device
    w, h = int(intrinsics.width), int(intrinsics.height)
    n = w * h
    pose = np.asarray(pose, dtype=np.float64)
    if pose.shape != (4, 4):
        raise ValueError(f"pose must be 4x4, got {pose.shape}")
    bg = object_map.background
    if bg is None:
        raise ValueError("object map has no background instance")
    sp = _lib.stream_ptr()
    dirs = torch.empty((n, 3), dtype=torch.float64, device=dev)
    scale = torch.empty(n, dtype=torch.float64, device=dev)
    intr = (C.c_double * 4)(intrinsics.fx, intrinsics.fy, intrinsics.cx, intrinsics.cy)
    pz = (C.c_double * 16)(*pose.reshape(16).tolist())
    _lib.check(lib.vm_view_rays(intr, w, h, pz, dirs.data_ptr(), scale.data_ptr(), sp), "view_rays")
    origin = pose[:3, 3]
    bg_box = bg.aabb.padded(bound_pad)
    c_op, c_dep, c_col = _eval_rays(bg_params, bg.model_index, bg_box, bg.pe_scale, origin, dirs, None, n, None,
                                    None, t_near, t_far, samples_background, chunk)
    r_dep, r_col = c_dep, c_col
    if samples_refine > 0:
        lo = torch.empty(n, dtype=torch.float64, device=dev)
        hi = torch.empty(n, dtype=torch.float64, device=dev)
        _lib.check(lib.vm_view_compose(0, n, c_dep.data_ptr(), None, None, None, None, None, float(t_near),
                                       float(t_far), float(refine_window), 0, lo.data_ptr(), hi.data_ptr(), None,
                                       None, sp), "view_compose")
        _, r_dep, r_col = _eval_rays(bg_params, bg.model_index, bg_box, bg.pe_scale, origin, dirs, None, n, lo, hi,
                                     0.0, 0.0, samples_refine, chunk)
    depth = torch.empty(n, dtype=torch.float64, device=dev)
    colour = torch.empty((n, 3), dtype=torch.float64, device=dev)
    instance = torch.empty(n, dtype=torch.int32, device=dev)
    best = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.check(lib.vm_view_compose(1, n, c_op.data_ptr(), c_dep.data_ptr(), c_col.data_ptr(), r_dep.data_ptr(),
                                   r_col.data_ptr(), None, 0.0, 0.0, 0.0, 1 if samples_refine > 0 else 0,
                                   depth.data_ptr(), colour.data_ptr(), instance.data_ptr(), best.data_ptr(), sp),
               "view_compose")
    sel = torch.empty(n, dtype=torch.int32, device=dev)
    lo = torch.empty(n, dtype=torch.float64, device=dev)
    hi = torch.empty(n, dtype=torch.float64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    for inst in object_map.objects():
        box = inst.aabb.padded(bound_pad)
        _lib.check(lib.vm_ray_box_select(_d3(origin), dirs.data_ptr(), n, _d3(box.min), _d3(box.max),
                                         float(t_near), sel.data_ptr(), cnt.data_ptr(), lo.data_ptr(),
                                         hi.data_ptr(), sp), "ray_box_select")
        m = int(cnt.item())
        if m == 0:
            continue
        op, dep, col = _eval_rays(obj_params, inst.model_index, box, inst.pe_scale, origin, dirs, sel, m, lo, hi,
                                  0.0, 0.0, samples_object, chunk)
        _lib.check(lib.vm_view_compose(2, m, sel.data_ptr(), op.data_ptr(), dep.data_ptr(), col.data_ptr(), None,
                                       None, float(threshold), 0.0, 0.0, int(inst.object_id), best.data_ptr(),
                                       depth.data_ptr(), colour.data_ptr(), instance.data_ptr(), sp),
                   "view_compose")
    rgb = torch.empty((n, 3), dtype=torch.float32, device=dev)
    z = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.check(lib.vm_view_compose(3, n, depth.data_ptr(), scale.data_ptr(), colour.data_ptr(), None, None, None,
                                   0.0, 0.0, 0.0, 0, rgb.data_ptr(), z.data_ptr(), None, None, sp), "view_compose")
    return RenderedView(rgb=rgb.reshape(h, w, 3).cpu().numpy(), depth=z.reshape(h, w).cpu().numpy(),
                        instance=instance.reshape(h, w).cpu().numpy())
