"""Rendering, losses and sampling configuration (drop-in for vobj/render.py).

Reference: /root/reference/pkg/src/vobj/render.py.  The per-ray math runs in
csrc/vm_render.cu with the reference's float32 operation order, so given the
same per-sample occupancy/colour the outputs are bit-identical.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .models import DEVICE, _as_device


@dataclass(frozen=True)
class CameraIntrinsics:
    """render.py:18-35."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError(f"focal lengths must be positive, got fx={self.fx}, fy={self.fy}")
        if self.width <= 0 or self.height <= 0:
            raise ValueError(f"image size must be positive, got {self.width}x{self.height}")
        if not (0 < self.cx < self.width) or not (0 < self.cy < self.height):
            raise ValueError(
                f"principal point ({self.cx}, {self.cy}) outside image {self.width}x{self.height}")


@dataclass(frozen=True)
class SamplingConfig:
    """render.py:38-58."""

    t_near: float = 0.0
    t_far: float = 8.0
    n_stratified: int = 5
    n_surface: int = 5
    surface_std: float = 0.03

    def __post_init__(self):
        if self.t_far <= self.t_near:
            raise ValueError(f"t_far ({self.t_far}) must exceed t_near ({self.t_near})")
        if self.n_stratified < 1 or self.n_surface < 0:
            raise ValueError("need at least one stratified sample and non-negative surface count")
        if self.surface_std <= 0:
            raise ValueError(f"surface_std must be positive, got {self.surface_std}")

    @property
    def n_points(self) -> int:
        return self.n_stratified + self.n_surface


@dataclass(frozen=True)
class LossWeights:
    """render.py:61-64."""

    colour: float = 5.0
    occupancy: float = 10.0

    def vm(self) -> _lib.VmLossWeights:
        return _lib.VmLossWeights(float(np.float32(self.colour)), float(np.float32(self.occupancy)))


@dataclass
class RenderResult:
    opacity: torch.Tensor
    depth: torch.Tensor
    colour: torch.Tensor
    weights: torch.Tensor
    transmittance: torch.Tensor


def render_rays(occupancy, colour, t) -> RenderResult:
    """render.py:230-246 (vm_render_forward)."""
    occ = _as_device(occupancy)
    col = _as_device(colour)
    tt = _as_device(t)
    lead, s = tuple(occ.shape[:-1]), occ.shape[-1]
    n = int(np.prod(lead)) if lead else 1
    opacity = torch.empty(lead, dtype=torch.float32, device=occ.device)
    depth = torch.empty(lead, dtype=torch.float32, device=occ.device)
    rgb = torch.empty(lead + (3,), dtype=torch.float32, device=occ.device)
    w = torch.empty_like(occ)
    trans = torch.empty_like(occ)
    _lib.check(_lib.load().vm_render_forward(n, s, occ.data_ptr(), col.data_ptr(), tt.data_ptr(),
                                             opacity.data_ptr(), depth.data_ptr(), rgb.data_ptr(),
                                             w.data_ptr(), trans.data_ptr(), _lib.stream_ptr()),
               "render_rays")
    return RenderResult(opacity, depth, rgb, w, trans)


def render_backward(occupancy, colour, t, result: RenderResult, grad_opacity, grad_depth, grad_colour):
    """render.py:249-281 (vm_render_backward) -> (d_occ, d_colour)."""
    occ = _as_device(occupancy)
    col = _as_device(colour)
    tt = _as_device(t)
    lead, s = tuple(occ.shape[:-1]), occ.shape[-1]
    n = int(np.prod(lead)) if lead else 1
    gO, gD, gC = _as_device(grad_opacity), _as_device(grad_depth), _as_device(grad_colour)
    d_occ = torch.empty_like(occ)
    d_col = torch.empty_like(col)
    _lib.check(_lib.load().vm_render_backward(n, s, occ.data_ptr(), col.data_ptr(), tt.data_ptr(),
                                              result.weights.data_ptr(), result.transmittance.data_ptr(),
                                              gO.data_ptr(), gD.data_ptr(), gC.data_ptr(), d_occ.data_ptr(),
                                              d_col.data_ptr(), _lib.stream_ptr()), "render_backward")
    return d_occ, d_col


def _loss_call(result, target_depth, target_colour, target_mask, valid_depth, ray_ok, weights, grads: bool):
    D = _as_device(result.depth)
    lead = tuple(D.shape)
    if len(lead) == 1:
        k, r = 1, lead[0]
    else:
        k, r = int(np.prod(lead[:-1])), lead[-1]
    u8 = lambda x: _as_device(x, dtype=torch.uint8)
    O, C3 = _as_device(result.opacity), _as_device(result.colour)
    tD, tC = _as_device(target_depth), _as_device(target_colour)
    m, v, ok = u8(target_mask), u8(valid_depth), u8(ray_ok)
    dev = D.device
    outs = [torch.empty(lead[:-1] if len(lead) > 1 else (), dtype=torch.float32, device=dev) for _ in range(4)]
    g = [torch.empty(lead, dtype=torch.float32, device=dev), torch.empty(lead, dtype=torch.float32, device=dev),
         torch.empty(lead + (3,), dtype=torch.float32, device=dev)] if grads else [None, None, None]
    _lib.check(_lib.load().vm_losses(k, r, O.data_ptr(), D.data_ptr(), C3.data_ptr(), tD.data_ptr(),
                                     tC.data_ptr(), m.data_ptr(), v.data_ptr(), ok.data_ptr(), weights.vm(),
                                     *[o.data_ptr() for o in outs], *[_lib.ptr(x) for x in g],
                                     _lib.stream_ptr()), "compute_losses")
    return outs, g


def compute_losses(result, target_depth, target_colour, target_mask, valid_depth, ray_ok, weights: LossWeights):
    """render.py:284-309 -> (L_depth, L_colour, L_occ, total), pairwise-summed over rays."""
    outs, _ = _loss_call(result, target_depth, target_colour, target_mask, valid_depth, ray_ok, weights, False)
    return tuple(outs)


def loss_output_grads(result, target_depth, target_colour, target_mask, valid_depth, ray_ok,
                      weights: LossWeights):
    """render.py:312-333 -> (d_opacity, d_depth, d_colour)."""
    _, g = _loss_call(result, target_depth, target_colour, target_mask, valid_depth, ray_ok, weights, True)
    return tuple(g)
