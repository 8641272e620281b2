"""Per-frame ingestion (drop-in for vobj/objects.py:160-277 and the
detection half of trainer.py:226-265 `process_frame`).

The O(pixels) work -- per-instance pixel counts and 2D boxes, backprojection
of every valid pixel, the per-axis quantile trims of AABB.from_points and the
subsampled scene bounds -- runs on the device (csrc/vm_ingest.cu) from the
frame's depth and instance mask uploaded once through pinned memory.  The
host keeps what is per detection: the mask crop, association
(objects.py:233-259), box growth and keyframe decisions.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .geometry import AABB
from .objects import AssociationConfig, ObjectInstance, ObjectMap
from .render import CameraIntrinsics


@dataclass
class Frame:
    """datasets.py:26-33."""

    frame_id: int
    rgb: np.ndarray    # [H, W, 3] float32 in [0, 1]
    depth: np.ndarray  # [H, W] float32 metres, 0 = invalid
    mask: np.ndarray   # [H, W] int32 instance ids, 0 = background
    pose: np.ndarray   # [4, 4] float64 camera-to-world


@dataclass
class Detection:
    """objects.py:74-83."""

    frame_id: int
    semantic_class: int
    bbox: tuple
    n_pixels: int
    mask: np.ndarray
    aabb: AABB


class FrameIngestor:
    """Device buffers of one frame (pinned staging + depth/mask on the device)
    and the ingestion workspace; reused across frames of one size."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.shape = None

    def _ensure(self, h: int, w: int) -> None:
        if self.shape == (h, w):
            return
        self.shape = (h, w)
        self.pin_depth = torch.empty((h, w), dtype=torch.float32, pin_memory=True)
        self.pin_mask = torch.empty((h, w), dtype=torch.int32, pin_memory=True)
        self.depth = torch.empty((h, w), dtype=torch.float32, device=self.device)
        self.mask = torch.empty((h, w), dtype=torch.int32, device=self.device)
        nb = _lib.load().vm_ingest_workspace_bytes(w, h)
        self.ws = torch.empty(nb, dtype=torch.uint8, device=self.device)
        self.cap = 4096
        self.out = (_lib.VmDetection * self.cap)()

    def upload(self, depth: np.ndarray, mask: np.ndarray) -> None:
        h, w = depth.shape
        self._ensure(h, w)
        self.pin_depth.numpy()[:] = depth
        self.pin_mask.numpy()[:] = mask
        self.depth.copy_(self.pin_depth, non_blocking=True)
        self.mask.copy_(self.pin_mask, non_blocking=True)

    def set_device_frame(self, depth: torch.Tensor, mask: torch.Tensor) -> None:
        """Use a frame already decoded on the device (datasets.Dataset.frame_device)."""
        h, w = depth.shape
        self._ensure(h, w)
        self.depth.copy_(depth)
        self.mask.copy_(mask)

    def run(self, intr: CameraIntrinsics, pose: np.ndarray, acfg: AssociationConfig, scene_stride: int = 4,
            scene_trim: float = 0.01):
        """-> (list of (instance_id, n_pixels, n_valid, bbox, AABB)), scene AABB or None."""
        h, w = self.shape
        lib = _lib.load()
        ci = (C.c_double * 4)(intr.fx, intr.fy, intr.cx, intr.cy)
        cp = (C.c_double * 16)(*np.asarray(pose, np.float64).reshape(16).tolist())
        n = C.c_int32()
        ok = C.c_int32()
        sb = (C.c_double * 6)()
        _lib.check(lib.vm_ingest_frame(self.depth.data_ptr(), self.mask.data_ptr(), w, h, ci, cp,
                                       int(acfg.min_pixels), float(acfg.outlier_trim), int(scene_stride),
                                       float(scene_trim), self.out, self.cap, C.byref(n), sb, C.byref(ok),
                                       self.ws.data_ptr(), self.ws.numel(), _lib.stream_ptr()), "ingest_frame")
        dets = []
        for d in self.out[:n.value]:
            dets.append((int(d.instance_id), int(d.n_pixels), int(d.n_valid), (d.u0, d.v0, d.u1, d.v1),
                         AABB(list(d.box_min), list(d.box_max))))
        scene = AABB(list(sb[:3]), list(sb[3:])) if ok.value else None
        return dets, scene


def extract_detections_device(ing: FrameIngestor, frame: Frame, intr: CameraIntrinsics, classes: dict,
                              acfg: AssociationConfig, uploaded: bool = False):
    """extract_detections (objects.py:170-217) + scene_bounds (:220-230) of
    one frame: boxes and counts from the device, mask crops on the host."""
    if frame.pose is None:
        raise ValueError(f"frame {frame.frame_id} has no pose; cannot lift detections")
    if not uploaded:
        ing.upload(frame.depth, frame.mask)
    raw, scene = ing.run(intr, frame.pose, acfg)
    dets = []
    for inst_id, _n_all, n_valid, (u0, v0, u1, v1), box in raw:
        dets.append(Detection(frame_id=frame.frame_id, semantic_class=int(classes.get(inst_id, 1)),
                              bbox=(u0, v0, u1, v1), n_pixels=n_valid,
                              mask=frame.mask[v0:v1, u0:u1] == inst_id, aabb=box))
    return dets, scene


def associate(detections: list, object_map: ObjectMap, cfg: AssociationConfig) -> list:
    """objects.py:233-259: greedy one-to-one matching by descending 3D IoU
    (ties: lower object id, then lower detection index).  The detection x
    object IoU matrix is formed in one vectorised pass with aabb_iou's
    operation order (per-axis max/min, the product x*y*z, (va + vb) - inter),
    so every IoU -- and hence the match -- is bit-identical to the pairwise
    loop; only the candidates that pass the threshold are sorted."""
    objs = list(object_map.objects())
    if not detections or not objs:
        return [None] * len(detections)
    dmin = np.stack([np.asarray(d.aabb.min, np.float64) for d in detections])[:, None, :]
    dmax = np.stack([np.asarray(d.aabb.max, np.float64) for d in detections])[:, None, :]
    omin = np.stack([np.asarray(o.aabb.min, np.float64) for o in objs])[None, :, :]
    omax = np.stack([np.asarray(o.aabb.max, np.float64) for o in objs])[None, :, :]
    lo = np.maximum(dmin, omin)
    hi = np.minimum(dmax, omax)
    overlap = ~np.any(hi <= lo, axis=-1)
    inter = np.prod(hi - lo, axis=-1)
    vd = np.prod(dmax - dmin, axis=-1)
    vo = np.prod(omax - omin, axis=-1)
    with np.errstate(divide="ignore", invalid="ignore"):
        iou = np.where(overlap, inter / ((vd + vo) - inter), 0.0)
    dcls = np.array([d.semantic_class for d in detections])[:, None]
    ocls = np.array([o.semantic_class for o in objs])[None, :]
    ok = (dcls == ocls) & (iou >= cfg.iou_threshold)
    di, oi = np.nonzero(ok)
    oid = np.array([o.object_id for o in objs])[oi]
    order = np.lexsort((di, oid, -iou[di, oi]))  # key order: -iou, object id, detection index
    assigned = [None] * len(detections)
    used = set()
    for j in order:
        d, o = int(di[j]), int(oid[j])
        if assigned[d] is not None or o in used:
            continue
        assigned[d] = o
        used.add(o)
    return assigned


def update_bounds(inst: ObjectInstance, det_aabb: AABB) -> None:
    """objects.py:262-264: grow, never shrink."""
    inst.aabb = inst.aabb.union(det_aabb)


def keyframe_due(inst: ObjectInstance, cfg: AssociationConfig) -> bool:
    """objects.py:267-277."""
    if inst.obs_count < 1:
        raise ValueError("keyframe_due called before the observation was counted")
    stride = cfg.keyframe_stride_background if inst.is_background else cfg.keyframe_stride_object
    return (inst.obs_count - 1) % stride == 0
