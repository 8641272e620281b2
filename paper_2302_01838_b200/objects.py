"""Object instances and keyframe buffers (drop-in for vobj/objects.py:21-109,
:280-320).  Keyframe crops are mirrored into a device texel arena
(keyframes.py) that the CUDA sampler gathers from; detection/association
(objects.py:45-259) is per-frame host work outside the training step."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .geometry import AABB

BACKGROUND_CLASS = 0


@dataclass(frozen=True)
class AssociationConfig:
    iou_threshold: float = 0.2
    outlier_trim: float = 0.02
    bound_pad: float = 0.10
    min_pixels: int = 100
    keyframe_stride_object: int = 25
    keyframe_stride_background: int = 50
    bbox_margin_px: int = 10

    def __post_init__(self):
        if not (0.0 < self.iou_threshold <= 1.0):
            raise ValueError(f"iou_threshold must be in (0, 1], got {self.iou_threshold}")
        if self.keyframe_stride_object < 1 or self.keyframe_stride_background < 1:
            raise ValueError("keyframe strides must be >= 1")
        if self.min_pixels < 1:
            raise ValueError(f"min_pixels must be >= 1, got {self.min_pixels}")
        if self.bbox_margin_px < 0:
            raise ValueError(f"bbox_margin_px must be >= 0, got {self.bbox_margin_px}")


@dataclass
class Keyframe:
    """objects.py:86-93; host copies of the crop plus its arena slot."""

    frame_id: int
    pose: np.ndarray
    bbox: tuple
    mask: np.ndarray
    rgb: np.ndarray
    depth: np.ndarray
    texel_off: int = -1  # offset of the crop in the device texel arena (-1: not uploaded)


@dataclass
class ObjectInstance:
    """objects.py:96-109."""

    object_id: int
    semantic_class: int
    aabb: AABB
    pe_scale: float
    model_index: int
    is_background: bool = False
    active: bool = True
    obs_count: int = 0
    keyframes: list = field(default_factory=list)
    # rays drawn per training step when fewer than TrainConfig.rays_per_object
    # (mixed per-object ray counts, BASELINE config 3); the batch rows beyond
    # are zero padding with ray_ok = False.  None: rays_per_object.
    n_rays: int | None = None

    def padded_aabb(self, fraction: float) -> AABB:
        return self.aabb.padded(fraction)


class ObjectMap:
    """objects.py:112-159: registry of mapped instances; id 0 is the background."""

    def __init__(self):
        self.instances: dict[int, ObjectInstance] = {}
        self._next_id = 1

    @property
    def background(self) -> ObjectInstance | None:
        return self.instances.get(0)

    def objects(self) -> list[ObjectInstance]:
        return [inst for oid, inst in sorted(self.instances.items()) if oid != 0]

    def add_background(self, aabb: AABB, pe_scale: float, model_index: int) -> ObjectInstance:
        if 0 in self.instances:
            raise ValueError("background instance already registered")
        inst = ObjectInstance(0, BACKGROUND_CLASS, aabb, pe_scale, model_index, is_background=True)
        self.instances[0] = inst
        return inst

    def add_object(self, semantic_class: int, aabb: AABB, pe_scale: float, model_index: int,
                   object_id: int | None = None) -> ObjectInstance:
        """objects.py:140-147.  `object_id` pins the id (object-sharded ranks
        register their share of a global map under the global ids)."""
        if object_id is None:
            oid = self._next_id
        else:
            oid = int(object_id)
            if oid <= 0 or oid in self.instances:
                raise ValueError(f"object id {oid} is reserved or already registered")
        self._next_id = max(self._next_id, oid + 1)
        inst = ObjectInstance(oid, semantic_class, aabb, pe_scale, model_index)
        self.instances[oid] = inst
        return inst

    def restore(self, inst: ObjectInstance) -> None:
        if inst.object_id in self.instances:
            raise ValueError(f"duplicate object id {inst.object_id}")
        self.instances[inst.object_id] = inst
        if not inst.is_background:
            self._next_id = max(self._next_id, inst.object_id + 1)


def dilate_bbox(bbox, mask, margin: int, image_shape):
    """objects.py:280-298."""
    h, w = image_shape
    u0, v0, u1, v1 = bbox
    nu0, nv0 = max(u0 - margin, 0), max(v0 - margin, 0)
    nu1, nv1 = min(u1 + margin, w), min(v1 + margin, h)
    grown = np.zeros((nv1 - nv0, nu1 - nu0), dtype=bool)
    grown[v0 - nv0:v1 - nv0, u0 - nu0:u1 - nu0] = mask
    return (nu0, nv0, nu1, nv1), grown


def add_keyframe(inst: ObjectInstance, frame_id: int, pose, bbox, mask, rgb, depth) -> Keyframe:
    """objects.py:301-320 (crops are copied; the Mapper uploads them)."""
    u0, v0, u1, v1 = bbox
    kf = Keyframe(frame_id=frame_id, pose=np.asarray(pose, dtype=np.float64).copy(), bbox=tuple(int(x) for x in bbox),
                  mask=np.asarray(mask, bool).copy(),
                  rgb=np.asarray(rgb[v0:v1, u0:u1], dtype=np.float32).copy(),
                  depth=np.asarray(depth[v0:v1, u0:u1], dtype=np.float32).copy())
    inst.keyframes.append(kf)
    return kf
