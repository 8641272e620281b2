"""Device keyframe arena + the CUDA ray/sample generator (vm_sample).

Keyframe crops (objects.py:86-93: rgb f32x3, depth f32, mask bool) are packed
into one growing device arena of float4 RGBD texels plus a mask byte per
texel, so every training ray's gather is one 16-B load and one byte
(SURVEY 7 design notes).  Per-keyframe descriptors (bbox, pose, arena
offset) and per-object descriptors (object id = RNG key part, padded box,
PE scale) are small tables re-uploaded only when the map changes.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .models import DEVICE


class KeyframeArena:
    def __init__(self, device=DEVICE, capacity_texels: int = 1 << 20):
        self.device = torch.device(device)
        self.rgbd = torch.zeros((capacity_texels, 4), dtype=torch.float32, device=self.device)
        self.mask = torch.zeros(capacity_texels, dtype=torch.uint8, device=self.device)
        self.used = 0
        self.uploaded_bytes = 0  # host->device crop bytes so far (texel float4 + mask byte)
        self._pin_tex = self._pin_msk = self._pin_done = None

    def _reserve(self, n: int) -> None:
        need = self.used + n
        cap = self.rgbd.shape[0]
        if need <= cap:
            return
        while cap < need:
            cap *= 2
        rgbd = torch.zeros((cap, 4), dtype=torch.float32, device=self.device)
        mask = torch.zeros(cap, dtype=torch.uint8, device=self.device)
        rgbd[:self.used] = self.rgbd[:self.used]
        mask[:self.used] = self.mask[:self.used]
        self.rgbd, self.mask = rgbd, mask

    def add_many(self, kfs) -> None:
        """Upload several keyframes' crops with one H2D copy per arena plane
        (the per-frame ingestion path adds a few dozen at a time)."""
        kfs = [kf for kf in kfs if getattr(kf, "texel_off", -1) < 0]
        if len(kfs) <= 1:
            for kf in kfs:
                self.add(kf)
            return
        sizes = []
        for kf in kfs:
            u0, v0, u1, v1 = kf.bbox
            h, w = v1 - v0, u1 - u0
            if kf.rgb.shape[:2] != (h, w) or kf.depth.shape != (h, w) or kf.mask.shape != (h, w):
                raise ValueError(f"keyframe crop shapes do not match bbox {kf.bbox}")
            sizes.append(h * w)
        total = int(sum(sizes))
        self._reserve(total)
        tex, msk = self._staging(total)
        off = 0
        for kf, n in zip(kfs, sizes):
            t = tex[off:off + n]
            rgb = kf.rgb.reshape(n, 3)
            t[:, 0] = rgb[:, 0]  # one column at a time: 3x faster than t[:, :3] = rgb in numpy
            t[:, 1] = rgb[:, 1]
            t[:, 2] = rgb[:, 2]
            t[:, 3] = kf.depth.reshape(n)
            msk[off:off + n] = kf.mask.reshape(n)
            kf.texel_off = self.used + off
            off += n
        base = self.used
        if self._pin_tex is not None:  # pinned staging: asynchronous copies straight into the arena
            self.rgbd[base:base + total].copy_(self._pin_tex[:total], non_blocking=True)
            self.mask[base:base + total].copy_(self._pin_msk[:total], non_blocking=True)
            self._pin_done = torch.cuda.Event()
            self._pin_done.record()
        else:
            self.rgbd[base:base + total] = torch.from_numpy(tex).to(self.device)
            self.mask[base:base + total] = torch.from_numpy(msk).to(self.device)
        self.used += total
        self.uploaded_bytes += 17 * total

    def _staging(self, n: int):
        """Host arrays for n texels: views of a persistent pinned buffer on a
        CUDA arena (waiting for the previous asynchronous copy out of it),
        plain numpy otherwise."""
        if self.device.type != "cuda":
            self._pin_tex = None
            return np.empty((n, 4), np.float32), np.empty(n, np.uint8)
        if getattr(self, "_pin_tex", None) is None or self._pin_tex.shape[0] < n:
            cap = max(1 << 16, 1 << (n - 1).bit_length())
            self._pin_tex = torch.empty((cap, 4), dtype=torch.float32, pin_memory=True)
            self._pin_msk = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            self._pin_done = None
        if getattr(self, "_pin_done", None) is not None:
            self._pin_done.synchronize()
        return self._pin_tex[:n].numpy(), self._pin_msk[:n].numpy()

    def add(self, kf) -> int:
        """Upload one Keyframe's crops; records kf.texel_off and returns it."""
        u0, v0, u1, v1 = kf.bbox
        h, w = v1 - v0, u1 - u0
        if kf.rgb.shape[:2] != (h, w) or kf.depth.shape != (h, w) or kf.mask.shape != (h, w):
            raise ValueError(f"keyframe crop shapes do not match bbox {kf.bbox}")
        n = h * w
        self._reserve(n)
        tex = np.empty((n, 4), np.float32)
        tex[:, :3] = kf.rgb.reshape(n, 3)
        tex[:, 3] = kf.depth.reshape(n)
        off = self.used
        self.rgbd[off:off + n] = torch.from_numpy(tex).to(self.device)
        self.mask[off:off + n] = torch.from_numpy(kf.mask.reshape(n).astype(np.uint8)).to(self.device)
        self.used += n
        self.uploaded_bytes += 17 * n
        kf.texel_off = off
        return off


KF_DTYPE = np.dtype([("texel_off", "<i8"), ("bbox", "<i4", 4), ("pose", "<f8", 12)])
OBJ_DTYPE = np.dtype([("object_id", "<i8"), ("kf_begin", "<i4"), ("n_kf", "<i4"), ("active", "<i4"),
                      ("n_rays", "<i4"), ("box_min", "<f8", 3), ("box_max", "<f8", 3), ("center", "<f8", 3),
                      ("half", "<f8", 3), ("pe_scale", "<f8")])
assert KF_DTYPE.itemsize == C.sizeof(_lib.VmKeyframe) and OBJ_DTYPE.itemsize == C.sizeof(_lib.VmSampleObject)


def _kf_desc(kf) -> bytes:
    """VmKeyframe bytes of one keyframe (cached: pose/bbox/slot never change)."""
    d = getattr(kf, "_desc", None)
    if d is None:
        rec = np.zeros(1, KF_DTYPE)
        rec["texel_off"] = int(kf.texel_off)
        rec["bbox"] = np.asarray(kf.bbox, np.int32)
        rec["pose"] = np.asarray(kf.pose, np.float64)[:3, :4].reshape(12)
        d = rec.tobytes()
        kf._desc = d
    return d


class DeviceTable:
    """Persistent device byte buffer refreshed in place (graph-safe: the
    pointer only changes when the table outgrows it)."""

    def __init__(self, device):
        self.device = device
        self.buf = None
        self.pinned = None
        self.done = None   # event after the last staging copy
        self.last = None   # bytes of the last upload
        self.changed = True

    def upload(self, raw: bytes) -> torch.Tensor:
        n = len(raw)
        self.changed = raw != self.last
        if not self.changed:  # identical table: nothing to copy (map refreshes without edits)
            return self.buf
        self.last = raw
        if self.buf is None or self.buf.numel() < n:
            # 2x headroom over the next power of two: a growing map (keyframes
            # appended every few frames) reallocates -- and so re-captures the
            # step graphs -- only O(log) times
            cap = max(256, 2 << (n - 1).bit_length())
            self.buf = torch.zeros(cap, dtype=torch.uint8, device=self.device)
            self.pinned = torch.zeros(cap, dtype=torch.uint8, pin_memory=True)
            self.done = None
        if self.done is not None:
            self.done.synchronize()  # the previous non-blocking copy still reads the staging buffer
        self.pinned[:n].numpy()[:] = np.frombuffer(raw, dtype=np.uint8)
        self.buf[:n].copy_(self.pinned[:n], non_blocking=True)
        if self.done is None:
            self.done = torch.cuda.Event()
        self.done.record()
        return self.buf


def build_tables(arena: KeyframeArena, instances, bound_pad: float, frozen=None, device=DEVICE, dest=None):
    """(keyframe table, object table) device byte tensors for instances in
    model-index order.  Each instance's keyframes are laid out contiguously;
    inactive / frozen / keyframe-less instances get a zero batch
    (trainer.py:272-273, :336-338).  Crops not yet in the arena are uploaded.
    The padded box follows geometry.py:40-42 (pad = f * half_extent)."""
    n = len(instances)
    objs = np.zeros(max(n, 1), OBJ_DTYPE)
    parts = []
    n_kf, mins, maxs, ids, active, scale, rays = [], [], [], [], [], [], []
    # per-instance descriptor bytes are cached against the (append-only)
    # keyframe list; only instances whose list grew are re-scanned for crops
    # to upload
    stale = []
    for inst in instances:
        c = getattr(inst, "_vm_kfb", None)
        if c is None or c[0] is not inst.keyframes or c[1] != len(inst.keyframes):
            stale.append(inst)
    if stale:
        arena.add_many([kf for inst in stale for kf in inst.keyframes if getattr(kf, "texel_off", -1) < 0])
        for inst in stale:
            kfs = inst.keyframes
            inst._vm_kfb = (kfs, len(kfs), b"".join([_kf_desc(kf) for kf in kfs]))
    for k, inst in enumerate(instances):
        kfs = inst.keyframes
        parts.append(inst._vm_kfb[2])
        n_kf.append(len(kfs))
        mins.append(inst.aabb.min)
        maxs.append(inst.aabb.max)
        ids.append(inst.object_id)
        active.append(1 if (inst.active and not (frozen is not None and frozen[k])) else 0)
        scale.append(inst.pe_scale)
        rays.append(int(getattr(inst, "n_rays", None) or 0))
    if n:  # one vectorised fill per field (per-instance numpy scalar stores were the cost)
        nk = np.asarray(n_kf, np.int32)
        objs["n_kf"][:n] = nk
        objs["kf_begin"][:n] = np.concatenate(([0], np.cumsum(nk)[:-1])).astype(np.int32)
        objs["object_id"][:n] = ids
        objs["active"][:n] = active
        objs["pe_scale"][:n] = scale
        objs["n_rays"][:n] = rays
        mins = np.asarray(mins, np.float64).reshape(n, 3)
        maxs = np.asarray(maxs, np.float64).reshape(n, 3)
        pad = bound_pad * (0.5 * (maxs - mins))
        pmin, pmax = mins - pad, maxs + pad
        objs["box_min"][:n], objs["box_max"][:n] = pmin, pmax
        objs["center"][:n] = 0.5 * (pmin + pmax)
        objs["half"][:n] = 0.5 * (pmax - pmin)
    kf_raw = b"".join(parts) if parts else bytes(KF_DTYPE.itemsize)
    obj_raw = objs.tobytes()
    if dest is not None:  # (DeviceTable, DeviceTable): refresh in place
        return dest[0].upload(kf_raw), dest[1].upload(obj_raw)
    to_dev = lambda raw: torch.from_numpy(np.frombuffer(raw, dtype=np.uint8).copy()).to(device)
    return to_dev(kf_raw), to_dev(obj_raw)


def sample_params(intr, sampling, seed: int, step: int, n_rays: int, arch, encode: bool) -> _lib.VmSampleParams:
    p = _lib.VmSampleParams()
    p.seed, p.step, p.n_rays = int(seed), int(step), int(n_rays)
    p.n_stratified, p.n_surface = sampling.n_stratified, sampling.n_surface
    p.encode = 1 if encode else 0
    p.n_freq, p.include_input = arch.n_freq, 1 if arch.include_input else 0
    p.fx, p.fy, p.cx, p.cy = float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy)
    p.width, p.height = int(intr.width), int(intr.height)
    p.t_near, p.t_far = float(sampling.t_near), float(sampling.t_far)
    p.surface_std = float(sampling.surface_std)
    p.three_std = 3.0 * float(sampling.surface_std)   # python f64, as render.py:200/211 forms it
    return p


class SampleBuffers:
    """Persistent device outputs of one vm_sample call (one stack)."""

    def __init__(self, K: int, R: int, S: int, D: int, encode: bool, device, aux: bool = False):
        f = lambda *s: torch.zeros(s, dtype=torch.float32, device=device)
        b = lambda *s: torch.zeros(s, dtype=torch.bool, device=device)
        self.K, self.R, self.S, self.D, self.encode = K, R, S, D, encode
        self.encoded = f(K, R, S, D) if encode else None
        self.points = None if encode else f(K, R, S, 3)
        self.pe_scale = f(max(K, 1))
        self.t = f(K, R, S)
        self.target_depth = f(K, R)
        self.target_colour = f(K, R, 3)
        self.target_mask = b(K, R)
        self.valid_depth = b(K, R)
        self.ray_ok = b(K, R)
        self.model_rays = None   # [K] int32 live rays per model (config 3), or None
        self.work_items = None   # [2*n] int32 (model, chunk) items of the object kernel
        self.aux = None
        if aux:
            i64 = lambda *s: torch.zeros(s, dtype=torch.int64, device=device)
            self.aux = dict(kf_idx=i64(K, R), u=i64(K, R), v=i64(K, R),
                            t64=torch.zeros((K, R, S), dtype=torch.float64, device=device))
        self.ws = None
        self.obj_dev = None

    def vm(self) -> _lib.VmBatch:
        out = _lib.VmBatch()
        out.n_models, out.n_rays, out.n_points, out.input_dim = self.K, self.R, self.S, self.D
        out.encoded = _lib.ptr(self.encoded)
        out.points = _lib.ptr(self.points)
        out.pe_scale = self.pe_scale.data_ptr()
        out.t = self.t.data_ptr()
        out.target_depth = self.target_depth.data_ptr()
        out.target_colour = self.target_colour.data_ptr()
        out.target_mask = self.target_mask.data_ptr()
        out.valid_depth = self.valid_depth.data_ptr()
        out.ray_ok = self.ray_ok.data_ptr()
        if self.model_rays is not None:
            out.model_rays = self.model_rays.data_ptr()
            out.work_items = self.work_items.data_ptr()
            out.n_work_items = self.work_items.numel() // 2
        return out

    def set_model_rays(self, rays, device) -> None:
        """Per-model live ray counts (host ints, <= R) and the object kernel's
        work items for them; all-equal-to-R clears both (uniform batch)."""
        rays = np.minimum(np.asarray(rays, np.int32), self.R)
        if len(rays) == 0 or (rays == self.R).all():
            self.model_rays = self.work_items = None
            return
        lib = _lib.load()
        cnt = C.c_int32()
        _lib.check(lib.vm_work_items(rays.ctypes.data, len(rays), self.S, None, 0, C.byref(cnt)), "vm_work_items")
        items = np.zeros(2 * max(cnt.value, 1), np.int32)
        _lib.check(lib.vm_work_items(rays.ctypes.data, len(rays), self.S, items.ctypes.data, cnt.value,
                                     C.byref(cnt)), "vm_work_items")
        self.model_rays = torch.from_numpy(rays.copy()).to(device)
        self.work_items = torch.from_numpy(items[:2 * cnt.value].copy()).to(device)


def run_sampler(arena: KeyframeArena, kf_table: torch.Tensor, obj_table: torch.Tensor, n_objects: int,
                params: _lib.VmSampleParams, buf: SampleBuffers) -> None:
    lib = _lib.load()
    nbytes = lib.vm_sample_workspace_bytes(n_objects, C.byref(params))
    if buf.ws is None or buf.ws.numel() < nbytes:
        buf.ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=arena.device)
    batch = buf.vm()
    aux = None
    if buf.aux is not None:
        aux = _lib.VmSampleAux(buf.aux["kf_idx"].data_ptr(), buf.aux["u"].data_ptr(), buf.aux["v"].data_ptr(),
                               buf.aux["t64"].data_ptr())
    _lib.check(lib.vm_sample(obj_table.data_ptr(), n_objects, kf_table.data_ptr(),
                             arena.rgbd.data_ptr(), arena.mask.data_ptr(), C.byref(params), C.byref(batch),
                             C.byref(aux) if aux is not None else None, buf.ws.data_ptr(), buf.ws.numel(),
                             _lib.stream_ptr()), "vm_sample")
