"""Mapper: the per-step map update on the B200 (drop-in for vobj Mapper.train_step).

Reference: trainer.py:203-402.  One `train_step` is, on the device:
  vm_sample(objects) + vm_sample(background)   -- KS, bit-exact pixel/ray/t draws
  vm_train_step([objects, background])         -- KF fused MLP fwd/bwd (+ PE) and KA Adam
followed by ONE device->host copy of the per-model losses and status words,
from which the StepReport and the reference's exceptions are built.
Batch buffers, tables and workspaces persist across steps, so a step is four
kernel launches and one small D2H copy.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import _lib
from .keyframes import KeyframeArena, SampleBuffers, build_tables, run_sampler, sample_params
from .models import DEVICE, append_model, init_stacked, set_frozen
from .objects import ObjectMap, add_keyframe
from .render import CameraIntrinsics
from .rng import PURPOSE_INIT_BACKGROUND, PURPOSE_INIT_OBJECT
from .trainer import StepReport, TrainConfig, TrainWorkspace, launch_train


class Mapper:
    """Owns the object map and both model stacks (trainer.py:203-222)."""

    def __init__(self, intrinsics: CameraIntrinsics, cfg: TrainConfig | None = None, device=DEVICE,
                 object_id_base: int = 0, init_index_base: int = 0, background_init_index: int = 0):
        self.cfg = cfg if cfg is not None else TrainConfig()
        self.intrinsics = intrinsics
        self.device = torch.device(device)
        self.map = ObjectMap()
        self.map._next_id = object_id_base + 1   # globally unique ids across object-sharded ranks
        self._init_base = init_index_base
        self._bg_init = background_init_index
        self._io = (0, 0)
        c = self.cfg
        self.obj_params, self.obj_state = init_stacked(c.arch_object, 0, c.seed, PURPOSE_INIT_OBJECT, lr=c.lr,
                                                       beta1=c.beta1, beta2=c.beta2, eps=c.eps, device=device)
        self.bg_params, self.bg_state = init_stacked(c.arch_background, 0, c.seed, PURPOSE_INIT_BACKGROUND,
                                                     lr=c.lr, beta1=c.beta1, beta2=c.beta2, eps=c.eps,
                                                     device=device)
        self.model_to_object: list[int] = []
        self.global_step = 0
        self.frames_seen = 0
        self.last_frame_id = -1
        self.arena = KeyframeArena(device)
        self._ws = TrainWorkspace()
        self._sig = None
        self._tables = None
        self._buf_obj = None
        self._buf_bg = None
        self._host_out = None

    # ------------------------------------------------------------ building
    def add_background(self, aabb, pe_scale: float | None = None):
        idx = append_model(self.bg_params, self.bg_state, self.cfg.seed, PURPOSE_INIT_BACKGROUND,
                           init_index=self._bg_init + self.bg_params.count)
        scale = self.cfg.pe_scale_background if pe_scale is None else pe_scale
        return self.map.add_background(aabb, scale, idx)

    def add_object(self, semantic_class: int, aabb, pe_scale: float | None = None):
        """append_model + ObjectMap.add_object + model_to_object (trainer.py:254-256)."""
        idx = append_model(self.obj_params, self.obj_state, self.cfg.seed, PURPOSE_INIT_OBJECT,
                           init_index=self._init_base + self.obj_params.count)
        scale = self.cfg.pe_scale_object if pe_scale is None else pe_scale
        inst = self.map.add_object(semantic_class, aabb, scale, idx)
        self.model_to_object.append(inst.object_id)
        return inst

    def add_keyframe(self, inst, frame_id, pose, bbox, mask, rgb, depth):
        kf = add_keyframe(inst, frame_id, pose, bbox, mask, rgb, depth)
        self.arena.add(kf)
        self.invalidate()
        return kf

    def invalidate(self) -> None:
        """Force the device tables to be rebuilt (after editing boxes/keyframes)."""
        self._sig = None

    def freeze_object(self, object_id: int, frozen: bool = True) -> None:
        inst = self.map.instances[object_id]
        params = self.bg_params if inst.is_background else self.obj_params
        set_frozen(params, inst.model_index, frozen)
        self.invalidate()

    def instance_for_model(self, index: int):
        return self.map.instances[self.model_to_object[index]]

    # ------------------------------------------------------------ device sync
    def _signature(self):
        objs = [self.map.instances[o] for o in self.model_to_object]
        bg = self.map.background
        return (len(objs), sum(len(i.keyframes) for i in objs), bg is not None,
                len(bg.keyframes) if bg is not None else 0,
                self.obj_params.frozen[:self.obj_params.count].tobytes(),
                self.bg_params.frozen[:self.bg_params.count].tobytes())

    def _sync(self) -> None:
        sig = self._signature()
        if sig == self._sig:
            return
        c = self.cfg
        S = c.points_per_ray
        objs = [self.map.instances[o] for o in self.model_to_object]
        pad = c.association.bound_pad
        t_obj = build_tables(self.arena, objs, pad, self.obj_params.frozen, self.device) if objs else None
        bg = self.map.background
        t_bg = build_tables(self.arena, [bg], pad, self.bg_params.frozen[bg.model_index:bg.model_index + 1],
                            self.device) if bg is not None else None
        K = len(objs)
        if K and (self._buf_obj is None or self._buf_obj.K != K):
            self._buf_obj = SampleBuffers(K, c.rays_per_object, S, c.arch_object.input_dim, False, self.device)
        if bg is not None and self._buf_bg is None:
            self._buf_bg = SampleBuffers(1, c.rays_background, S, c.arch_background.input_dim, False, self.device)
        if K:
            self._buf_obj.pe_scale[:K] = torch.tensor([float(i.pe_scale) for i in objs], device=self.device)
        if bg is not None:
            self._buf_bg.pe_scale[:1] = float(bg.pe_scale)
        self._tables = (t_obj, t_bg)
        self._sig = sig
        up = sum(t.numel() for tab in self._tables if tab is not None for t in tab) + 4 * (K + (bg is not None))
        self._io = (up, self._io[1])

    # ------------------------------------------------------------ sampling API
    def assemble(self, step: int, background: bool = False, encode: bool = True, aux: bool = False) -> SampleBuffers:
        """Device RaySampleBatch for every object model (or the background) at
        `step` -- the batched equivalent of trainer.py:269-318 / :332-352.
        With encode=True the positional encoding is materialised in f64->f32
        exactly like models.py:286-308 (reference layout)."""
        c = self.cfg
        self._sync()
        t_obj, t_bg = self._tables
        if background:
            arch, n, tabs, R = c.arch_background, 1, t_bg, c.rays_background
        else:
            arch, n, tabs, R = c.arch_object, self.obj_params.count, t_obj, c.rays_per_object
        buf = SampleBuffers(n, R, c.points_per_ray, arch.input_dim, encode, self.device, aux=aux)
        if n and tabs is not None:
            p = sample_params(self.intrinsics, c.sampling, c.seed, step, R, arch, encode)
            run_sampler(self.arena, tabs[0], tabs[1], n, p, buf)
        return buf

    # ------------------------------------------------------------ training
    def enqueue_step(self, step: int):
        """Launch sampling + fused training for `step` without host sync.

        Returns (losses [K(+1), 3], status) device tensors and the stack list.
        """
        c = self.cfg
        self._sync()
        t_obj, t_bg = self._tables
        stacks = []
        if self.obj_params.count > 0:
            p = sample_params(self.intrinsics, c.sampling, c.seed, step, c.rays_per_object, c.arch_object, False)
            run_sampler(self.arena, t_obj[0], t_obj[1], self.obj_params.count, p, self._buf_obj)
            stacks.append((self.obj_params, self.obj_state, self._buf_obj))
        bg = self.map.background
        if c.train_background and bg is not None:
            p = sample_params(self.intrinsics, c.sampling, c.seed, step, c.rays_background, c.arch_background,
                              False)
            run_sampler(self.arena, t_bg[0], t_bg[1], 1, p, self._buf_bg)
            stacks.append((self.bg_params, self.bg_state, self._buf_bg))
        if not stacks:
            return None, None, stacks
        losses, status = launch_train(stacks, c.loss_weights, self._ws)
        return losses, status, stacks

    def last_io_bytes(self) -> tuple[int, int]:
        """(host->device bytes of the last table upload, device->host bytes per step)."""
        return self._io

    def train_step(self, mode: str = "vectorised") -> StepReport:
        """trainer.py:356-402."""
        if mode not in ("vectorised", "sequential"):
            raise ValueError(f"unknown training mode {mode!r}")
        step = self.global_step
        t0 = time.perf_counter()
        losses, status, stacks = self.enqueue_step(step)
        report_losses: dict[int, tuple[float, float, float]] = {}
        k_models = 0
        if stacks:
            n = losses.shape[0]
            packed = torch.cat([losses.reshape(-1).view(torch.int32), status])
            if self._host_out is None or self._host_out.numel() != packed.numel():
                self._host_out = torch.empty(packed.numel(), dtype=torch.int32, pin_memory=True)
            self._host_out.copy_(packed)  # one D2H copy per step (synchronises)
            self._io = (self._io[0], packed.numel() * 4)
            host = self._host_out.numpy()
            l = host[:3 * n].view(np.float32).reshape(n, 3)
            st = host[3 * n:].reshape(-1, 4)
            row = 0
            for si, (params, _, _) in enumerate(stacks):
                is_bg = params is self.bg_params
                kk = params.count
                if st[si, 0] < kk:
                    raise FloatingPointError(f"non-finite gradient for model index {int(st[si, 0])}")
                for j in range(kk):
                    oid = 0 if is_bg else self.model_to_object[j]
                    vals = l[row + j]
                    if not np.all(np.isfinite(vals)):
                        raise FloatingPointError(f"non-finite loss for object {oid}")
                    report_losses[oid] = (float(vals[0]), float(vals[1]), float(vals[2]))
                row += kk
                k_models += kk
        w = self.cfg.loss_weights
        total = sum(d + w.colour * c + w.occupancy * o for d, c, o in report_losses.values())
        self.global_step += 1
        return StepReport(step=step, frame_id=self.last_frame_id, k_models=k_models, losses=report_losses,
                          total=float(total), ms=(time.perf_counter() - t0) * 1e3)
