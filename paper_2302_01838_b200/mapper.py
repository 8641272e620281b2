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

import os
import time

import numpy as np
import torch

from . import _lib
from .keyframes import DeviceTable, KeyframeArena, SampleBuffers, build_tables, run_sampler, sample_params
from .models import DEVICE, append_model, init_stacked, set_frozen
from .ingest import FrameIngestor, associate, extract_detections_device, keyframe_due, update_bounds
from .objects import ObjectMap, add_keyframe, dilate_bbox
from .render import CameraIntrinsics
from .rng import PURPOSE_INIT_BACKGROUND, PURPOSE_INIT_OBJECT
from .trainer import StepReport, TrainConfig, TrainWorkspace, launch_train


class Mapper:
    """Owns the object map and both model stacks (trainer.py:203-222)."""

    def __init__(self, intrinsics: CameraIntrinsics, cfg: TrainConfig | None = None, device=DEVICE,
                 object_id_base: int = 0, init_index_base: int = 0, background_init_index: int = 0,
                 use_graphs: bool = True, fused_pe: bool | None = None):
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
        self.use_graphs = use_graphs
        # The sampler materialises the positional encoding in f64 -> f32
        # exactly like models.py:286-308 (bit-identical MLP inputs); with
        # fused_pe the MLP kernels encode f32 points on the fly instead
        # (fewer bytes, f32 sincospif: tolerance-level inputs).
        if fused_pe is None:
            fused_pe = os.environ.get("VM_FUSED_PE", "0") == "1"
        self.encode = not fused_pe
        self._g = None          # graph-replay state (see _graph_step)
        self._dev_tables = [(DeviceTable(self.device), DeviceTable(self.device)) for _ in range(2)]
        self._dirty = True
        self._pin_scale = None
        self._pin_done = None
        self._last_scales = None
        self._tables_gen = 0
        self._n_kf = 0
        self._ingest = None

    # ------------------------------------------------------------ building
    def add_background(self, aabb, pe_scale: float | None = None):
        idx = append_model(self.bg_params, self.bg_state, self.cfg.seed, PURPOSE_INIT_BACKGROUND,
                           init_index=self._bg_init + self.bg_params.count)
        scale = self.cfg.pe_scale_background if pe_scale is None else pe_scale
        return self.map.add_background(aabb, scale, idx)

    def add_object(self, semantic_class: int, aabb, pe_scale: float | None = None, object_id: int | None = None,
                   init_index: int | None = None, n_rays: int | None = None):
        """append_model + ObjectMap.add_object + model_to_object (trainer.py:254-256).

        `object_id` / `init_index` place a shard of a global map: the object
        keeps its global id (sampling streams are keyed by it, objects.py:335)
        and its global append index as the init key (models.py:264-267,
        SURVEY 8e init-key caveat), so every rank reproduces the single-stack
        run for the objects it owns."""
        if init_index is None:
            init_index = self._init_base + self.obj_params.count
        idx = append_model(self.obj_params, self.obj_state, self.cfg.seed, PURPOSE_INIT_OBJECT,
                           init_index=init_index)
        scale = self.cfg.pe_scale_object if pe_scale is None else pe_scale
        inst = self.map.add_object(semantic_class, aabb, scale, idx, object_id=object_id)
        if n_rays is not None:
            if not 1 <= int(n_rays) <= self.cfg.rays_per_object:
                raise ValueError(f"n_rays must be in [1, rays_per_object={self.cfg.rays_per_object}]")
            inst.n_rays = int(n_rays)
        self.model_to_object.append(inst.object_id)
        return inst

    def add_keyframe(self, inst, frame_id, pose, bbox, mask, rgb, depth):
        kf = add_keyframe(inst, frame_id, pose, bbox, mask, rgb, depth)
        self.invalidate()  # the crop is uploaded with the frame's others at the next table build
        return kf

    # ------------------------------------------------------------ ingestion
    def process_frame(self, frame, classes: dict | None = None) -> None:
        """trainer.py:226-265: scene bounds and instance detections of the
        frame (device kernels, ingest.py), association, box growth,
        new objects and keyframes at the per-object stride."""
        cfg = self.cfg
        acfg = cfg.association
        classes = classes if classes is not None else {}
        if self._ingest is None:
            self._ingest = FrameIngestor(self.device)
        detections, bounds = extract_detections_device(self._ingest, frame, self.intrinsics, classes, acfg)
        bg = self.map.background
        if bg is None:
            if bounds is None:
                raise ValueError(f"frame {frame.frame_id}: no valid depth to bound the scene")
            bg = self.add_background(bounds)
        elif bounds is not None:
            update_bounds(bg, bounds)
        bg.obs_count += 1
        if keyframe_due(bg, acfg):
            h, w = frame.depth.shape
            self.add_keyframe(bg, frame.frame_id, frame.pose, (0, 0, w, h), frame.mask == 0, frame.rgb, frame.depth)
        assignments = associate(detections, self.map, acfg)
        for det, assigned in zip(detections, assignments):
            if assigned is None:
                inst = self.add_object(det.semantic_class, det.aabb)
            else:
                inst = self.map.instances[assigned]
                update_bounds(inst, det.aabb)
            inst.obs_count += 1
            if keyframe_due(inst, acfg):
                bbox, mask = dilate_bbox(det.bbox, det.mask, acfg.bbox_margin_px, frame.depth.shape)
                self.add_keyframe(inst, frame.frame_id, frame.pose, bbox, mask, frame.rgb, frame.depth)
        self.frames_seen += 1
        self.last_frame_id = frame.frame_id
        self.invalidate()  # boxes may have grown

    def invalidate(self) -> None:
        """Force the device tables to be rebuilt (after editing boxes/keyframes,
        as process_frame does); the captured step graphs stay valid because the
        tables are refreshed in place."""
        self._dirty = True

    def freeze_object(self, object_id: int, frozen: bool = True) -> None:
        inst = self.map.instances[object_id]
        params = self.bg_params if inst.is_background else self.obj_params
        set_frozen(params, inst.model_index, frozen)
        self.invalidate()

    def instance_for_model(self, index: int):
        return self.map.instances[self.model_to_object[index]]

    # ------------------------------------------------------------ device sync
    def _signature(self):
        """Cheap structural signature: model counts, keyframe count, frozen bits."""
        n_kf = sum(len(self.map.instances[o].keyframes) for o in self.model_to_object) if self._dirty else self._n_kf
        bg = self.map.background
        return (len(self.model_to_object), n_kf, bg is not None, len(bg.keyframes) if bg is not None else 0,
                self.obj_params.frozen[:self.obj_params.count].tobytes(),
                self.bg_params.frozen[:self.bg_params.count].tobytes())

    def _sync(self) -> None:
        if not self._dirty and self._sig is not None:
            # fast path: only the frozen bits can change behind our back
            if (self.obj_params.frozen[:self.obj_params.count].tobytes() == self._sig[4]
                    and self.bg_params.frozen[:self.bg_params.count].tobytes() == self._sig[5]):
                return
        sig = self._signature()
        c = self.cfg
        S = c.points_per_ray
        objs = [self.map.instances[o] for o in self.model_to_object]
        self._n_kf = sum(len(i.keyframes) for i in objs)
        pad = c.association.bound_pad
        t_obj = build_tables(self.arena, objs, pad, self.obj_params.frozen, self.device,
                             dest=self._dev_tables[0]) if objs else None
        bg = self.map.background
        t_bg = build_tables(self.arena, [bg], pad, self.bg_params.frozen[bg.model_index:bg.model_index + 1],
                            self.device, dest=self._dev_tables[1]) if bg is not None else None
        K = len(objs)
        if K and (self._buf_obj is None or self._buf_obj.K != K):
            self._buf_obj = SampleBuffers(K, c.rays_per_object, S, c.arch_object.input_dim, self.encode, self.device)
            self._g = None  # batch buffers reallocated: the step graphs must be recaptured
        if K:  # per-object ray counts (config 3): live rows + the object kernel's work items
            rays = tuple(int(i.n_rays or c.rays_per_object) for i in objs)
            if rays != getattr(self._buf_obj, "_rays_sig", None):
                self._buf_obj.set_model_rays(rays, self.device)
                self._buf_obj._rays_sig = rays
                self._g = None  # grid size / table pointers changed
        if bg is not None and self._buf_bg is None:
            self._buf_bg = SampleBuffers(1, c.rays_background, S, c.arch_background.input_dim, self.encode,
                                         self.device)
            self._g = None
        # frozen bits live in persistent device buffers the graphs read
        if self.obj_params.count:
            self.obj_params.frozen_device()
        if self.bg_params.count:
            self.bg_params.frozen_device()
        # PE scales through one pinned staging buffer (non-blocking uploads)
        sc = np.array([float(i.pe_scale) for i in objs] + ([float(bg.pe_scale)] if bg is not None else []),
                      np.float32)
        regraph = self._g is None
        same_len = self._last_scales is not None and len(sc) == len(self._last_scales)
        obj_changed = (not same_len or any(d.changed for d in self._dev_tables[0])
                       or not np.array_equal(sc[:K], self._last_scales[:K]))
        bg_changed = (not same_len or any(d.changed for d in self._dev_tables[1])
                      or not np.array_equal(sc[K:], self._last_scales[K:]))
        unchanged = not regraph and not obj_changed and not bg_changed
        self._last_scales = sc
        if unchanged:
            # a refresh without edits (e.g. invalidate() after a frame that
            # changed nothing): the tables, scales and the prefetched batch stay valid
            self._tables = (t_obj, t_bg)
            self._tables_gen += 1
            self._sig = sig
            self._dirty = False
            self._io = (0, self._io[1])
            return
        if self._pin_scale is None or self._pin_scale.numel() < max(len(sc), 1):
            self._pin_scale = torch.empty(max(len(sc), 64), dtype=torch.float32, pin_memory=True)
        if len(sc):
            if self._pin_done is not None:
                self._pin_done.synchronize()  # previous non-blocking upload still reads it
            self._pin_scale[:len(sc)].numpy()[:] = sc
        if K:
            self._buf_obj.pe_scale[:K].copy_(self._pin_scale[:K], non_blocking=True)
        if bg is not None:
            self._buf_bg.pe_scale[:1].copy_(self._pin_scale[K:K + 1], non_blocking=True)
        if len(sc):
            if self._pin_done is None:
                self._pin_done = torch.cuda.Event()
            self._pin_done.record()
        if self._g is not None:  # keep the graphs' second batch buffers' PE scales in step
            for a, b in zip(self._g["bufs"], (self._buf_obj, self._buf_bg)):
                if a is not None and b is not None:
                    a.pe_scale.copy_(b.pe_scale)
            # tables changed: drop the prefetched batch of the stack(s) concerned
            if obj_changed:
                self._g["next_ready_obj"] = None
            if bg_changed:
                self._g["next_ready_bg"] = None
        self._tables = (t_obj, t_bg)
        self._tables_gen += 1
        self._sig = sig
        self._dirty = False
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
            p = sample_params(self.intrinsics, c.sampling, c.seed, step, c.rays_per_object, c.arch_object,
                              self.encode)
            run_sampler(self.arena, t_obj[0], t_obj[1], self.obj_params.count, p, self._buf_obj)
            stacks.append((self.obj_params, self.obj_state, self._buf_obj))
        bg = self.map.background
        if c.train_background and bg is not None:
            p = sample_params(self.intrinsics, c.sampling, c.seed, step, c.rays_background, c.arch_background,
                              self.encode)
            run_sampler(self.arena, t_bg[0], t_bg[1], 1, p, self._buf_bg)
            stacks.append((self.bg_params, self.bg_state, self._buf_bg))
        if not stacks:
            return None, None, stacks
        losses, status = launch_train(stacks, c.loss_weights, self._ws)
        return losses, status, stacks

    # ------------------------------------------------------------ graph replay
    def _graph_key(self):
        """Everything a captured step graph bakes in: device pointers and the
        model counts (grid sizes).  Keyframe counts, boxes, active and frozen
        bits are NOT part of it -- they live in device tables refreshed in
        place, so map growth at the steps_per_frame cadence replays the same
        graphs (only arena or table reallocation forces a recapture)."""
        tabs = tuple(t.data_ptr() for tab in self._tables if tab is not None for t in tab)
        bufs = tuple(b.t.data_ptr() for b in (self._buf_obj, self._buf_bg) if b is not None)
        frz = tuple(p.frozen_device().data_ptr() for p in (self.obj_params, self.bg_params) if p.count)
        rays = getattr(self._buf_obj, "_rays_sig", None)
        return (tabs, bufs, frz, rays, self.arena.rgbd.data_ptr(), self.arena.mask.data_ptr(),
                self.obj_params.arena.data_ptr(), self.bg_params.arena.data_ptr(),
                self.obj_params.count, self.bg_params.count, self.cfg.train_background)

    def _build_graphs(self):
        """Capture two CUDA graphs (step parity p = 0, 1).  Graph p trains
        step t from batch buffer p while a forked stream samples step t+1 into
        buffer 1-p (the sampler only reads keyframes, never parameters, so it
        overlaps training); then it copies losses/status to pinned host memory
        and bumps the device step counter."""
        c = self.cfg
        dev = self.device
        objs_n = self.obj_params.count
        bg = self.map.background
        has_bg = c.train_background and bg is not None
        S = c.points_per_ray
        bufs_o = [self._buf_obj, SampleBuffers(objs_n, c.rays_per_object, S, c.arch_object.input_dim, self.encode, dev)
                  ] if objs_n else [None, None]
        bufs_b = [self._buf_bg, SampleBuffers(1, c.rays_background, S, c.arch_background.input_dim, self.encode, dev)
                  ] if has_bg else [None, None]
        if objs_n:
            bufs_o[1].pe_scale.copy_(bufs_o[0].pe_scale)
            bufs_o[1].model_rays, bufs_o[1].work_items = bufs_o[0].model_rays, bufs_o[0].work_items
        if has_bg:
            bufs_b[1].pe_scale.copy_(bufs_b[0].pe_scale)
        step_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        t_obj, t_bg = self._tables

        def sample_obj(p, offset):
            if objs_n:
                sp = sample_params(self.intrinsics, c.sampling, c.seed, 0, c.rays_per_object, c.arch_object,
                                   self.encode)
                sp.step_dev, sp.step_offset = step_dev.data_ptr(), offset
                run_sampler(self.arena, t_obj[0], t_obj[1], objs_n, sp, bufs_o[p])

        def sample_bg(p, offset):
            if has_bg:
                sp = sample_params(self.intrinsics, c.sampling, c.seed, 0, c.rays_background, c.arch_background,
                                   self.encode)
                sp.step_dev, sp.step_offset = step_dev.data_ptr(), offset
                run_sampler(self.arena, t_bg[0], t_bg[1], 1, sp, bufs_b[p])

        def sample(p, offset):
            sample_obj(p, offset)
            sample_bg(p, offset)

        def stacks(p):
            out = []
            if objs_n:
                out.append((self.obj_params, self.obj_state, bufs_o[p]))
            if has_bg:
                out.append((self.bg_params, self.bg_state, bufs_b[p]))
            return out

        # eager warm-up of both buffers/workspaces (allocations must precede capture)
        for p in (0, 1):
            sample(p, 0)
        launch_train(stacks(0), c.loss_weights, self._ws, bump_version=False)  # state restored by caller
        torch.cuda.synchronize(dev)
        n = sum(p.count for p, _, _ in stacks(0))
        n_st = len(stacks(0))
        host_io = torch.empty(3 * max(n, 1) + 4 * n_st, dtype=torch.int32, pin_memory=True)
        host_l = host_io[:3 * max(n, 1)].view(torch.float32).view(max(n, 1), 3)[:n]
        host_s = host_io[3 * max(n, 1):]
        side = torch.cuda.Stream(dev)
        side_bg = torch.cuda.Stream(dev)
        sample_first = os.environ.get("VM_SAMPLE_FIRST", "0") == "1"  # A/B: capture the sampler first
        graphs = []
        for p in (0, 1):
            g = torch.cuda.CUDAGraph()
            main = torch.cuda.Stream(dev)
            with torch.cuda.stream(main):
                # relaxed: a capture-unsafe call elsewhere in the process (e.g. a
                # previous Mapper's graphs or pinned buffers being released by
                # the garbage collector) must not invalidate this capture
                with torch.cuda.graph(g, stream=main, capture_error_mode="relaxed"):
                    cur = torch.cuda.current_stream()
                    # step t+1's objects and background are sampled on two
                    # forked streams, concurrently with each other and with
                    # step t's training
                    side.wait_stream(cur)
                    side_bg.wait_stream(cur)
                    if sample_first:
                        with torch.cuda.stream(side):
                            sample_obj(1 - p, 1)
                        with torch.cuda.stream(side_bg):
                            sample_bg(1 - p, 1)
                    losses, status = launch_train(stacks(p), c.loss_weights, self._ws, bump_version=False)
                    if not sample_first:
                        # captured after the training kernels (they still do not
                        # depend on each other), so the graph launches the
                        # training grids first and the sampler's many small CTAs
                        # fill in behind them instead of delaying them
                        with torch.cuda.stream(side):
                            sample_obj(1 - p, 1)
                        with torch.cuda.stream(side_bg):
                            sample_bg(1 - p, 1)
                    cur.wait_stream(side)
                    cur.wait_stream(side_bg)
                    # losses + status straight into pinned host memory, and the
                    # device step counter bump, in one kernel
                    res = self._ws.results(n, n_st)
                    _lib.check(_lib.load().vm_step_finish(res.data_ptr(), host_io.data_ptr(), res.numel(),
                                                          step_dev.data_ptr(), 1, _lib.stream_ptr()),
                               "vm_step_finish")
            graphs.append(g)
        execs = []
        for g in graphs:
            try:
                execs.append(int(g.raw_cuda_graph_exec()))
            except (AttributeError, RuntimeError):
                execs.append(0)
        self._g = dict(execs=execs, key=self._graph_key(), graphs=graphs, step_dev=step_dev, host_l=host_l, host_s=host_s,
                       stacks=[stacks(0), stacks(1)], sample_obj=sample_obj, sample_bg=sample_bg,
                       next_ready_obj=None, next_ready_bg=None,
                       bufs=(bufs_o[1], bufs_b[1]))

    def enqueue_graph_step(self, step: int):
        """Replay the captured step graph for `step` on the current stream
        (no host sync).  Results land in pinned host memory when the stream
        reaches them."""
        self._sync()
        # the full graph key (device pointers of every table and buffer) is
        # re-derived only after a table rebuild; in between, model counts and
        # arena pointers guard against growth outside the Mapper's API
        quick = (self.obj_params.count, self.bg_params.count, self.obj_params.arena.data_ptr(),
                 self.bg_params.arena.data_ptr(), self._tables_gen)
        if self._g is None or self._g.get("quick") != quick:
            if self._g is None or self._g["key"] != self._graph_key():
                self._snapshot_for_graph_build()
                self._build_graphs()
                self._restore_after_graph_build()
            self._g["quick"] = quick
        g = self._g
        p = step & 1
        if g.get("dev_step") != step:  # the graph bumps the device counter itself
            g["step_dev"].fill_(step)
        # no prefetched batch for this step (first step, or that stack's map
        # changed): sample it now
        if g["next_ready_obj"] != step:
            g["sample_obj"](p, 0)
        if g["next_ready_bg"] != step:
            g["sample_bg"](p, 0)
        ex = g["execs"][p] if _DIRECT_LAUNCH else 0
        if ex:  # the instantiated graph straight through cudaGraphLaunch (no Python replay wrapper)
            _lib.check(_lib.load().vm_graph_launch(ex, _lib.stream_ptr()), "vm_graph_launch")
        else:
            g["graphs"][p].replay()
        g["next_ready_obj"] = g["next_ready_bg"] = step + 1
        g["dev_step"] = step + 1
        for params, _, _ in g["stacks"][p]:
            params.version += 1
        return g["stacks"][p]

    def _graph_step(self, step: int):
        stacks = self.enqueue_graph_step(step)
        torch.cuda.current_stream().synchronize()
        g = self._g
        return g["host_l"].numpy(), g["host_s"].numpy().reshape(-1, 4), stacks

    def _snapshot_for_graph_build(self):
        """Graph capture needs one eager warm-up launch; keep the model state
        untouched by saving/restoring params, Adam moments and step counters."""
        self._sync()
        snap = []
        for p, s in ((self.obj_params, self.obj_state), (self.bg_params, self.bg_state)):
            snap.append((p.arena.clone(), s.m_arena.clone(), s.v_arena.clone(), s.step.clone(), p.version))
        self._snap = snap

    def _restore_after_graph_build(self):
        for (a, m, v, st, ver), (p, s) in zip(self._snap, ((self.obj_params, self.obj_state),
                                                        (self.bg_params, self.bg_state))):
            p.arena.copy_(a)
            s.m_arena.copy_(m)
            s.v_arena.copy_(v)
            s.step.copy_(st)
            p.version = ver
        self._snap = None
        torch.cuda.synchronize(self.device)

    def kernels_per_step(self) -> int:
        """Kernels of ours one graph-replayed step launches: per stack a sampler
        prep + ray kernel, plus the fused MLP, Adam, the partial reduce when a
        model is split over CTAs, and the step-counter bump."""
        n_st = (self.obj_params.count > 0) + (self.cfg.train_background and self.map.background is not None)
        split = 1 if (self.cfg.train_background and self.map.background is not None) else 0
        return 2 * n_st + 2 + split + 1

    def last_io_bytes(self) -> tuple[int, int]:
        """(host->device bytes of the last table upload, device->host bytes per step)."""
        return self._io

    def train_step(self, mode: str = "vectorised") -> StepReport:
        """trainer.py:356-402."""
        if mode not in ("vectorised", "sequential"):
            raise ValueError(f"unknown training mode {mode!r}")
        step = self.global_step
        t0 = time.perf_counter()
        report_losses: dict[int, tuple[float, float, float]] = {}
        k_models = 0
        self._sync()
        has_work = self.obj_params.count > 0 or (self.cfg.train_background and self.map.background is not None)
        if has_work and self.use_graphs and mode == "vectorised":
            l, st, stacks = self._graph_step(step)
            self._io = (self._io[0], l.nbytes + st.nbytes)
        elif has_work:
            losses, status, stacks = self.enqueue_step(step)
            n = losses.shape[0]
            packed = torch.cat([losses.reshape(-1).view(torch.int32), status])
            if self._host_out is None or self._host_out.numel() != packed.numel():
                self._host_out = torch.empty(packed.numel(), dtype=torch.int32, pin_memory=True)
            self._host_out.copy_(packed)  # one D2H copy per step (synchronises)
            self._io = (self._io[0], packed.numel() * 4)
            host = self._host_out.numpy()
            l = host[:3 * n].view(np.float32).reshape(n, 3)
            st = host[3 * n:].reshape(-1, 4)
        else:
            stacks = []
        w = self.cfg.loss_weights
        wc, wo = w.colour, w.occupancy
        total = 0
        counts = [params.count for params, _, _ in stacks]
        n_rows = sum(counts)
        v64 = l[:n_rows].astype(np.float64) if stacks else None
        fast = not stacks or (all(st[si, 0] >= kk and st[si, 1] >= kk for si, kk in enumerate(counts))
                              and bool(np.isfinite(v64).all()))
        if not stacks:
            pass
        elif fast:
            # one conversion for every model's row, no per-stack Python loop
            ids = []
            for params, _, _ in stacks:
                ids.extend([0] if params is self.bg_params else self.model_to_object[:params.count])
            report_losses = dict(zip(ids, map(tuple, v64.tolist())))
            k_models = n_rows
            if len(report_losses) == n_rows and n_rows:
                # the reference's left-to-right sum over report.losses.values()
                # (np.add.accumulate is sequential; same f64 operations and order)
                total = np.add.accumulate(v64[:, 0] + wc * v64[:, 1] + wo * v64[:, 2])[-1]
            else:
                for d, c, o in report_losses.values():
                    total += d + wc * c + wo * o
        else:  # a status word or a loss is bad: raise the reference's error, in stack order
            row = 0
            for si, (params, _, _) in enumerate(stacks):
                is_bg = params is self.bg_params
                kk = params.count
                if st[si, 0] < kk:
                    raise FloatingPointError(f"non-finite gradient for model index {int(st[si, 0])}")
                vals = l[row:row + kk]
                ids = [0] if is_bg else self.model_to_object
                if st[si, 1] < kk or not np.isfinite(vals).all():
                    bad = int(np.flatnonzero(~np.isfinite(vals).all(axis=1))[0])
                    raise FloatingPointError(f"non-finite loss for object {ids[bad]}")
                row += kk
            raise FloatingPointError("non-finite loss")
        self.global_step += 1
        return StepReport(step=step, frame_id=self.last_frame_id, k_models=k_models, losses=report_losses,
                          total=float(total), ms=(time.perf_counter() - t0) * 1e3)


# VM_GRAPH_LAUNCH=1 launches the step graphs through vm_graph_launch
# (cudaGraphLaunch) instead of torch's CUDAGraph.replay(): measured no
# faster (0.1408 vs 0.1398 ms/step), so replay stays the default
_DIRECT_LAUNCH = os.environ.get("VM_GRAPH_LAUNCH", "0") == "1"


def run_mapping(dataset, cfg: TrainConfig | None = None, mode: str = "vectorised", progress: bool = False,
                device=DEVICE):
    """trainer.py:541-569: per frame, ingest then train steps_per_frame
    steps.  Frames are decoded ahead on a worker thread (datasets.FramePrefetcher)."""
    from .datasets import FramePrefetcher
    cfg = cfg if cfg is not None else TrainConfig()
    mapper = Mapper(dataset.intrinsics, cfg, device=device)
    reports = []
    n_frames = len(dataset) if cfg.max_frames is None else min(len(dataset), cfg.max_frames)
    for i, frame in enumerate(FramePrefetcher(dataset, n_frames)):
        try:
            mapper.process_frame(frame, dataset.classes)
        except Exception as exc:
            raise RuntimeError(f"failed on frame {i}: {exc}") from exc
        for _ in range(cfg.steps_per_frame):
            reports.append(mapper.train_step(mode=mode))
        if progress and (i % 20 == 0 or i == n_frames - 1):
            last = reports[-1]
            print(f"frame {i + 1}/{n_frames}  K={last.k_models}  total={last.total:.3f}  step_ms={last.ms:.1f}",
                  flush=True)
    return mapper, reports
