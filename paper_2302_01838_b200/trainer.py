"""Vectorised training step on the B200 (drop-in for vobj/trainer.py).

Reference: /root/reference/pkg/src/vobj/trainer.py.  `train_on_batch` keeps
the reference signature and semantics (trainer.py:480-506) but runs the whole
forward -> render -> loss -> backward -> Adam chain as one fused kernel plus
one Adam launch (csrc/vm_mlp.cu).  `Mapper.train_step` lives in mapper.py.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .models import (DEVICE, ModelArch, OptimState, StackedModelParams, _as_device, init_stacked,
                     vm_stack)
from .objects import AssociationConfig
from .render import LossWeights, SamplingConfig
from .rng import PURPOSE_BENCH, keyed_rng


@dataclass
class TrainConfig:
    """trainer.py:61-92 (same fields and defaults)."""

    seed: int = 0
    steps_per_frame: int = 10
    rays_per_object: int = 120
    rays_background: int = 1200
    sampling: SamplingConfig = field(default_factory=SamplingConfig)
    loss_weights: LossWeights = field(default_factory=LossWeights)
    association: AssociationConfig = field(default_factory=AssociationConfig)
    arch_object: ModelArch = field(default_factory=lambda: ModelArch(n_layers=4, hidden=32, n_freq=5))
    arch_background: ModelArch = field(default_factory=lambda: ModelArch(n_layers=4, hidden=128, n_freq=5))
    pe_scale_object: float = 10.0
    pe_scale_background: float = 15.0
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    train_background: bool = True
    max_frames: int | None = None
    mesh_resolution_object: int = 64
    mesh_resolution_scene: int = 256
    eval_samples_background: int = 48
    eval_samples_object: int = 48

    def __post_init__(self):
        for name in ("steps_per_frame", "rays_per_object", "rays_background"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be positive")

    @property
    def points_per_ray(self) -> int:
        return self.sampling.n_points


@dataclass
class RaySampleBatch:
    """trainer.py:162-173, device tensors with a leading model axis."""

    encoded: torch.Tensor        # [K, R, S, D] f32
    t: torch.Tensor              # [K, R, S] f32
    target_depth: torch.Tensor   # [K, R] f32
    target_colour: torch.Tensor  # [K, R, 3] f32
    target_mask: torch.Tensor    # [K, R] bool
    valid_depth: torch.Tensor    # [K, R] bool
    ray_ok: torch.Tensor         # [K, R] bool
    has_rays: bool = True

    @staticmethod
    def from_arrays(encoded, t, target_depth, target_colour, target_mask, valid_depth, ray_ok,
                    has_rays=True, device=DEVICE) -> "RaySampleBatch":
        f = lambda x: _as_device(x, device=device)
        b = lambda x: _as_device(x, dtype=torch.bool, device=device)
        return RaySampleBatch(f(encoded), f(t), f(target_depth), f(target_colour), b(target_mask),
                              b(valid_depth), b(ray_ok), bool(has_rays))

    def vm(self) -> _lib.VmBatch:
        k, r, s, d = self.encoded.shape
        out = _lib.VmBatch()
        out.n_models, out.n_rays, out.n_points, out.input_dim = k, r, s, d
        out.encoded = self.encoded.data_ptr()
        out.t = self.t.data_ptr()
        out.target_depth = self.target_depth.data_ptr()
        out.target_colour = self.target_colour.data_ptr()
        out.target_mask = self.target_mask.data_ptr()
        out.valid_depth = self.valid_depth.data_ptr()
        out.ray_ok = self.ray_ok.data_ptr()
        return out


@dataclass
class StepReport:
    """trainer.py:176-187."""

    step: int
    frame_id: int
    k_models: int
    losses: dict
    total: float
    ms: float

    @staticmethod
    def csv_header() -> str:
        return "step,frame,k,object_id,l_depth,l_colour,l_occ,total,ms"


class TrainWorkspace:
    """Device buffers one fused training call needs (reused across calls)."""

    def __init__(self):
        self.ws = None
        self.io = None       # int32: losses [K, 3] (f32 bits) then status [4 * stacks], contiguous
        self.losses = None
        self.status = None

    def ensure(self, nbytes: int, n_models: int, n_stacks: int, device) -> None:
        if self.ws is None or self.ws.numel() < nbytes:
            self.ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
        need = 3 * max(n_models, 1) + 4 * max(n_stacks, 2)
        if self.io is None or self.io.numel() < need:
            self.io = torch.zeros(2 * need, dtype=torch.int32, device=device)
        # status right behind this call's losses: one device->host copy reads both
        self.losses = self.io[:3 * max(n_models, 1)].view(torch.float32).view(max(n_models, 1), 3)
        self.status = self.io[3 * max(n_models, 1):3 * max(n_models, 1) + 4 * max(n_stacks, 2)]

    def results(self, n_models: int, n_stacks: int) -> torch.Tensor:
        """The contiguous int32 view [losses (3 n_models) | status (4 n_stacks)]."""
        return self.io[:3 * max(n_models, 1) + 4 * n_stacks]


_default_ws = TrainWorkspace()


def launch_train(stacks, weights: LossWeights, ws: TrainWorkspace | None = None, bump_version: bool = True):
    """Enqueue one fused step for [(params, state, batch), ...] (no host sync).

    Returns (losses [sum K, 3] device tensor, status device tensor).
    """
    ws = ws or _default_ws
    n = len(stacks)
    vs = (_lib.VmStack * n)()
    vb = (_lib.VmBatch * n)()
    keep = []
    for i, (p, s, b) in enumerate(stacks):
        vs[i] = vm_stack(p, s)
        vb[i] = b.vm()
        keep.append(b)
    lib = _lib.load()
    nbytes = lib.vm_train_workspace_bytes(vs, vb, n)
    if nbytes == 0:
        _lib.check(_lib.VM_ERR_SHAPE, "train_on_batch")
    kt = sum(p.count for p, _, _ in stacks)
    dev = stacks[0][0].arena.device
    ws.ensure(nbytes, kt, n, dev)
    _lib.check(lib.vm_train_step(vs, vb, n, weights.vm(), ws.losses.data_ptr(), ws.status.data_ptr(),
                                 ws.ws.data_ptr(), ws.ws.numel(), _lib.stream_ptr()), "train_on_batch")
    if bump_version:
        for p, _, _ in stacks:
            p.version += 1
    return ws.losses[:kt], ws.status[:4 * n]


def train_on_batch(params: StackedModelParams, state: OptimState, batch: RaySampleBatch,
                   weights: LossWeights, sync: bool = True):
    """trainer.py:480-506: fused forward/render/loss/backward/Adam for all K models.

    Returns per-model (L_depth, L_colour, L_occ) as float32 numpy arrays (the
    reference's return type); with ``sync=False`` device tensors are returned
    and the non-finite check is left to the caller.
    """
    if not isinstance(batch, RaySampleBatch):
        batch = RaySampleBatch.from_arrays(**batch)
    k = params.count
    if batch.encoded.shape[0] != k:
        raise ValueError(f"expected leading model axis of size {k}, got shape {tuple(batch.encoded.shape)}")
    if batch.encoded.shape[-1] != params.arch.input_dim:
        raise ValueError(f"encoding dim {batch.encoded.shape[-1]} does not match arch input dim "
                         f"{params.arch.input_dim}")
    losses, status = launch_train([(params, state, batch)], weights)
    if not sync:
        return losses[:, 0], losses[:, 1], losses[:, 2]
    host = torch.cat([losses.reshape(-1).view(torch.int32), status]).cpu()
    st = host[3 * k:].numpy()
    l = host[:3 * k].view(torch.float32).numpy().reshape(k, 3)
    if st[0] < k:
        raise FloatingPointError(f"non-finite gradient for model index {int(st[0])}")
    return l[:, 0].copy(), l[:, 1].copy(), l[:, 2].copy()


def train_on_batch_sequential(params: StackedModelParams, state: OptimState, batch: RaySampleBatch,
                              weights: LossWeights):
    """trainer.py:509-538: the same update one model at a time (baseline path)."""
    k = params.count
    ld = np.zeros(k, np.float64)
    lc = np.zeros(k, np.float64)
    lo = np.zeros(k, np.float64)
    for i in range(k):
        sub = RaySampleBatch(batch.encoded[i:i + 1], batch.t[i:i + 1], batch.target_depth[i:i + 1],
                             batch.target_colour[i:i + 1], batch.target_mask[i:i + 1],
                             batch.valid_depth[i:i + 1], batch.ray_ok[i:i + 1])
        d, c, o = train_on_batch(params.model_view(i), state.model_view(i), sub, weights)
        ld[i], lc[i], lo[i] = d[0], c[0], o[0]
    params.version += 1
    return ld, lc, lo


def _synthetic_batch(arch: ModelArch, k: int, rays: int, points: int, seed: int) -> RaySampleBatch:
    """trainer.py:594-606 (same keyed stream, uploaded to the device)."""
    rng = keyed_rng(seed, PURPOSE_BENCH, k, arch.hidden)
    t = np.sort(rng.random((k, rays, points)).astype(np.float32) * 4.0, axis=-1)
    return RaySampleBatch.from_arrays(
        encoded=(rng.standard_normal((k, rays, points, arch.input_dim)) * 0.7).astype(np.float32),
        t=t,
        target_depth=(rng.random((k, rays)) * 4.0).astype(np.float32),
        target_colour=rng.random((k, rays, 3)).astype(np.float32),
        target_mask=rng.random((k, rays)) < 0.6,
        valid_depth=np.ones((k, rays), dtype=bool),
        ray_ok=np.ones((k, rays), dtype=bool),
        has_rays=True,
    )


@dataclass
class BenchRow:
    mode: str
    k: int
    hidden: int
    ms: float


def benchmark(k_list, hidden_list, cfg: TrainConfig | None = None, timed_steps: int = 50,
              warmup_steps: int = 10, modes=("sequential", "vectorised")) -> list[BenchRow]:
    """trainer.py:609-642 with device timing (CUDA events around the loop)."""
    cfg = cfg if cfg is not None else TrainConfig()
    rows = []
    for hidden in hidden_list:
        arch = ModelArch(n_layers=cfg.arch_object.n_layers, hidden=hidden, n_freq=cfg.arch_object.n_freq)
        for k in k_list:
            batch = _synthetic_batch(arch, k, cfg.rays_per_object, cfg.points_per_ray, cfg.seed)
            for mode in modes:
                params, state = init_stacked(arch, k, cfg.seed, PURPOSE_BENCH, lr=cfg.lr, beta1=cfg.beta1,
                                             beta2=cfg.beta2, eps=cfg.eps)
                if mode == "vectorised":
                    step = lambda: train_on_batch(params, state, batch, cfg.loss_weights, sync=False)
                else:
                    step = lambda: train_on_batch_sequential(params, state, batch, cfg.loss_weights)
                for _ in range(warmup_steps):
                    step()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(timed_steps):
                    step()
                e1.record()
                torch.cuda.synchronize()
                rows.append(BenchRow(mode, k, hidden, e0.elapsed_time(e1) / timed_steps))
    return rows
