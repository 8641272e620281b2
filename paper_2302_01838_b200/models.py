"""Stacked per-object MLP fields on the B200 (drop-in for vobj/models.py).

Reference: /root/reference/pkg/src/vobj/models.py.  Same names, argument
meaning and errors; storage is a model-major device arena (one contiguous
block per model, see include/vmap_b200.h) and every compute call goes
through libvmap_b200.so.  `weights[l]` / `biases[l]` are strided torch views
of the arena with the reference's [capacity, fan_out, fan_in] shape
(models.py:69-71), so in-place edits through them reach the kernels.

Host-side setup (initialisation, growth, freezing) mirrors the reference
exactly: initial values are drawn with the same keyed numpy streams
(models.py:159-174) and uploaded once.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .rng import PURPOSE_INIT_OBJECT, keyed_rng

DEVICE = "cuda"


@dataclass(frozen=True)
class ModelArch:
    """models.py:19-55."""

    n_layers: int = 4
    hidden: int = 32
    n_freq: int = 5
    include_input: bool = True

    def __post_init__(self):
        if self.n_layers < 2:
            raise ValueError(f"need at least input and output layers, got n_layers={self.n_layers}")
        if self.hidden < 1:
            raise ValueError(f"hidden width must be positive, got {self.hidden}")
        if self.n_freq < 0:
            raise ValueError(f"n_freq must be non-negative, got {self.n_freq}")
        if self.input_dim == 0:
            raise ValueError("encoding is empty: n_freq=0 with include_input=False")

    @property
    def input_dim(self) -> int:
        return (3 if self.include_input else 0) + 6 * self.n_freq

    @property
    def output_dim(self) -> int:
        return 4

    def layer_dims(self) -> list[tuple[int, int]]:
        dims = [(self.hidden, self.input_dim)]
        dims += [(self.hidden, self.hidden)] * (self.n_layers - 2)
        dims.append((self.output_dim, self.hidden))
        return dims

    def vm_arch(self) -> _lib.VmArch:
        return _lib.VmArch(self.n_layers, self.hidden, self.input_dim, 0)


class _Arena:
    """Layout helper: views of a [capacity, block] arena in reference shapes."""

    def __init__(self, arch: ModelArch):
        self.arch = arch
        self.L = _lib.layout(arch.n_layers, arch.hidden, arch.input_dim)
        self.block = int(self.L.block)
        self.n_params = int(self.L.n_params)

    def weight_view(self, arena: torch.Tensor, l: int) -> torch.Tensor:
        cap = arena.shape[0]
        fo, fi, fip = self.L.fo[l], self.L.fi[l], self.L.fi_pad[l]
        return arena.as_strided((cap, fo, fi), (self.block, fip, 1), arena.storage_offset() + self.L.w_off[l])

    def bias_view(self, arena: torch.Tensor, l: int) -> torch.Tensor:
        cap = arena.shape[0]
        return arena.as_strided((cap, self.L.fo[l]), (self.block, 1), arena.storage_offset() + self.L.b_off[l])

    def pack(self, ws, bs) -> np.ndarray:
        """Host block(s) [n, block] from per-layer arrays [n, fo, fi] / [n, fo]."""
        n = ws[0].shape[0]
        out = np.zeros((n, self.block), np.float32)
        for l, (w, b) in enumerate(zip(ws, bs)):
            fo, fi, fip = self.L.fo[l], self.L.fi[l], self.L.fi_pad[l]
            o = self.L.w_off[l]
            blk = out[:, o:o + self.L.fo_pad[l] * fip].reshape(n, self.L.fo_pad[l], fip)
            blk[:, :fo, :fi] = np.asarray(w, np.float32)
            out[:, self.L.b_off[l]:self.L.b_off[l] + fo] = np.asarray(b, np.float32)
        return out


@dataclass(eq=False)
class StackedModelParams:
    """Weights of up to ``capacity`` models, ``count`` live (models.py:58-98).

    ``arena`` is the device storage [capacity, block]; ``weights``/``biases``
    are views into it.  ``frozen`` stays a host bool array (it is read by the
    host-side batch assembly, trainer.py:336) and is mirrored to the device
    before each kernel call.
    """

    arch: ModelArch
    count: int
    arena: torch.Tensor
    frozen: np.ndarray
    version: int = 0
    _layout: _Arena = field(default=None, repr=False)
    _frozen_dev: torch.Tensor = field(default=None, repr=False)
    _frozen_seen: np.ndarray = field(default=None, repr=False)

    def __post_init__(self):
        if self._layout is None:
            self._layout = _Arena(self.arch)

    @property
    def capacity(self) -> int:
        return self.frozen.shape[0]

    @property
    def dtype(self):
        return np.dtype(np.float32)

    @property
    def block(self) -> int:
        return self._layout.block

    @property
    def weights(self) -> list[torch.Tensor]:
        return [self._layout.weight_view(self.arena, l) for l in range(self.arch.n_layers)]

    @property
    def biases(self) -> list[torch.Tensor]:
        return [self._layout.bias_view(self.arena, l) for l in range(self.arch.n_layers)]

    def frozen_device(self) -> torch.Tensor:
        """uint8 [capacity] device mirror of ``frozen`` (re-uploaded on change)."""
        if self._frozen_dev is None or self._frozen_dev.numel() != self.capacity:
            self._frozen_seen = self.frozen.copy()
            self._frozen_dev = torch.from_numpy(self.frozen.astype(np.uint8)).to(self.arena.device)
        elif not np.array_equal(self._frozen_seen, self.frozen):
            # in place: captured step graphs keep reading the same buffer
            self._frozen_seen = self.frozen.copy()
            self._frozen_dev.copy_(torch.from_numpy(self.frozen.astype(np.uint8)))
        return self._frozen_dev

    def model_view(self, index: int) -> "StackedModelParams":
        """Single-model window sharing memory with this stack (models.py:82-98)."""
        if not (0 <= index < self.count):
            raise IndexError(f"model index {index} out of range for count {self.count}")
        return StackedModelParams(self.arch, 1, self.arena[index:index + 1],
                                  self.frozen[index:index + 1], self.version, self._layout)


@dataclass(eq=False)
class OptimState:
    """Adam state mirroring a parameter stack (models.py:101-126)."""

    m_arena: torch.Tensor
    v_arena: torch.Tensor
    step: torch.Tensor  # [capacity] int64 on device
    arch: ModelArch
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    _layout: _Arena = field(default=None, repr=False)
    _corr: tuple = field(default=None, repr=False)

    def __post_init__(self):
        if self._layout is None:
            self._layout = _Arena(self.arch)

    m_weights = property(lambda s: [s._layout.weight_view(s.m_arena, l) for l in range(s.arch.n_layers)])
    v_weights = property(lambda s: [s._layout.weight_view(s.v_arena, l) for l in range(s.arch.n_layers)])
    m_biases = property(lambda s: [s._layout.bias_view(s.m_arena, l) for l in range(s.arch.n_layers)])
    v_biases = property(lambda s: [s._layout.bias_view(s.v_arena, l) for l in range(s.arch.n_layers)])

    def model_view(self, index: int) -> "OptimState":
        return OptimState(self.m_arena[index:index + 1], self.v_arena[index:index + 1],
                          self.step[index:index + 1], self.arch, self.lr, self.beta1, self.beta2,
                          self.eps, self._layout, self._corr)

    def corrections(self, device) -> tuple[torch.Tensor, torch.Tensor, int]:
        """f32(1 - beta**t) for t = 1..n computed in f64 like models.py:434-436.

        The table runs until both corrections round to 1.0f (t = 165 / 17,330
        for the default betas), capped at 2**18 entries; past the table the
        kernels evaluate the same f64 expression with the device pow().
        """
        key = (self.beta1, self.beta2)
        if self._corr is None or self._corr[0] != key:
            n = corrections_table_len(self.beta1, self.beta2)
            t = np.arange(1, n + 1, dtype=np.float64)
            c1 = (1.0 - self.beta1 ** t).astype(np.float32)
            c2 = (1.0 - self.beta2 ** t).astype(np.float32)
            self._corr = (key, torch.from_numpy(c1).to(device), torch.from_numpy(c2).to(device), n)
        return self._corr[1], self._corr[2], self._corr[3]


def corrections_table_len(beta1: float, beta2: float, cap: int = 1 << 18) -> int:
    """Smallest power-of-two table length after which f32(1 - beta**t) == 1.0f
    for both betas (models.py:434-436 arithmetic), at most `cap`."""
    n = 1024
    while n < cap:
        t = np.float64(n)
        if np.float32(1.0 - beta1 ** t) == 1.0 and np.float32(1.0 - beta2 ** t) == 1.0:
            break
        n *= 2
    return min(n, cap)


@dataclass
class FieldOutput:
    occupancy: torch.Tensor  # [K, ...]
    colour: torch.Tensor     # [K, ..., 3]


@dataclass
class Gradients:
    d_weights: list
    d_biases: list
    arena: torch.Tensor | None = None  # [K, block] when produced by backward()


@dataclass
class ActivationCache:
    """What backward() needs: the encoded input (activations are recomputed on
    chip by the fused kernel) plus the outputs for inspection."""

    version: int
    lead_shape: tuple
    encoded: torch.Tensor
    occupancy: torch.Tensor
    colour: torch.Tensor


# ------------------------------------------------------------------ setup


def _init_model_arrays(arch: ModelArch, seed: int, model_index: int, stream: int):
    """models.py:159-174 (same keyed numpy stream -> identical init)."""
    rng = keyed_rng(seed, stream, model_index)
    ws, bs = [], []
    for fan_out, fan_in in arch.layer_dims():
        bound = 1.0 / np.sqrt(fan_in)
        ws.append(rng.uniform(-bound, bound, size=(fan_out, fan_in)).astype(np.float32))
        bs.append(rng.uniform(-bound, bound, size=fan_out).astype(np.float32))
    return ws, bs


def _capacity_for(count: int) -> int:
    return max(1, int(2 ** np.ceil(np.log2(max(count, 1)))))


def init_stacked(arch: ModelArch, count: int, seed: int, stream: int = PURPOSE_INIT_OBJECT,
                 dtype=np.float32, lr: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999,
                 eps: float = 1e-8, device=DEVICE) -> tuple[StackedModelParams, OptimState]:
    """models.py:199-219."""
    if count < 0:
        raise ValueError(f"count must be non-negative, got {count}")
    if np.dtype(dtype) != np.float32:
        raise NotImplementedError("the B200 kernels train float32 stacks only")
    lay = _Arena(arch)
    cap = _capacity_for(count)
    host = np.zeros((cap, lay.block), np.float32)
    for i in range(count):
        ws, bs = _init_model_arrays(arch, seed, i, stream)
        host[i] = lay.pack([w[None] for w in ws], [b[None] for b in bs])[0]
    arena = torch.from_numpy(host).to(device)
    params = StackedModelParams(arch, count, arena, np.zeros(cap, bool), 0, lay)
    state = OptimState(torch.zeros_like(arena), torch.zeros_like(arena),
                       torch.zeros(cap, dtype=torch.int64, device=device), arch, lr, beta1, beta2, eps, lay)
    return params, state


def _grow(params: StackedModelParams, state: OptimState, min_capacity: int) -> None:
    """models.py:229-250: next power of two, live blocks preserved."""
    new_cap = _capacity_for(min_capacity)
    if new_cap <= params.capacity:
        return
    k = params.count

    def grow(t):
        out = torch.zeros((new_cap,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        out[:k] = t[:k]
        return out

    params.arena = grow(params.arena)
    state.m_arena = grow(state.m_arena)
    state.v_arena = grow(state.v_arena)
    state.step = grow(state.step)
    frozen = np.zeros(new_cap, bool)
    frozen[:k] = params.frozen[:k]
    params.frozen = frozen


def append_model(params: StackedModelParams, state: OptimState, seed: int,
                 stream: int = PURPOSE_INIT_OBJECT, init_index: int | None = None) -> int:
    """models.py:253-277.  ``init_index`` (default: the new slot) is the model
    index the init stream is keyed by; object-sharded ranks pass the object's
    global append index so their weights equal a single-stack run's."""
    idx = params.count
    if idx + 1 > params.capacity:
        _grow(params, state, idx + 1)
    ws, bs = _init_model_arrays(params.arch, seed, idx if init_index is None else init_index, stream)
    blk = params._layout.pack([w[None] for w in ws], [b[None] for b in bs])[0]
    params.arena[idx] = torch.from_numpy(blk).to(params.arena.device)
    state.m_arena[idx] = 0
    state.v_arena[idx] = 0
    state.step[idx] = 0
    params.frozen[idx] = False
    params.count = idx + 1
    params.version += 1
    return idx


def set_frozen(params: StackedModelParams, index: int, frozen: bool) -> None:
    """models.py:280-283."""
    if not (0 <= index < params.count):
        raise IndexError(f"model index {index} out of range for count {params.count}")
    params.frozen[index] = frozen


# ------------------------------------------------------------------ C structs


def vm_stack(params: StackedModelParams, state: OptimState | None = None) -> _lib.VmStack:
    """VmStack describing a (params, state) pair for the C ABI."""
    s = _lib.VmStack()
    s.arch = params.arch.vm_arch()
    s.count = params.count
    s.capacity = params.capacity
    s.params = params.arena.data_ptr()
    s.frozen = params.frozen_device().data_ptr()
    if state is not None:
        c1, c2, n = state.corrections(params.arena.device)
        s.m = state.m_arena.data_ptr()
        s.v = state.v_arena.data_ptr()
        s.step = state.step.data_ptr()
        s.corr1, s.corr2, s.corr_len = c1.data_ptr(), c2.data_ptr(), n
        f32 = np.float32
        s.beta1f = float(f32(state.beta1))
        s.omb1 = float(f32(1.0 - state.beta1))
        s.beta2f = float(f32(state.beta2))
        s.omb2 = float(f32(1.0 - state.beta2))
        s.eps = float(f32(state.eps))
        s.lr = float(f32(state.lr))
        s.beta1, s.beta2 = float(state.beta1), float(state.beta2)
    return s


def _as_device(x, dtype=torch.float32, device=DEVICE) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x))).to(device=device, dtype=dtype)


# ------------------------------------------------------------------ compute


def positional_encode(points, center, half_extent, arch: ModelArch, scale: float):
    """models.py:286-308 (float64 like the reference; torch on the input's device).

    The training hot path never calls this: the CUDA sampler encodes samples
    in-kernel (vm_sample).  It is kept for API compatibility.
    """
    pts = points if isinstance(points, torch.Tensor) else torch.as_tensor(np.asarray(points))
    center = torch.as_tensor(np.asarray(center, dtype=np.float64), dtype=pts.dtype, device=pts.device)
    half = torch.as_tensor(np.asarray(half_extent, dtype=np.float64), dtype=pts.dtype, device=pts.device)
    if bool((half <= 0).any()):
        raise ValueError(f"half_extent must be positive, got {half}")
    if scale <= 0:
        raise ValueError(f"scale must be positive, got {scale}")
    p = (pts - center) / half
    parts = [p] if arch.include_input else []
    for i in range(arch.n_freq):
        arg = (np.pi * (2.0 ** i) / scale) * p
        parts += [torch.sin(arg), torch.cos(arg)]
    return torch.cat(parts, dim=-1)


def forward(params: StackedModelParams, encoded) -> tuple[FieldOutput, ActivationCache]:
    """models.py:311-355 on the device (vm_forward)."""
    k = params.count
    if encoded.ndim < 2 or encoded.shape[0] != k:
        raise ValueError(f"expected leading model axis of size {k}, got shape {tuple(encoded.shape)}")
    if encoded.shape[-1] != params.arch.input_dim:
        raise ValueError(
            f"encoding dim {encoded.shape[-1]} does not match arch input dim {params.arch.input_dim}")
    lead = tuple(encoded.shape[1:-1])
    x = _as_device(encoded, device=params.arena.device).reshape(k, -1, params.arch.input_dim)
    n = x.shape[1]
    occ = torch.empty((k, n), dtype=torch.float32, device=x.device)
    col = torch.empty((k, n, 3), dtype=torch.float32, device=x.device)
    st = vm_stack(params)
    _lib.check(_lib.load().vm_forward(C.byref(st), x.data_ptr(), n, occ.data_ptr(), col.data_ptr(),
                                      _lib.stream_ptr()), "forward")
    cache = ActivationCache(params.version, lead, x, occ, col)
    return FieldOutput(occ.reshape((k,) + lead), col.reshape((k,) + lead + (3,))), cache


def backward(params: StackedModelParams, cache: ActivationCache, grad_occupancy, grad_colour) -> Gradients:
    """models.py:358-398 (vm_backward recomputes activations on chip)."""
    if cache.version != params.version:
        raise ValueError(
            f"stale activation cache (cache version {cache.version}, params version {params.version})")
    k, n = params.count, cache.encoded.shape[1]
    dev = params.arena.device
    go = _as_device(grad_occupancy, device=dev).reshape(k, n)
    gc = _as_device(grad_colour, device=dev).reshape(k, n, 3)
    grads = torch.empty((max(k, 1), params.block), dtype=torch.float32, device=dev)[:k]
    st = vm_stack(params)
    _lib.check(_lib.load().vm_backward(C.byref(st), cache.encoded.data_ptr(), n, go.data_ptr(),
                                       gc.data_ptr(), grads.data_ptr(), _lib.stream_ptr()), "backward")
    lay = params._layout
    return Gradients([lay.weight_view(grads, l) for l in range(params.arch.n_layers)],
                     [lay.bias_view(grads, l) for l in range(params.arch.n_layers)], grads)


def _grads_arena(params: StackedModelParams, grads: Gradients) -> torch.Tensor:
    k = params.count
    if grads.arena is not None and grads.arena.shape[0] == k:
        return grads.arena
    lay = params._layout
    dev = params.arena.device
    out = torch.zeros((k, lay.block), dtype=torch.float32, device=dev)
    for l in range(params.arch.n_layers):
        lay.weight_view(out, l).copy_(_as_device(grads.d_weights[l], device=dev).reshape(k, *lay.weight_view(out, l).shape[1:]))
        lay.bias_view(out, l).copy_(_as_device(grads.d_biases[l], device=dev).reshape(k, -1))
    return out


def adam_step(params: StackedModelParams, state: OptimState, grads: Gradients, update_mask=None) -> None:
    """models.py:401-467: one masked Adam update in place (vm_adam)."""
    k = params.count
    dev = params.arena.device
    mask = None
    if update_mask is not None:
        mask = _as_device(np.asarray(update_mask.cpu() if isinstance(update_mask, torch.Tensor) else update_mask,
                                     dtype=bool).reshape(k), dtype=torch.uint8, device=dev)
    g = _grads_arena(params, grads)
    status = torch.empty(1, dtype=torch.int32, device=dev)
    st = vm_stack(params, state)
    _lib.check(_lib.load().vm_adam(C.byref(st), g.data_ptr(), _lib.ptr(mask), status.data_ptr(),
                                   _lib.stream_ptr()), "adam_step")
    bad = int(status.item())
    params.version += 1
    if bad >= 0:
        raise FloatingPointError(f"non-finite gradient for model index {bad}")
