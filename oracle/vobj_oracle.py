"""CPU oracle for vMAP's vectorised object-mapping step -- TEST INFRASTRUCTURE ONLY.

This module is a from-scratch numpy restatement of the reference `vobj`
package's hot path (`/root/reference/pkg/src/vobj`).  It exists so that the
CUDA implementation in `paper_2302_01838_b200` can be checked on identical
seeded inputs.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it; the
product path never does (it fails loudly without its CUDA library).

Parity pinning: every function here is checked against golden vectors that
`tests/golden/make_golden.py` produced by running the real reference in the
build container (`tests/test_oracle_golden.py`).  Integer/RNG outputs and all
f64 geometry are compared bit-exactly; BLAS-backed f32 matmul results are
compared bit-exactly on the host that produced the goldens and to 1e-6
elsewhere (OpenBLAS kernels differ per CPU).

Each function cites the reference `file:line` whose arithmetic it restates.
Operation order is deliberately the same as the reference's numpy expression
order, because f32 results depend on it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import expit

# Purpose codes, rng.py:15-21 (part of the replay contract).
INIT_OBJECT, INIT_BACKGROUND, PIXELS, SAMPLES, BENCH = 1, 2, 3, 4, 5


def keyed_rng(seed: int, purpose: int, *extra: int) -> np.random.Generator:
    """rng.py:24-34 -- numpy Generator(PCG64(SeedSequence(key)))."""
    key = (seed, purpose) + tuple(extra)
    if any(k < 0 for k in key):
        raise ValueError(f"rng key parts must be non-negative, got {key}")
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(key)))


# --------------------------------------------------------------------------
# model stacks (models.py)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Arch:
    """models.py:19-55."""
    n_layers: int = 4
    hidden: int = 32
    n_freq: int = 5
    include_input: bool = True

    @property
    def input_dim(self) -> int:
        return 6 * self.n_freq + (3 if self.include_input else 0)

    def dims(self) -> list[tuple[int, int]]:
        """(fan_out, fan_in) first to last -- models.py:50-55."""
        h = self.hidden
        return [(h, self.input_dim)] + [(h, h)] * (self.n_layers - 2) + [(4, h)]


@dataclass
class Stack:
    """Params + Adam state of K models (models.py:58-126)."""
    arch: Arch
    count: int
    W: list
    b: list
    frozen: np.ndarray
    mW: list
    vW: list
    mb: list
    vb: list
    step: np.ndarray
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    def copy(self) -> "Stack":
        c = lambda xs: [x.copy() for x in xs]
        return Stack(self.arch, self.count, c(self.W), c(self.b), self.frozen.copy(),
                     c(self.mW), c(self.vW), c(self.mb), c(self.vb), self.step.copy(),
                     self.lr, self.beta1, self.beta2, self.eps)


def init_model_arrays(arch: Arch, seed: int, model_index: int, stream: int, dtype=np.float32):
    """models.py:159-174: U(-1/sqrt(fi), 1/sqrt(fi)) weights then bias, per layer."""
    g = keyed_rng(seed, stream, model_index)
    ws, bs = [], []
    for fo, fi in arch.dims():
        lim = 1.0 / np.sqrt(fi)
        ws.append(g.uniform(-lim, lim, size=(fo, fi)).astype(dtype))
        bs.append(g.uniform(-lim, lim, size=fo).astype(dtype))
    return ws, bs


def new_stack(arch: Arch, count: int, seed: int, stream: int = INIT_OBJECT, dtype=np.float32,
              lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8) -> Stack:
    """init_stacked, models.py:199-219 (capacity = next power of two)."""
    cap = max(1, int(2 ** np.ceil(np.log2(max(count, 1)))))
    W = [np.zeros((cap, fo, fi), dtype) for fo, fi in arch.dims()]
    b = [np.zeros((cap, fo), dtype) for fo, _ in arch.dims()]
    st = Stack(arch, 0, W, b, np.zeros(cap, bool),
               [np.zeros_like(x) for x in W], [np.zeros_like(x) for x in W],
               [np.zeros_like(x) for x in b], [np.zeros_like(x) for x in b],
               np.zeros(cap, np.int64), lr, beta1, beta2, eps)
    for i in range(count):
        ws, bs = init_model_arrays(arch, seed, i, stream, dtype)
        for l in range(len(ws)):
            st.W[l][i] = ws[l]
            st.b[l][i] = bs[l]
    st.count = count
    return st


def append(st: Stack, seed: int, stream: int = INIT_OBJECT) -> int:
    """append_model, models.py:229-277 (grow to next pow2, init slot `count`)."""
    k = st.count
    if k + 1 > len(st.frozen):
        cap = max(1, int(2 ** np.ceil(np.log2(k + 1))))
        def grow(a):
            out = np.zeros((cap,) + a.shape[1:], a.dtype)
            out[:k] = a[:k]
            return out
        for name in ("W", "b", "mW", "vW", "mb", "vb"):
            setattr(st, name, [grow(a) for a in getattr(st, name)])
        st.frozen = grow(st.frozen)
        st.step = grow(st.step)
    ws, bs = init_model_arrays(st.arch, seed, k, stream, st.W[0].dtype)
    for l in range(len(ws)):
        st.W[l][k], st.b[l][k] = ws[l], bs[l]
        for arr in (st.mW, st.vW):
            arr[l][k] = 0
        for arr in (st.mb, st.vb):
            arr[l][k] = 0
    st.step[k] = 0
    st.frozen[k] = False
    st.count = k + 1
    return k


def positional_encode(points, center, half, arch: Arch, scale: float) -> np.ndarray:
    """models.py:286-308: p=(x-c)/h ; [p, sin(pi 2^i p/s), cos(...)] per band."""
    x = np.asarray(points)
    c = np.asarray(center, dtype=x.dtype)
    h = np.asarray(half, dtype=x.dtype)
    if np.any(h <= 0):
        raise ValueError(f"half_extent must be positive, got {h}")
    if scale <= 0:
        raise ValueError(f"scale must be positive, got {scale}")
    p = (x - c) / h
    feats = [p] if arch.include_input else []
    for band in range(arch.n_freq):
        a = (np.pi * (2.0 ** band) / scale) * p
        feats += [np.sin(a), np.cos(a)]
    return np.concatenate(feats, axis=-1)


def mlp_forward(st: Stack, enc: np.ndarray):
    """models.py:311-355.  Returns (occ [K,N], col [K,N,3], inputs, masks)."""
    k = st.count
    x = np.ascontiguousarray(enc.reshape(k, -1, enc.shape[-1]))
    inputs, masks = [], []
    last = len(st.W) - 1
    for l in range(last + 1):
        inputs.append(x)
        z = np.matmul(x, st.W[l][:k].transpose(0, 2, 1))
        z += st.b[l][:k][:, None, :]
        if l == last:
            x = z
        else:
            masks.append(z > 0)
            x = np.maximum(z, 0.0, out=z)
    return expit(x[..., 0]), expit(x[..., 1:]), inputs, masks


def mlp_backward(st: Stack, occ, col, inputs, masks, g_occ, g_col):
    """models.py:358-398: sigmoid heads, then per layer dW=dz^T x, db=1^T dz, dx=dz W."""
    k, n = occ.shape
    dz = np.empty((k, n, 4), dtype=occ.dtype)
    dz[..., 0] = np.asarray(g_occ).reshape(k, n) * occ * (1.0 - occ)
    dz[..., 1:] = np.asarray(g_col).reshape(k, n, 3) * col * (1.0 - col)
    ones = np.ones((1, 1, n), dtype=dz.dtype)
    dW = [None] * len(st.W)
    db = [None] * len(st.W)
    for l in reversed(range(len(st.W))):
        dW[l] = np.matmul(dz.transpose(0, 2, 1), inputs[l])
        db[l] = np.matmul(ones, dz)[:, 0, :]
        if l:
            nxt = np.matmul(dz, st.W[l][:k])
            nxt *= masks[l - 1]
            dz = nxt
    return dW, db


def adam_update(st: Stack, dW, db, update_mask=None) -> None:
    """models.py:401-467, op-for-op (f32 with f64 bias corrections)."""
    k = st.count
    act = ~st.frozen[:k]
    if update_mask is not None:
        act = act & np.asarray(update_mask, bool).reshape(k)
    sel = np.flatnonzero(act)
    if sel.size == 0:
        return
    bad = np.zeros(k, bool)
    for gw, gb in zip(dW, db):
        bad |= ~np.isfinite(gw).all(axis=(1, 2)) | ~np.isfinite(gb).all(axis=1)
    bad &= act
    if bad.any():
        raise FloatingPointError(f"non-finite gradient for model index {int(np.flatnonzero(bad)[0])}")
    dt = st.W[0].dtype
    b1, b2 = st.beta1, st.beta2
    tt = (st.step[sel] + 1).astype(np.float64)
    c1 = (1.0 - b1 ** tt).astype(dt)
    c2 = (1.0 - b2 ** tt).astype(dt)
    lr = dt.type(st.lr)
    every = sel.size == k

    def one(p, m_all, v_all, g_all, shape):
        g = g_all if every else g_all[sel]
        m = m_all[:k] if every else m_all[sel]
        v = v_all[:k] if every else v_all[sel]
        m *= b1
        m += (1.0 - b1) * g
        g2 = np.square(g)
        g2 *= 1.0 - b2
        v *= b2
        v += g2
        if not every:
            m_all[sel] = m
            v_all[sel] = v
        den = np.sqrt(v / c2.reshape(shape))
        den += st.eps
        upd = m / c1.reshape(shape)
        upd /= den
        upd *= lr
        if every:
            p[:k] -= upd
        else:
            p[sel] -= upd

    for l in range(len(st.W)):
        one(st.W[l], st.mW[l], st.vW[l], dW[l], (-1, 1, 1))
        one(st.b[l], st.mb[l], st.vb[l], db[l], (-1, 1))
    st.step[sel] += 1


# --------------------------------------------------------------------------
# rendering and losses (render.py)
# --------------------------------------------------------------------------

def render_forward(occ, col, t):
    """render.py:230-246 -> (opacity, depth, colour, weights, trans)."""
    occ = np.asarray(occ)
    om = 1.0 - occ
    T = np.empty_like(om)
    T[..., 0] = 1.0
    np.cumprod(om[..., :-1], axis=-1, out=T[..., 1:])
    w = occ * T
    return w.sum(axis=-1), (w * t).sum(axis=-1), (w[..., None] * col).sum(axis=-2), w, T


def render_backward(occ, col, t, w, T, dO, dD, dC):
    """render.py:249-281."""
    g = dO[..., None] + dD[..., None] * t + (dC[..., None, :] * col).sum(axis=-1)
    d_col = w[..., None] * dC[..., None, :]
    gw = g * w
    rev = np.flip(np.cumsum(np.flip(gw, axis=-1), axis=-1), axis=-1)
    d_occ = g * T - (rev - gw) / np.maximum(1.0 - occ, 1e-7)
    return d_occ, d_col


def _loss_masks(mask, valid, ok, dtype):
    mask = np.asarray(mask, bool)
    m_ok = mask & ok
    return (mask.astype(dtype), (m_ok & valid).astype(dtype), m_ok.astype(dtype),
            np.asarray(ok, bool).astype(dtype))


def losses(O, D, C, tgt_d, tgt_c, mask, valid, ok, w_colour=5.0, w_occ=10.0):
    """render.py:284-309 -> (L_depth, L_colour, L_occ, total) summed over rays."""
    m_ind, wd, wc, wo = _loss_masks(mask, valid, ok, D.dtype)
    ld = (wd * np.abs(D - tgt_d)).sum(axis=-1)
    lc = (wc * np.abs(C - tgt_c).sum(axis=-1)).sum(axis=-1)
    lo = (wo * np.abs(O - m_ind)).sum(axis=-1)
    return ld, lc, lo, ld + w_colour * lc + w_occ * lo


def loss_grads(O, D, C, tgt_d, tgt_c, mask, valid, ok, w_colour=5.0, w_occ=10.0):
    """render.py:312-333 -> (dO, dD, dC); sign(0) = 0."""
    m_ind, wd, wc, wo = _loss_masks(mask, valid, ok, D.dtype)
    return (w_occ * wo * np.sign(O - m_ind), wd * np.sign(D - tgt_d),
            (w_colour * wc)[..., None] * np.sign(C - tgt_c))


def train_on_batch(st: Stack, batch: dict, w_colour=5.0, w_occ=10.0):
    """trainer.py:480-506: forward -> render -> losses -> grads -> backward -> Adam."""
    occ, col, xs, ms = mlp_forward(st, batch["encoded"])
    k = st.count
    lead = batch["encoded"].shape[1:-1]
    occ_r, col_r = occ.reshape((k,) + lead), col.reshape((k,) + lead + (3,))
    O, D, C, w, T = render_forward(occ_r, col_r, batch["t"])
    args = (batch["target_depth"], batch["target_colour"], batch["target_mask"],
            batch["valid_depth"], batch["ray_ok"], w_colour, w_occ)
    ld, lc, lo, _ = losses(O, D, C, *args)
    dO, dD, dC = loss_grads(O, D, C, *args)
    d_occ, d_col = render_backward(occ_r, col_r, batch["t"], w, T, dO, dD, dC)
    dW, db = mlp_backward(st, occ, col, xs, ms, d_occ, d_col)
    adam_update(st, dW, db, update_mask=batch["ray_ok"].any(axis=-1))
    return ld, lc, lo


def synthetic_batch(arch: Arch, k: int, rays: int, points: int, seed: int) -> dict:
    """trainer.py:594-606 (the reference's own benchmark input)."""
    g = keyed_rng(seed, BENCH, k, arch.hidden)
    t = np.sort(g.random((k, rays, points)).astype(np.float32) * 4.0, axis=-1)
    return dict(
        encoded=(g.standard_normal((k, rays, points, arch.input_dim)) * 0.7).astype(np.float32),
        t=t,
        target_depth=(g.random((k, rays)) * 4.0).astype(np.float32),
        target_colour=g.random((k, rays, 3)).astype(np.float32),
        target_mask=g.random((k, rays)) < 0.6,
        valid_depth=np.ones((k, rays), bool),
        ray_ok=np.ones((k, rays), bool),
    )


# --------------------------------------------------------------------------
# rays and depth-guided sampling (render.py, objects.py, trainer.py)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Sampling:
    """render.py:38-58 defaults."""
    t_near: float = 0.0
    t_far: float = 8.0
    n_stratified: int = 5
    n_surface: int = 5
    surface_std: float = 0.03


def ray_box(origins, dirs, bmin, bmax):
    """render.py:111-139 slab test -> (t_entry, t_exit, hit)."""
    o = np.atleast_2d(np.asarray(origins, np.float64))
    d = np.atleast_2d(np.asarray(dirs, np.float64))
    with np.errstate(divide="ignore", invalid="ignore"):
        r = 1.0 / d
        ta = (bmin - o) * r
        tb = (bmax - o) * r
    lo, hi = np.minimum(ta, tb), np.maximum(ta, tb)
    flat = d == 0
    if flat.any():
        inside = (o >= bmin) & (o <= bmax)
        lo = np.where(flat, np.where(inside, -np.inf, np.inf), lo)
        hi = np.where(flat, np.where(inside, np.inf, -np.inf), hi)
    t_in, t_out = lo.max(axis=-1), hi.min(axis=-1)
    entry = np.maximum(t_in, 0.0)
    return entry, t_out, (t_out >= entry) & (t_out >= 0.0)


def _bins(u, lo, hi):
    """render.py:142-146."""
    n = u.shape[-1]
    return lo[..., None] + ((np.arange(n) + u) / n) * (hi - lo)[..., None]


def sample_along_rays(g, surf, valid, in_mask, far, cfg: Sampling, near=None):
    """render.py:149-227.  Draw order is fixed: u_strat, z_surf, u_fallback."""
    surf = np.asarray(surf, np.float64)
    r = surf.shape[0]
    u_s = g.random((r, cfg.n_stratified))
    z = g.standard_normal((r, cfg.n_surface))
    u_f = g.random((r, cfg.n_stratified + cfg.n_surface))
    lo = np.full(r, cfg.t_near) if near is None else np.asarray(near, np.float64)
    far = np.maximum(np.asarray(far, np.float64), lo)
    valid = np.asarray(valid, bool)
    in_mask = np.asarray(in_mask, bool)
    has_d = valid & (surf > lo)
    blocked = valid & ~has_d
    over = in_mask & has_d & (surf > far + 3.0 * cfg.surface_std)
    guided = in_mask & has_d & ~over
    band_hi = np.minimum(surf + 3.0 * cfg.surface_std, far)
    tg = np.concatenate([_bins(u_s, lo, surf),
                         np.clip(surf[:, None] + cfg.surface_std * z, lo[:, None], band_hi[:, None])],
                        axis=1)
    up = np.where(in_mask, far, np.where(has_d, np.minimum(surf, far), far))
    tf = _bins(u_f, lo, np.maximum(up, lo))
    t = np.where(guided[:, None], tg, tf)
    ok = (guided | (up > lo)) & ~blocked & ~over
    t.sort(axis=1)
    return t, ok


def sample_training_pixels(keyframes, object_id: int, seed: int, step: int, n_rays: int):
    """objects.py:323-352 -> (kf_idx, u, v, in_mask)."""
    if not keyframes:
        raise ValueError(f"object {object_id} has no keyframes to sample from")
    g = keyed_rng(seed, PIXELS, object_id, step)
    kf = g.integers(0, len(keyframes), size=n_rays)
    uv = g.random((n_rays, 2))
    u = np.empty(n_rays, np.int64)
    v = np.empty(n_rays, np.int64)
    hit = np.empty(n_rays, bool)
    for k in np.unique(kf):
        s = kf == k
        u0, v0, u1, v1 = keyframes[int(k)].bbox
        uu = np.minimum(u0 + np.floor(uv[s, 0] * (u1 - u0)).astype(np.int64), u1 - 1)
        vv = np.minimum(v0 + np.floor(uv[s, 1] * (v1 - v0)).astype(np.int64), v1 - 1)
        u[s], v[s] = uu, vv
        hit[s] = keyframes[int(k)].mask[vv - v0, uu - u0]
    return kf, u, v, hit


def zero_batch(rays: int, points: int, input_dim: int) -> dict:
    """trainer.py:190-200."""
    z = lambda *s: np.zeros(s, np.float32)
    return dict(encoded=z(rays, points, input_dim), t=z(rays, points), target_depth=z(rays),
                target_colour=z(rays, 3), target_mask=np.zeros(rays, bool),
                valid_depth=np.zeros(rays, bool), ray_ok=np.zeros(rays, bool))


def assemble_batch(inst, intr, arch: Arch, n_rays: int, step: int, seed: int,
                   cfg: Sampling = Sampling(), bound_pad: float = 0.10, with_aux: bool = False):
    """trainer.py:269-318 for one instance (object or background).

    ``inst`` needs object_id, keyframes (bbox/mask/rgb/depth/pose), aabb
    (min/max f64), pe_scale and active.  ``intr`` needs fx, fy, cx, cy, width,
    height.  With ``with_aux`` the pixel draws and f64 rays are returned too.
    """
    pts_per_ray = cfg.n_stratified + cfg.n_surface
    if not inst.keyframes or not getattr(inst, "active", True):
        out = zero_batch(n_rays, pts_per_ray, arch.input_dim)
        return (out, None) if with_aux else out
    kf, u, v, in_mask = sample_training_pixels(inst.keyframes, inst.object_id, seed, step, n_rays)
    rgb = np.empty((n_rays, 3), np.float64)
    z = np.empty(n_rays, np.float64)
    pose = np.empty((n_rays, 3, 4), np.float64)
    for k in np.unique(kf):
        frame = inst.keyframes[int(k)]
        s = kf == k
        du, dv = u[s] - frame.bbox[0], v[s] - frame.bbox[1]
        rgb[s] = frame.rgb[dv, du]
        z[s] = frame.depth[dv, du]
        pose[s] = frame.pose[:3, :]
    # camera_dirs, render.py:76-86
    px = np.stack([u, v], axis=1).astype(np.float64)
    if (np.any(px[:, 0] < 0) or np.any(px[:, 0] >= intr.width) or np.any(px[:, 1] < 0)
            or np.any(px[:, 1] >= intr.height)):
        raise ValueError("pixel coordinates outside the image")
    dc = np.empty((n_rays, 3))
    dc[:, 0] = (px[:, 0] - intr.cx) / intr.fx
    dc[:, 1] = (px[:, 1] - intr.cy) / intr.fy
    dc[:, 2] = 1.0
    to_t = np.linalg.norm(dc, axis=-1)
    # np.einsum("rij,rj->ri", R, dc) (trainer.py:292).  numpy's 2-lane SIMD
    # sum-of-products evaluates (r0*d0 + r2*d2) + r1*d1 without FMA; spelled
    # out so the oracle is machine-independent (pinned by the goldens).
    R = pose[:, :, :3]
    d = (R[:, :, 0] * dc[:, None, 0] + R[:, :, 2] * dc[:, None, 2]) + R[:, :, 1] * dc[:, None, 1]
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    o = pose[:, :, 3]
    valid = z > 0
    surf = z * to_t
    bmin, bmax = np.asarray(inst.aabb.min, np.float64), np.asarray(inst.aabb.max, np.float64)
    pad = bound_pad * (0.5 * (bmax - bmin))          # geometry.py:40-42
    pmin, pmax = bmin - pad, bmax + pad
    t0, t1, hit = ray_box(o, d, pmin, pmax)
    near = np.where(hit, np.maximum(t0, cfg.t_near), cfg.t_near)
    far = np.where(hit & (t1 > near), t1, cfg.t_far)
    t, ok = sample_along_rays(keyed_rng(seed, SAMPLES, inst.object_id, step), surf, valid, in_mask,
                              far, cfg, near=near)
    pts = o[:, None, :] + t[:, :, None] * d[:, None, :]
    enc = positional_encode(pts, 0.5 * (pmin + pmax), 0.5 * (pmax - pmin), arch, inst.pe_scale)
    out = dict(encoded=enc.astype(np.float32), t=t.astype(np.float32),
               target_depth=surf.astype(np.float32), target_colour=rgb.astype(np.float32),
               target_mask=in_mask, valid_depth=valid, ray_ok=ok)
    if with_aux:
        return out, dict(kf_idx=kf, u=u, v=v, in_mask=in_mask, origins=o, dirs=d, near=near,
                         far=far, t64=t, surface_t=surf)
    return out


def pad_batch(b: dict, rays: int, points: int, input_dim: int) -> dict:
    """Config 3: an object that drew fewer rays than the batch
    width is padded with the reference's zero-batch rows (trainer.py:190-200,
    ray_ok = False), which render.py:301-333 excludes from every loss and
    gradient term."""
    n = b["t"].shape[0]
    if n == rays:
        return b
    z = zero_batch(rays - n, points, input_dim)
    return {key: np.concatenate([b[key], z[key]]) for key in b}


def object_rays(inst, default: int) -> int:
    """Rays this instance draws: its own count (config 3) or the batch width."""
    n = getattr(inst, "n_rays", None)
    return int(n) if n else default


def stack_batches(batches: list) -> dict:
    """trainer.py:320-330."""
    return {key: np.stack([b[key] for b in batches]) for key in batches[0]}


@dataclass
class MapState:
    """The Mapper fields the step touches (trainer.py:203-222)."""
    intr: object
    objects: list             # instances in model-index order (model_to_object)
    background: object | None
    obj: Stack
    bg: Stack
    seed: int = 0
    rays_object: int = 120
    rays_background: int = 1200
    sampling: Sampling = field(default_factory=Sampling)
    bound_pad: float = 0.10
    w_colour: float = 5.0
    w_occ: float = 10.0
    train_background: bool = True
    global_step: int = 0


def map_update_step(ms: MapState) -> dict:
    """Mapper.train_step(mode="vectorised"), trainer.py:356-402.

    Returns {object_id: (L_depth, L_colour, L_occ)} like StepReport.losses.
    """
    step = ms.global_step
    out = {}
    pts = ms.sampling.n_stratified + ms.sampling.n_surface
    if ms.obj.count > 0:
        bs = []
        for k in range(ms.obj.count):
            if ms.obj.frozen[k]:
                bs.append(zero_batch(ms.rays_object, pts, ms.obj.arch.input_dim))
            else:
                nr = object_rays(ms.objects[k], ms.rays_object)
                b = assemble_batch(ms.objects[k], ms.intr, ms.obj.arch, nr, step, ms.seed, ms.sampling,
                                   ms.bound_pad)
                bs.append(pad_batch(b, ms.rays_object, pts, ms.obj.arch.input_dim))
        ld, lc, lo = train_on_batch(ms.obj, stack_batches(bs), ms.w_colour, ms.w_occ)
        for k in range(ms.obj.count):
            vals = (ld[k], lc[k], lo[k])
            oid = ms.objects[k].object_id
            if not all(np.isfinite(x) for x in vals):
                raise FloatingPointError(f"non-finite loss for object {oid}")
            out[oid] = tuple(float(x) for x in vals)
    bg = ms.background
    if ms.train_background and bg is not None:
        if ms.bg.frozen[bg.model_index]:
            b = zero_batch(ms.rays_background, pts, ms.bg.arch.input_dim)
        else:
            b = assemble_batch(bg, ms.intr, ms.bg.arch, ms.rays_background, step, ms.seed,
                               ms.sampling, ms.bound_pad)
        ld, lc, lo = train_on_batch(ms.bg, stack_batches([b]), ms.w_colour, ms.w_occ)
        vals = (ld[0], lc[0], lo[0])
        if not all(np.isfinite(x) for x in vals):
            raise FloatingPointError("non-finite loss for object 0")
        out[0] = tuple(float(x) for x in vals)
    ms.global_step += 1
    return out


# --------------------------------------------------------------------------
# forward-only inference (meshing.py) -- SURVEY 8f #1
# --------------------------------------------------------------------------

def _model_view(st: Stack, index: int) -> Stack:
    """StackedModelParams.model_view (models.py:90-98): one model as a stack."""
    v = st.copy()
    v.W = [w[index:index + 1] for w in st.W]
    v.b = [b[index:index + 1] for b in st.b]
    v.count = 1
    return v


def query_grid(st: Stack, model_index: int, bmin, bmax, pe_scale: float, resolution, chunk=None) -> np.ndarray:
    """meshing.py:64-97: occupancy on np.linspace grids (meshgrid 'ij'),
    f32 points encoded in f32 and run through the forward pass in chunks."""
    if isinstance(resolution, int):
        resolution = (resolution,) * 3
    if any(r < 2 for r in resolution):
        raise ValueError(f"grid resolution must be >= 2 per axis, got {resolution}")
    bmin, bmax = np.asarray(bmin, np.float64), np.asarray(bmax, np.float64)
    center, half = 0.5 * (bmin + bmax), 0.5 * (bmax - bmin)
    axes = [np.linspace(bmin[i], bmax[i], resolution[i]) for i in range(3)]
    view = _model_view(st, model_index)
    if chunk is None:
        chunk = 65536 if st.arch.hidden <= 64 else 16384
    n = int(np.prod(resolution))
    out = np.empty(n, np.float32)
    gx, gy, gz = np.meshgrid(*axes, indexing="ij")
    pts = np.stack([gx, gy, gz], axis=-1).reshape(-1, 3)
    for a in range(0, n, chunk):
        b = min(a + chunk, n)
        enc = positional_encode(pts[a:b].astype(np.float32), center, half, st.arch, pe_scale)
        occ, _, _, _ = mlp_forward(view, enc[None])
        out[a:b] = occ[0]
    return out.reshape(resolution)


def eval_field(st: Stack, model_index: int, bmin, bmax, pe_scale: float, points, chunk: int):
    """meshing.py:453-476 -> occupancy [N,S], colour [N,S,3]."""
    bmin, bmax = np.asarray(bmin, np.float64), np.asarray(bmax, np.float64)
    center, half = 0.5 * (bmin + bmax), 0.5 * (bmax - bmin)
    view = _model_view(st, model_index)
    n, s, _ = points.shape
    occ = np.empty((n, s), np.float32)
    col = np.empty((n, s, 3), np.float32)
    rows = max(1, chunk // max(s, 1))
    for a in range(0, n, rows):
        b = min(a + rows, n)
        enc = positional_encode(points[a:b].astype(np.float32), center, half, st.arch, pe_scale)
        o, c, _, _ = mlp_forward(view, enc.reshape(1, -1, enc.shape[-1]))
        occ[a:b] = o.reshape(b - a, s)
        col[a:b] = c.reshape(b - a, s, 3)
    return occ, col


def _midpoints(lo, hi, n):
    """meshing.py:479-482."""
    centres = (np.arange(n) + 0.5) / n
    return lo[:, None] + centres * (hi - lo)[:, None]


def _padded(bmin, bmax, fraction):
    bmin, bmax = np.asarray(bmin, np.float64), np.asarray(bmax, np.float64)
    pad = fraction * (0.5 * (bmax - bmin))
    return bmin - pad, bmax + pad


def render_view(obj: Stack, bg: Stack, objects, background, intr, pose, t_near=0.0, t_far=8.0,
                samples_object=48, samples_background=48, samples_refine=32, refine_window=0.25,
                bound_pad=0.10, threshold=0.5, chunk=65536):
    """meshing.py:485-579.  `objects`: instances (object_id, aabb, pe_scale,
    model_index) in ascending id order; `background` likewise.
    Returns (rgb [H,W,3] f32, depth [H,W] f32, instance [H,W] i32)."""
    w, h = intr.width, intr.height
    uu, vv = np.meshgrid(np.arange(w), np.arange(h))
    pix = np.stack([uu.ravel(), vv.ravel()], axis=1).astype(np.float64)
    n_pix = pix.shape[0]
    d_cam = np.empty((n_pix, 3))
    d_cam[:, 0] = (pix[:, 0] - intr.cx) / intr.fx
    d_cam[:, 1] = (pix[:, 1] - intr.cy) / intr.fy
    d_cam[:, 2] = 1.0
    scale = np.linalg.norm(d_cam, axis=-1)
    pose = np.asarray(pose, np.float64)
    dirs = d_cam @ pose[:3, :3].T
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    origins = np.broadcast_to(pose[:3, 3], dirs.shape)
    bmin, bmax = _padded(background.aabb.min, background.aabb.max, bound_pad)
    t_bg = _midpoints(np.full(n_pix, t_near), np.full(n_pix, t_far), samples_background)
    occ, col = eval_field(bg, background.model_index, bmin, bmax, background.pe_scale,
                          origins[:, None, :] + t_bg[:, :, None] * dirs[:, None, :], chunk)
    c_op, c_dep, c_col, _, _ = render_forward(occ, col, t_bg)
    if samples_refine > 0:
        centre = np.clip(c_dep, t_near + refine_window, t_far - refine_window)
        lo_r = np.maximum(centre - refine_window, t_near)
        hi_r = np.minimum(centre + refine_window, t_far)
        t_r = _midpoints(lo_r, hi_r, samples_refine)
        occ, col = eval_field(bg, background.model_index, bmin, bmax, background.pe_scale,
                              origins[:, None, :] + t_r[:, :, None] * dirs[:, None, :], chunk)
        _, r_dep, r_col, _, _ = render_forward(occ, col, t_r)
        use = c_op >= 0.5
        bg_depth = np.where(use, r_dep, c_dep)
        bg_col = np.where(use[:, None], r_col, c_col)
    else:
        bg_depth, bg_col = c_dep, c_col
    depth = bg_depth.astype(np.float64)
    colour = bg_col.astype(np.float64)
    instance = np.zeros(n_pix, np.int32)
    best = np.full(n_pix, np.inf)
    for inst in objects:
        omin, omax = _padded(inst.aabb.min, inst.aabb.max, bound_pad)
        t0, t1, hit = ray_box(origins, dirs, omin, omax)
        t0 = np.maximum(t0, t_near)
        sel = np.flatnonzero(hit & (t1 > t0))
        if sel.size == 0:
            continue
        t_o = _midpoints(t0[sel], t1[sel], samples_object)
        occ, col = eval_field(obj, inst.model_index, omin, omax, inst.pe_scale,
                              origins[sel, None, :] + t_o[:, :, None] * dirs[sel, None, :], chunk)
        op, dep, cl, _, _ = render_forward(occ, col, t_o)
        win = (op >= threshold) & (dep < best[sel])
        gi = sel[win]
        best[gi] = dep[win]
        depth[gi] = dep[win]
        colour[gi] = cl[win]
        instance[gi] = inst.object_id
    return (np.clip(colour, 0.0, 1.0).reshape(h, w, 3).astype(np.float32),
            (depth / scale).reshape(h, w).astype(np.float32), instance.reshape(h, w))


# --------------------------------------------------------------------------
# per-frame ingestion (objects.py:160-320, trainer.py:226-265) -- SURVEY 8f #2
# --------------------------------------------------------------------------

class Box:
    """AABB (geometry.py:10-46) with the fields the ingestion path uses."""

    def __init__(self, lo, hi):
        self.min = np.asarray(lo, np.float64).reshape(3)
        self.max = np.asarray(hi, np.float64).reshape(3)

    @property
    def volume(self):
        return float(np.prod(self.max - self.min))

    def union(self, o):
        return Box(np.minimum(self.min, o.min), np.maximum(self.max, o.max))


def from_points(points, trim=0.0, min_extent=1e-3) -> Box:
    """geometry.py:49-70."""
    pts = np.asarray(points, np.float64).reshape(-1, 3)
    if trim > 0.0 and pts.shape[0] > 10:
        lo = np.quantile(pts, trim, axis=0)
        hi = np.quantile(pts, 1.0 - trim, axis=0)
    else:
        lo, hi = pts.min(axis=0), pts.max(axis=0)
    thin = (hi - lo) < min_extent
    return Box(np.where(thin, lo - 0.5 * min_extent, lo), np.where(thin, hi + 0.5 * min_extent, hi))


def box_iou(a: Box, b: Box) -> float:
    """geometry.py:73-80."""
    lo, hi = np.maximum(a.min, b.min), np.minimum(a.max, b.max)
    if np.any(hi <= lo):
        return 0.0
    inter = float(np.prod(hi - lo))
    return inter / (a.volume + b.volume - inter)


def backproject(us, vs, z, intr, pose):
    """objects.py:160-167."""
    x = (us - intr.cx) / intr.fx * z
    y = (vs - intr.cy) / intr.fy * z
    return np.stack([x, y, z], axis=-1) @ pose[:3, :3].T + pose[:3, 3]


def extract_detections(depth, mask, intr, pose, classes, min_pixels=100, trim=0.02):
    """objects.py:170-217 -> [(class, bbox, n_valid, mask crop, Box)] in id order."""
    out = []
    for inst_id in np.unique(mask):
        if inst_id == 0:
            continue
        m = mask == inst_id
        valid = m & (depth > 0)
        n_valid = int(valid.sum())
        if n_valid < min_pixels:
            continue
        vs, us = np.nonzero(m)
        u0, u1, v0, v1 = int(us.min()), int(us.max()) + 1, int(vs.min()), int(vs.max()) + 1
        vv, uu = np.nonzero(valid)
        pts = backproject(uu.astype(np.float64), vv.astype(np.float64), depth[vv, uu], intr, pose)
        out.append(dict(cls=int(classes.get(int(inst_id), 1)), bbox=(u0, v0, u1, v1), n_pixels=n_valid,
                        mask=m[v0:v1, u0:u1], aabb=from_points(pts, trim=trim)))
    return out


def scene_bounds(depth, intr, pose, stride=4, trim=0.01):
    """objects.py:220-230."""
    d = depth[::stride, ::stride]
    vs, us = np.nonzero(d > 0)
    if vs.size < 16:
        return None
    pts = backproject((us * stride).astype(np.float64), (vs * stride).astype(np.float64), d[vs, us], intr, pose)
    return from_points(pts, trim=trim)


def associate_detections(dets, objects, iou_threshold=0.2):
    """objects.py:233-259 (objects: instances with object_id, cls, aabb)."""
    cand = []
    for di, det in enumerate(dets):
        for inst in objects:
            if inst.cls != det["cls"]:
                continue
            iou = box_iou(det["aabb"], inst.aabb)
            if iou >= iou_threshold:
                cand.append((-iou, inst.object_id, di))
    cand.sort()
    assigned, used = [None] * len(dets), set()
    for _, oid, di in cand:
        if assigned[di] is None and oid not in used:
            assigned[di] = oid
            used.add(oid)
    return assigned


class IngestMap:
    """The map bookkeeping process_frame mutates (trainer.py:226-265)."""

    def __init__(self, intr, stride_object=25, stride_background=50, margin=10, min_pixels=100, trim=0.02,
                 iou_threshold=0.2):
        self.intr = intr
        self.objects = []      # model-index order
        self.background = None
        self.next_id = 1
        self.cfg = dict(so=stride_object, sb=stride_background, margin=margin, min_pixels=min_pixels, trim=trim,
                        iou=iou_threshold)

    def process_frame(self, frame_id, rgb, depth, mask, pose, classes=None):
        c = self.cfg
        classes = classes or {}
        bounds = scene_bounds(depth, self.intr, pose)
        bg = self.background
        if bg is None:
            if bounds is None:
                raise ValueError(f"frame {frame_id}: no valid depth to bound the scene")
            bg = self.background = _NSI(object_id=0, cls=0, aabb=bounds, obs=0, kfs=[], is_bg=True)
        elif bounds is not None:
            bg.aabb = bg.aabb.union(bounds)
        bg.obs += 1
        h, w = depth.shape
        if (bg.obs - 1) % c["sb"] == 0:
            bg.kfs.append((frame_id, (0, 0, w, h)))
        dets = extract_detections(depth, mask, self.intr, pose, classes, c["min_pixels"], c["trim"])
        for det, oid in zip(dets, associate_detections(dets, self.objects, c["iou"])):
            if oid is None:
                inst = _NSI(object_id=self.next_id, cls=det["cls"], aabb=det["aabb"], obs=0, kfs=[], is_bg=False)
                self.next_id += 1
                self.objects.append(inst)
            else:
                inst = next(o for o in self.objects if o.object_id == oid)
                inst.aabb = inst.aabb.union(det["aabb"])
            inst.obs += 1
            if (inst.obs - 1) % c["so"] == 0:
                u0, v0, u1, v1 = det["bbox"]
                m = c["margin"]
                inst.kfs.append((frame_id, (max(u0 - m, 0), max(v0 - m, 0), min(u1 + m, w), min(v1 + m, h))))
        return dets, bounds


class _NSI:
    def __init__(self, **kw):
        self.__dict__.update(kw)
